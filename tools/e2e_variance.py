"""Per-call wall times of forward_stats at C3: device-resident vs from pageable
host arrays (the e2e path), to see the spread behind bench.py's e2e average.

    python tools/e2e_variance.py
"""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_2601_14821_b200 import device as D, rasterizer as R
from paper_2601_14821_b200.fixture import config_scene
from paper_2601_14821_b200.scene import Splats
splats, cams = config_scene("C3")
pert = splats.copy(); pert.opacities = pert.opacities * 0.97
targets = []
for t in R.render_targets(splats, cams):
    t.flags.writeable = False; targets.append(t)
host = Splats(*(np.array(getattr(pert, f), dtype=np.float64, copy=True) for f in ("positions", "sh", "opacities", "scales", "rotations")))
ds = D.DeviceSplats.from_host(host, D.current_device()); dt_ = D.targets_cache.get(targets, cams, D.current_device())
def t(fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); return (time.perf_counter() - t0) * 1e3
dev = [round(t(lambda: R.forward_stats_device(ds, cams, dt_)), 1) for _ in range(6)]
st = None
e2e = []
for _ in range(12):
    def f():
        global st
        st = R.forward_stats(host, cams, targets); _ = st.delta_mse[0]
    e2e.append(round(t(f), 1))
print("device", dev); print("e2e", e2e)
