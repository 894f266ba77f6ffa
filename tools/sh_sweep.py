"""SH recompute at the C3 / C4 shape over a lambda sweep: AC sparsity and the
device time of the accumulate (once) and of the solve (per lambda).

    python tools/sh_sweep.py [lambda ...]
"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2601_14821_b200 import _native, device as D, rasterizer as R  # noqa: E402
from paper_2601_14821_b200.fixture import config_scene  # noqa: E402

lams = [float(x) for x in sys.argv[1:]] or [1e-7, 1e-9, 1e-10, 1e-11, 1e-12, 1e-13, 1e-14]
splats, cams = config_scene("C3")
dev = D.current_device()
ds = D.DeviceSplats.from_host(splats, dev)
ctx = D.context()
imp, ci, _, _ = R.forward_stats_device(ds, cams, None)
n, S = ds.n, len(cams)
neq = torch.empty((_native.NEQ_STRIDE, n), dtype=torch.float64, device=dev)
rgb = torch.empty((n, 3, 16), dtype=torch.float64, device=dev)
yc = torch.empty((n, 3, 16), dtype=torch.float64, device=dev)
status = torch.empty(n, dtype=torch.int8, device=dev)
cam_arr = _native.camera_array(cams)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.call("potr_sh_normal_equations", ctypes.byref(ds.struct()), S, cam_arr, D.ptr(ci), D.ptr(neq))
    torch.cuda.synchronize()
    t_acc = time.perf_counter() - t0
seen = float(neq[184].mean().item())
print(f"accumulate {t_acc * 1e3:.1f} ms; seen views per splat {seen:.1f} of {S} ({seen / S:.2f})")
for lam in lams:
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.call("potr_sh_solve", ctypes.byref(ds.struct()), D.ptr(neq), ctypes.c_double(lam),
                 ctypes.c_double(0.8175744761936437), ctypes.c_double(0.5 / 51.0), D.ptr(rgb),
                 D.ptr(yc), D.ptr(status))
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
    sp = float((yc[:, :, 1:] == 0).double().mean().item())
    st = torch.bincount(status.to(torch.int64), minlength=4).tolist()
    print(f"lambda {lam:g}: solve {t * 1e3:.1f} ms, AC sparsity {sp:.4f}, status {st}")
