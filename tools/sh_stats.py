"""Distribution of the SH solve sizes at C3: |kept| after the parallel-column
sparsification (compaction.py:110-124), emulated in torch from the device
normal equations."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_14821_b200 import _native, device as D, rasterizer as R  # noqa: E402
from paper_2601_14821_b200.fixture import config_scene  # noqa: E402

splats, cams = config_scene(sys.argv[1] if len(sys.argv) > 1 else "C3")
dev = D.current_device()
ds = D.DeviceSplats.from_host(splats, dev)
ctx = D.context()
imp, ci, _, _ = R.forward_stats_device(ds, cams, None)
n, S = ds.n, len(cams)
neq = torch.empty((_native.NEQ_STRIDE, n), dtype=torch.float64, device=dev)
ctx.call("potr_sh_normal_equations", ctypes.byref(ds.struct()), S, _native.camera_array(cams),
         D.ptr(ci), D.ptr(neq))
tri = lambda i, j: i * 16 - (i * (i - 1)) // 2 + (j - i)  # noqa: E731
norms = torch.stack([neq[tri(i, i)].sqrt() for i in range(16)], 1)
kept = torch.zeros((n, 16), dtype=torch.bool, device=dev)
kept[:, 0] = True
for i in range(1, 16):
    par = torch.zeros(n, dtype=torch.bool, device=dev)
    for j in range(i):
        cs = neq[tri(j, i)].abs() / (norms[:, i] * norms[:, j])
        par |= kept[:, j] & (cs > 0.8175744761936437)
    kept[:, i] = (norms[:, i] != 0) & ~par
seen = neq[184] > 0
m = kept.sum(1)[seen]
print("seen splats", int(seen.sum()), "mean |kept|", float(m.double().mean()))
print("histogram of |kept| (1..16):", torch.bincount(m, minlength=17)[1:].tolist())
print("seen views: mean", float(neq[184][seen].mean()))
