"""Host -> device upload of the C3 splat arrays (1.42 GB): torch from pinned,
torch from pageable, and potr_copy_to_device from pageable; checks the bytes."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2601_14821_b200 import device as D  # noqa: E402

n = 3_000_000
rng = np.random.default_rng(0)
arrs = [rng.standard_normal((n, k)) for k in (3, 48, 1, 3, 4)]
dev = D.current_device()
ctx = D.context()


def run(kind):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    outs = []
    for a in arrs:
        if kind == "torch_pageable":
            outs.append(torch.from_numpy(a).to(dev))
        elif kind == "torch_pinned":
            outs.append(pinned[id(a)].to(dev, non_blocking=True))
        else:
            d = torch.empty(a.shape, dtype=torch.float64, device=dev)
            ctx.call("potr_copy_to_device", D.ptr(d), ctypes.c_void_p(a.ctypes.data),
                     ctypes.c_int64(a.nbytes))
            outs.append(d)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    ok = all(np.array_equal(o.cpu().numpy(), a) for o, a in zip(outs, arrs))
    gb = sum(a.nbytes for a in arrs) / 1e9
    print(f"{kind}: {dt * 1e3:.1f} ms, {gb / dt:.1f} GB/s, bytes ok: {ok}", flush=True)


pinned = {id(a): torch.from_numpy(a).pin_memory() for a in arrs}
for k in ("torch_pinned", "torch_pageable", "potr_copy_to_device"):
    run(k)
    run(k)
