"""device.TargetCache: which target arrays may be served from the device copy
made on an earlier call (the reference freezes its targets, rasterizer.py:
375-376; read-only alone does not make an array immutable).  CPU-only: the
cache logic with device='cpu' and small arrays."""

import numpy as np
import torch

from paper_2601_14821_b200.device import TargetCache
from paper_2601_14821_b200.fixture import camera_ring


def _cams():
    return camera_ring(2, width=6, height=4)


def _targets(writeable=False):
    ts = [np.random.default_rng(i).random((4, 6, 3)) for i in range(2)]
    for t in ts:
        t.flags.writeable = writeable
    return ts


def test_frozen_arrays_are_cached():
    c, cams, ts = TargetCache(), _cams(), _targets()
    a = c.get(ts, cams, torch.device("cpu"))
    b = c.get(ts, cams, torch.device("cpu"))
    assert all(x is y for x, y in zip(a, b))
    assert torch.equal(b[0], torch.from_numpy(ts[0]))


def test_writable_arrays_are_reuploaded():
    c, cams, ts = TargetCache(), _cams(), _targets(writeable=True)
    a = c.get(ts, cams, torch.device("cpu"))
    ts[0][0, 0, 0] = 42.0
    b = c.get(ts, cams, torch.device("cpu"))
    assert float(b[0][0, 0, 0]) == 42.0 and a[0] is not b[0]


def test_read_only_view_of_writable_base_is_not_cached():
    c, cams = TargetCache(), _cams()
    bases = [np.random.default_rng(i).random((4, 6, 3)) for i in range(2)]
    views = [b[:] for b in bases]
    for v in views:
        v.flags.writeable = False
    c.get(views, cams, torch.device("cpu"))
    bases[1][1, 1, 1] = -7.0  # the view changes under the cache
    out = c.get(views, cams, torch.device("cpu"))
    assert float(out[1][1, 1, 1]) == -7.0


def test_refrozen_modified_array_is_reuploaded():
    c, cams, ts = TargetCache(), _cams(), _targets()
    c.get(ts, cams, torch.device("cpu"))
    ts[0].flags.writeable = True
    ts[0][...] = 0.5
    ts[0].flags.writeable = False
    out = c.get(ts, cams, torch.device("cpu"))
    assert torch.equal(out[0], torch.full((4, 6, 3), 0.5, dtype=torch.float64))
