"""The two forms of the SH normal equations (include/potr_b200.h):
potr_sh_normal_equations overwrites, potr_sh_accumulate adds (for callers
that sum view shards).  Overwrite == accumulate into zeros, bit for bit; a
second accumulate doubles every entry exactly; the overwrite form ignores
whatever the buffer held."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_normal_equations_overwrite_vs_accumulate(cuda):
    import torch
    from paper_2601_14821_b200 import _native, device as D, rasterizer as R
    from paper_2601_14821_b200.fixture import make_fixture
    splats, cams = make_fixture(num_splats=5000, num_cameras=40, seed=3, width=64, height=48)
    ds = D.DeviceSplats.from_host(splats, cuda)
    _, ci, _, _ = R.forward_stats_device(ds, cams, None)
    n, S = ds.n, len(cams)
    ctx = D.context()
    cam_arr = _native.camera_array(cams)

    def run(name, init):
        neq = torch.full((_native.NEQ_STRIDE, n), init, dtype=torch.float64, device=cuda)
        ctx.call(name, ctypes.byref(ds.struct()), S, cam_arr, D.ptr(ci), D.ptr(neq))
        return neq

    acc = run("potr_sh_accumulate", 0.0)
    over = run("potr_sh_normal_equations", float("nan"))  # old contents must not matter
    assert torch.equal(acc, over)
    ctx.call("potr_sh_accumulate", ctypes.byref(ds.struct()), S, cam_arr, D.ptr(ci), D.ptr(acc))
    assert torch.equal(acc, 2.0 * over)
    assert float(over[184].min()) >= 0 and np.isfinite(over.cpu().numpy()).all()
