"""Overlapped splat upload (potr_upload_async + the scoring loop's lookahead):
forward_stats from host arrays bins its first view batches while the SH rows
are still on their way, each batch in its own buffer set, and colours them
once the rows are in.  None of that may change a bit of the result: compared
here against the same call on device-resident splats, across lookahead
depths, view-batch sizes, depth-key modes, record layouts, pinned and pageable
sources, and through the host C ABI."""

import ctypes

import numpy as np
import pytest

from tests.conftest import perturbed

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def scene(cuda):
    from paper_2601_14821_b200.fixture import make_fixture
    # 40k splats: 15 MB of SH rows, over the 8 MB async threshold
    splats, cams = make_fixture(num_splats=40_000, num_cameras=22, seed=5, width=96, height=72)
    from paper_2601_14821_b200 import rasterizer as R
    targets = R.render_targets(splats, cams)
    return perturbed(splats), cams, targets


def _device_reference(splats, cams, targets):
    """forward_stats on device-resident splats: no pending upload."""
    from paper_2601_14821_b200 import device as D
    from paper_2601_14821_b200 import rasterizer as R
    dev = D.current_device()
    ds = D.DeviceSplats.from_host(splats, dev, async_sh=False)
    dt = D.targets_cache.get(targets, cams, dev)
    imp, ci, dm, mse = R.forward_stats_device(ds, cams, dt)
    return (D.to_host(imp), D.to_host(ci), D.to_host(dm), float(D.to_host(mse)[0]))


def _same(st, ref):
    imp, ci, dm, mse = ref
    assert np.array_equal(st.importance, imp)
    assert np.array_equal(np.asarray(st.camera_importance), ci)
    assert np.array_equal(st.delta_mse, dm)
    assert st.mse == mse


@pytest.mark.parametrize("lookahead,batch,keys,spatial", [
    (6, 8, 0, 1), (1, 8, 0, 1), (3, 2, 0, 1), (8, 1, 0, 1), (4, 3, 1, 1), (2, 5, 2, 0),
    (5, 4, 0, 0)])
def test_async_upload_bit_identical(scene, lookahead, batch, keys, spatial):
    from paper_2601_14821_b200 import _native, device as D
    from paper_2601_14821_b200 import rasterizer as R
    splats, cams, targets = scene
    ctx = D.context()
    try:
        ctx.call("potr_set_option", _native.OPT_LOOKAHEAD, lookahead)
        ctx.call("potr_set_option", _native.OPT_VIEW_BATCH, batch)
        ctx.call("potr_set_option", _native.OPT_RAW_DEPTH_KEYS, keys)
        ctx.call("potr_set_option", _native.OPT_SPATIAL_RECORDS, spatial)
        ref = _device_reference(splats, cams, targets)
        st = R.forward_stats(splats, cams, targets)  # pageable host arrays: async SH
        _same(st, ref)
        st2 = R.forward_stats(splats, cams, targets)  # the sets are reused
        _same(st2, ref)
    finally:
        ctx.call("potr_set_option", _native.OPT_LOOKAHEAD, 6)
        ctx.call("potr_set_option", _native.OPT_VIEW_BATCH, 8)
        ctx.call("potr_set_option", _native.OPT_RAW_DEPTH_KEYS, 0)
        ctx.call("potr_set_option", _native.OPT_SPATIAL_RECORDS, 1)


def test_async_upload_pinned_source_and_importance_only(scene):
    import torch
    from paper_2601_14821_b200 import rasterizer as R
    from paper_2601_14821_b200.scene import Splats
    splats, cams, targets = scene
    ref = _device_reference(splats, cams, targets)
    pin = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
           for a in (splats.positions, splats.sh, splats.opacities, splats.scales,
                     splats.rotations)]
    st = R.forward_stats(Splats(*pin), cams, targets)
    _same(st, ref)
    imp_only = R.compute_importance(splats, cams)[0]
    assert np.array_equal(imp_only, ref[0])


def test_pending_upload_completed_by_other_entry_points(scene):
    """A pending upload is completed by whatever library call comes next."""
    import torch
    from paper_2601_14821_b200 import device as D
    from paper_2601_14821_b200 import rasterizer as R
    splats, cams, _ = scene
    dev = D.current_device()
    ds = D.DeviceSplats.from_host(splats, dev, async_sh=True)
    assert ds._pending_host is not None
    img = R.render_image(ds, cams[0])  # render path: joins before reading sh
    ref = R.render_image(splats, cams[0])
    assert np.array_equal(img, ref)
    ds.wait_upload()
    assert torch.equal(ds.sh.cpu(), torch.from_numpy(np.asarray(splats.sh).reshape(-1, 3, 16)))


def test_host_c_abi_overlapped(scene):
    """potr_forward_stats_host (which uploads its SH rows asynchronously)."""
    from paper_2601_14821_b200 import _native, device as D
    splats, cams, targets = scene
    ref = _device_reference(splats, cams, targets)
    n, S = len(splats.positions), len(cams)
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in
            (splats.positions, splats.sh, splats.opacities, splats.scales, splats.rotations)]
    tg = [np.ascontiguousarray(t, dtype=np.float64) for t in targets]
    tptr = (ctypes.c_void_p * S)(*[t.ctypes.data for t in tg])
    imp, ci, dm, mse = np.empty(n), np.empty((S, n)), np.empty(n), np.empty(1)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    D.context().call("potr_forward_stats_host", ctypes.c_int64(n), *map(p, arrs), S,
                     _native.camera_array(cams), tptr, p(imp), p(ci), p(dm), p(mse))
    assert np.array_equal(imp, ref[0]) and np.array_equal(ci, ref[1])
    assert np.array_equal(dm, ref[2]) and float(mse[0]) == ref[3]
