"""The library's hand-written primitives (csrc/sort.cu) against numpy: the
stable LSD radix sort (every bit width the pipeline uses goes through the
bit-exact depth-order / tile-list / records tests; here the raw entry point
with adversarial key distributions) and the device removal order of the
pruning controller (pruning.py:80-83, np.argsort(mapping_m(...),
kind="stable"))."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev(cuda):
    return cuda


def _sort(keys, vals, begin, end):
    import torch
    from paper_2601_14821_b200 import device as D
    k = torch.from_numpy(keys.copy()).to("cuda")
    v = torch.from_numpy(vals.copy()).to("cuda")
    D.context().call("potr_sort_pairs_u64", ctypes.c_int64(len(keys)), D.ptr(k), D.ptr(v),
                     begin, end)
    return k.cpu().numpy(), v.cpu().numpy()


@pytest.mark.parametrize("n,kind", [(1, "rand"), (4095, "rand"), (4097, "few"),
                                    (1_000_003, "rand"), (3_000_000, "few"), (777_777, "const"),
                                    (2_000_000, "skew")])
def test_radix_sort_stable_vs_numpy(dev, n, kind):
    rng = np.random.default_rng(n)
    if kind == "rand":
        keys = rng.integers(0, 2**63, n, dtype=np.uint64) * np.uint64(2) + \
            rng.integers(0, 2, n, dtype=np.uint64)
    elif kind == "few":
        keys = rng.integers(0, 7, n).astype(np.uint64) << np.uint64(40)
    elif kind == "const":
        keys = np.full(n, 0xDEADBEEF12345678, dtype=np.uint64)
    else:  # a few heavy digits plus a uniform tail
        keys = np.where(rng.uniform(size=n) < 0.9, rng.integers(0, 3, n),
                        rng.integers(0, 2**20, n)).astype(np.uint64)
    vals = np.arange(n, dtype=np.int64)
    for begin, end in ((0, 64), (0, 24), (8, 48)):
        sk, sv = _sort(keys, vals, begin, end)
        mask = np.uint64(((1 << (end - begin)) - 1) << begin) if end - begin < 64 else \
            np.uint64(2**64 - 1)
        order = np.argsort(keys & mask, kind="stable")
        assert np.array_equal(sv, order), (begin, end)
        assert np.array_equal(sk, keys[order])


def test_removal_order_matches_numpy(dev):
    import torch
    from paper_2601_14821_b200 import device as D, pruning
    rng = np.random.default_rng(5)
    n = 500_000
    dmax = 10.0 ** -9.8
    dm = rng.standard_normal(n) * dmax * rng.choice([1e-6, 1e-2, 1.0, 10.0], n)
    dm[::97] = 0.0
    dm[::89] = -0.0
    dm[1000:1100] = dm[2000]           # exact ties
    dm[5:50] = -dm[60:105]
    cand = np.nonzero(dm < dmax)[0]
    ref = cand[np.argsort(pruning.mapping_m(dm[cand] / dmax, 10.0), kind="stable")]
    got = pruning._removal_order_device(torch.from_numpy(dm).to("cuda"),
                                        torch.from_numpy(cand).to("cuda"), dmax, 10.0)
    assert np.array_equal(D.to_host(got), ref)
    full = pruning._removal_order_device(torch.from_numpy(dm).to("cuda"), None, dmax, 3.0)
    assert np.array_equal(D.to_host(full), pruning.removal_order(dm, dmax, 3.0))


def test_multi_group_tile_sort_vs_oracle_and_batch1(dev, oracle):
    """800x600 views have 15,000 tiles of 8x4, so an 8-view batch bins in two
    16-bit tile-sort groups (4 views each, pair indices offset by the group
    start): scores equal the single-view batches' bit for bit and the
    oracle's within the parity tolerance."""
    from paper_2601_14821_b200 import _native, device as D, rasterizer as R
    from paper_2601_14821_b200.fixture import make_fixture
    from tests.conftest import perturbed
    splats, cams = make_fixture(20000, 8, 4, width=800, height=600)
    targets = R.render_targets(splats, cams)
    pert = perturbed(splats)
    st8 = R.compute_delta_mse(pert, cams, targets)
    ctx = D.context()
    try:
        ctx.call("potr_set_option", _native.OPT_VIEW_BATCH, 1)
        st1 = R.compute_delta_mse(pert, cams, targets)
    finally:
        ctx.call("potr_set_option", _native.OPT_VIEW_BATCH, 8)
    assert np.array_equal(st8.importance, st1.importance)
    assert np.array_equal(st8.delta_mse, st1.delta_mse)
    imp, _, dm, mse = oracle.forward_stats(pert, cams, [np.asarray(t) for t in targets],
                                           threads=8)
    np.testing.assert_allclose(st8.importance, imp, rtol=1e-12, atol=1e-20)
    np.testing.assert_allclose(st8.delta_mse, dm, rtol=1e-9, atol=1e-22)


def test_staged_pageable_upload_bit_exact(dev):
    """potr_copy_to_device (pageable host -> device through the pinned ring):
    back-to-back calls whose sizes are not multiples of the ring chunk, so a
    call refills buffers whose previous DMA may still be in flight."""
    import torch
    from paper_2601_14821_b200 import device as D
    rng = np.random.default_rng(3)
    arrs = [rng.standard_normal(m) for m in (13_000_001, 4_194_305, 40_000_003, 9_999_999)]
    outs = [D.to_device(a, dev) for a in arrs]  # >= 8 MB pageable: the staged path
    torch.cuda.synchronize()
    for o, a in zip(outs, arrs):
        assert np.array_equal(o.cpu().numpy(), a)
