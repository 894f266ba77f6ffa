"""CUDA path vs golden vectors (reference outputs) and the CPU oracle.

Tolerances (SURVEY.md 8a / BASELINE north_star): splat order, tile keys,
projection and prune mask bit-exact; per-splat scores within 1e-4 relative
(we hold them to 1e-9: the path is fp64); SH coefficients and AC sparsity
within 1e-4 absolute; PSNR after pruning within 0.01 dB.
"""

import numpy as np
import pytest

from tests.conftest import (c3_scene, golden, oracle_scene, perturbed, score_close, sh_scene,
                            small_scene)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R(cuda):
    from paper_2601_14821_b200 import rasterizer
    return rasterizer


@pytest.fixture(scope="module")
def C(cuda):
    from paper_2601_14821_b200 import compaction
    return compaction


def test_native_library_is_loaded(R):
    import paper_2601_14821_b200._native as N
    from paper_2601_14821_b200 import device
    ctx = device.context()
    assert N._lib is not None
    before = ctx.launches()
    splats, cams = small_scene()
    R.render_image(splats, cams[0])
    assert ctx.launches() > before


def test_projection_bit_exact(R):
    splats, cams = small_scene()
    g = golden("small_scene")
    p = R.project_splats(splats, cams[0])
    assert np.array_equal(p.valid, g["proj_valid"])
    assert np.array_equal(p.mean2d, g["proj_mean2d"])
    assert np.array_equal(p.cov2d, g["proj_cov2d"])
    assert np.array_equal(p.view_depth, g["proj_depth"])
    assert np.array_equal(p.radius, g["proj_radius"])
    ids = g["colors0_ids"]
    col = R.splat_colors(splats.subset(ids), cams[0])
    np.testing.assert_allclose(col, g["colors0"], rtol=0, atol=1e-15)


def test_binning_bit_exact(R, oracle):
    """(tile, depth, id) lists of the GPU binning == the reference-derived lists."""
    from paper_2601_14821_b200 import binning
    splats, cams = small_scene()
    g = golden("small_scene")
    for c in (0, 1):
        order, offsets, lists = binning.tile_lists(splats, cams[c])
        assert np.array_equal(order, g[f"order{c}"])
        assert np.array_equal(offsets, g[f"tile_offsets{c}"])
        assert np.array_equal(lists, g[f"tile_splats{c}"])
    # a larger scene against the oracle restatement
    from paper_2601_14821_b200.fixture import make_fixture
    big, bc = make_fixture(60000, 2, 1, width=320, height=200)
    for cam in bc:
        order, offsets, lists = binning.tile_lists(big, cam)
        assert np.array_equal(order, oracle.depth_order(big, cam))
        off, lst = oracle.tile_lists(big, cam)
        assert np.array_equal(offsets, off)
        assert np.array_equal(lists, lst)


def test_render_targets(R):
    splats, cams = small_scene()
    g = golden("small_scene")
    imgs = R.render_targets(splats, cams)
    for s, img in enumerate(imgs):
        assert not img.flags.writeable
        np.testing.assert_allclose(img, g["targets"][s], rtol=0, atol=1e-14)


def test_forward_stats_small_scene(R):
    splats, cams = small_scene()
    g = golden("small_scene")
    targets = [t for t in g["targets"]]
    st = R.compute_delta_mse(perturbed(splats), cams, targets)
    np.testing.assert_allclose(st.importance, g["pert_importance"], rtol=1e-12, atol=1e-20)
    np.testing.assert_allclose(np.asarray(st.camera_importance), g["pert_camera_importance"],
                               rtol=1e-12, atol=1e-20)
    np.testing.assert_allclose(st.delta_mse, g["pert_delta_mse"], rtol=1e-9, atol=1e-22)
    assert score_close(st.delta_mse, g["pert_delta_mse"], rel=1e-4)
    assert st.mse == pytest.approx(float(g["pert_mse"]), rel=1e-12)
    st0 = R.compute_delta_mse(splats, cams, targets)
    np.testing.assert_allclose(st0.delta_mse, g["it1_delta_mse"], rtol=1e-9, atol=1e-22)
    imp, ci = R.compute_importance(splats, cams)
    np.testing.assert_allclose(imp, g["importance"], rtol=1e-12, atol=1e-20)
    np.testing.assert_allclose(np.asarray(ci), g["camera_importance"], rtol=1e-12, atol=1e-20)


@pytest.mark.parametrize("batch,raw", [(1, 0), (3, 0), (8, 1), (5, 1), (8, 2), (2, 2)])
def test_view_batching_and_key_modes_bit_identical(R, batch, raw):
    """Batch size and depth-key encoding never change a bit of the result."""
    from paper_2601_14821_b200 import _native, device
    splats, cams = small_scene()
    g = golden("small_scene")
    targets = [t for t in g["targets"]]
    ref = R.compute_delta_mse(perturbed(splats), cams, targets)
    ctx = device.context()
    try:
        ctx.call("potr_set_option", _native.OPT_VIEW_BATCH, batch)
        ctx.call("potr_set_option", _native.OPT_RAW_DEPTH_KEYS, raw)
        st = R.compute_delta_mse(perturbed(splats), cams, targets)
        from paper_2601_14821_b200 import binning
        order, off, lst = binning.tile_lists(splats, cams[0])
    finally:
        ctx.call("potr_set_option", _native.OPT_VIEW_BATCH, 8)
        ctx.call("potr_set_option", _native.OPT_RAW_DEPTH_KEYS, 0)
    assert np.array_equal(st.delta_mse, ref.delta_mse)
    assert np.array_equal(st.importance, ref.importance)
    assert np.array_equal(np.asarray(st.camera_importance), np.asarray(ref.camera_importance))
    assert st.mse == ref.mse
    assert np.array_equal(order, g["order0"]) and np.array_equal(lst, g["tile_splats0"])


def test_spatial_records_bit_identical(R, oracle):
    """The Morton record layout (POTR_OPT_SPATIAL_RECORDS) only moves records
    in HBM: scores, renders, records and tile lists are bit-identical with it
    off, and exact depth ties (duplicated splats) still break by ascending id."""
    from paper_2601_14821_b200 import _native, binning, device
    splats, cams = small_scene()
    g = golden("small_scene")
    targets = [t for t in g["targets"]]
    tied = splats.copy()
    for f in ("positions", "scales", "rotations", "sh", "opacities"):
        getattr(tied, f)[700:760] = getattr(tied, f)[100:160]   # exact duplicates
    # a run of 100 equal depth keys: longer than the run fixup takes, so the
    # batch falls back to the 64-bit sort in splat order
    stack = splats.copy()
    for f in ("positions", "scales", "rotations", "sh", "opacities"):
        getattr(stack, f)[200:300] = getattr(stack, f)[50]
    # every centre at one point: zero extent for the Morton code, one run of
    # equal depths across the whole view
    point = splats.copy()
    point.positions[:] = point.positions[7]
    ctx = device.context()

    def run(sc):
        st = R.compute_delta_mse(perturbed(sc), cams, targets)
        rec = R.render_with_records(sc, cams[1])
        return st, rec, binning.tile_lists(sc, cams[0])

    outs = {}
    try:
        for on in (0, 1):
            ctx.call("potr_set_option", _native.OPT_SPATIAL_RECORDS, on)
            outs[on] = [run(splats), run(tied), run(stack), run(point)]
    finally:
        ctx.call("potr_set_option", _native.OPT_SPATIAL_RECORDS, 1)
    for (st0, rec0, tl0), (st1, rec1, tl1) in zip(outs[0], outs[1]):
        assert np.array_equal(st0.delta_mse, st1.delta_mse)
        assert np.array_equal(st0.importance, st1.importance)
        assert np.array_equal(np.asarray(st0.camera_importance), np.asarray(st1.camera_importance))
        assert st0.mse == st1.mse
        for f in ("image", "transmittance", "splat_ids", "pixels", "alphas", "trans_at",
                  "partials", "colors"):
            assert np.array_equal(getattr(rec0, f), getattr(rec1, f)), f
        for a, b in zip(tl0, tl1):
            assert np.array_equal(a, b)
    for sc, out in ((tied, outs[1][1]), (stack, outs[1][2]), (point, outs[1][3])):
        order, off, lst = out[2]
        assert np.array_equal(order, oracle.depth_order(sc, cams[0]))
        o_off, o_lst = oracle.tile_lists(sc, cams[0])
        assert np.array_equal(off, o_off) and np.array_equal(lst, o_lst)


def test_score_rows_sum_to_fused_sums(R):
    """potr_score_views_rows' per-view rows, added in camera order (what the
    ordered multi-GPU chain does), equal potr_score_views' sums bit for bit."""
    import torch
    from paper_2601_14821_b200 import distributed, device
    splats, cams = small_scene()
    g = golden("small_scene")
    targets = [t for t in g["targets"]]
    pert = perturbed(splats)
    ci, dm_rows, mse_rows = distributed._gpu_score_rows(pert, cams, targets)
    n = len(pert.positions)
    acc = torch.zeros(2 * n + 1, dtype=torch.float64, device=ci.device)
    for v in range(len(cams)):
        acc[:n] += ci[v]
        acc[n:2 * n] += dm_rows[v]
        acc[2 * n:] += mse_rows[v:v + 1]
    st = R.compute_delta_mse(pert, cams, targets)
    host = distributed.finalize_sums(acc, n, len(cams)).cpu().numpy()
    assert np.array_equal(host[:n], st.importance)
    assert np.array_equal(host[n:2 * n], st.delta_mse)
    assert float(host[2 * n]) == st.mse
    assert np.array_equal(ci.cpu().numpy(), np.asarray(st.camera_importance))


def test_render_and_score_in_one_pass(R):
    """render_targets + compute_delta_mse against those targets == the fused
    self-target pass, bit for bit (the first scoring of an encode)."""
    from paper_2601_14821_b200.fixture import make_fixture
    for splats, cams in (small_scene(), make_fixture(20000, 10, 4, width=96, height=72)):
        tg = R.render_targets(splats, cams)
        st = R.compute_delta_mse(splats, cams, tg)
        tg2, st2 = R.render_targets_and_delta_mse(splats, cams)
        for a, b in zip(tg, tg2):
            assert np.array_equal(a, b) and not b.flags.writeable
        assert np.array_equal(st.importance, st2.importance)
        assert np.array_equal(st.delta_mse, st2.delta_mse)
        assert np.array_equal(np.asarray(st.camera_importance), np.asarray(st2.camera_importance))
        assert st.mse == st2.mse == 0.0


def test_forward_stats_bit_reproducible(R):
    splats, cams = small_scene()
    g = golden("small_scene")
    targets = [t for t in g["targets"]]
    runs = [R.compute_delta_mse(perturbed(splats), cams, targets, threads=t) for t in (1, 4, 1)]
    for other in runs[1:]:
        assert np.array_equal(runs[0].delta_mse, other.delta_mse)
        assert np.array_equal(runs[0].importance, other.importance)
        assert runs[0].mse == other.mse


def test_oracle_scenes(R):
    o = golden("oracle_scenes")
    for seed in range(20):
        splats, cams = oracle_scene(seed)
        targets = R.render_targets(splats, cams)
        np.testing.assert_allclose(targets[0], o[f"s{seed}_image0"], rtol=0, atol=1e-14)
        st = R.compute_delta_mse(perturbed(splats), cams, targets)
        np.testing.assert_allclose(st.importance, o[f"s{seed}_importance"], rtol=1e-12,
                                   atol=1e-20)
        np.testing.assert_allclose(st.delta_mse, o[f"s{seed}_delta_mse"], rtol=1e-9,
                                   atol=1e-22)


def test_records_mode(R):
    from paper_2601_14821_b200.fixture import random_scene
    g = golden("records")
    splats, cams = random_scene(4, num_splats=20)
    rec = R.render_with_records(splats, cams[0])
    assert np.array_equal(rec.splat_ids, g["splat_ids"])
    assert np.array_equal(rec.pixels, g["pixels"])
    np.testing.assert_allclose(rec.alphas, g["alphas"], rtol=1e-14, atol=0)
    np.testing.assert_allclose(rec.trans_at, g["trans_at"], rtol=1e-13, atol=0)
    np.testing.assert_allclose(rec.partials, g["partials"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(rec.colors, g["colors"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(rec.prune_deltas(), g["prune_deltas"], rtol=0, atol=1e-13)


def test_c1_config(R):
    from paper_2601_14821_b200.fixture import make_fixture
    g = golden("c1")
    splats, cams = make_fixture(10000, 8, 0, 128)
    targets = R.render_targets(splats, cams)
    st = R.compute_delta_mse(perturbed(splats), cams, targets)
    np.testing.assert_allclose(st.importance, g["pert_importance"], rtol=1e-11, atol=1e-20)
    np.testing.assert_allclose(st.delta_mse, g["pert_delta_mse"], rtol=1e-8, atol=1e-20)
    st0 = R.compute_delta_mse(splats, cams, targets)
    np.testing.assert_allclose(st0.delta_mse, g["it1_delta_mse"], rtol=1e-8, atol=1e-20)


def test_prune_mask_bit_exact_and_psnr(R):
    """The reference controller's 48 iterations driven by GPU scores reproduce
    the reference's kept set exactly; PSNR of the pruned renders within 0.01 dB."""
    from paper_2601_14821_b200 import pruning
    from paper_2601_14821_b200.metrics import psnr
    splats, cams = small_scene()
    g = golden("small_scene")
    targets = R.render_targets(splats, cams)
    cfg = pruning.PruneConfig(delta_mse_max=10.0 ** (-8.8 - 2.0 * 0.5))
    pruned, kept, reports = pruning.run_pruning(splats, cams, targets, cfg)
    assert np.array_equal(kept, g["prune_kept"])
    assert np.array_equal([r.removed for r in reports], g["prune_removed"])
    for s, cam in enumerate(cams):
        ours = R.render_image(pruned, cam)
        ref = g["pruned_images"][s]
        assert abs(psnr(ours, targets[s]) - psnr(ref, g["targets"][s])) <= 0.01


@pytest.mark.parametrize("config,q,iters", [("C1", 0.9, 6), ("C2", 0.5, 8)])
def test_prune_device_controller_matches_host_controller(R, monkeypatch, config, q, iters):
    """The device-resident controller (splats subset in HBM, GPU stable sort)
    and the host controller over the same GPU scores give identical reports,
    kept sets and pruned splats, on a scene with many removals per iteration
    (C1) and at the C2 shape (300k splats, 100 views at 800x800)."""
    from paper_2601_14821_b200 import pruning, fixture
    splats, cams = fixture.config_scene(config)
    targets = R.render_targets(splats, cams)
    cfg = pruning.PruneConfig(delta_mse_max=10.0 ** (-8.8 - 2.0 * q), iterations=iters)
    assert pruning._device_scorer_active()
    dev = pruning.run_pruning(splats, cams, targets, cfg)
    monkeypatch.setattr(pruning, "compute_delta_mse",
                        lambda *a, **k: R.compute_delta_mse(*a, **k))
    assert not pruning._device_scorer_active()
    host = pruning.run_pruning(splats, cams, targets, cfg)
    assert np.array_equal(dev[1], host[1])
    assert sum(r.removed for r in dev[2]) > 0
    for a, b in zip(dev[2], host[2]):
        assert a.to_dict() == b.to_dict()
    for f in ("positions", "sh", "opacities", "scales", "rotations"):
        assert np.array_equal(getattr(dev[0], f), getattr(host[0], f))


def test_pruning_to_counts_device_matches_host(R, monkeypatch):
    """The device-resident rate sweep (run_pruning_to_counts) equals the host
    loop over the same GPU scores, checkpoint by checkpoint."""
    from paper_2601_14821_b200 import pruning, fixture
    splats, cams = fixture.config_scene("C1")
    targets = R.render_targets(splats, cams)
    counts = [0, 500, 500, 2000, 10**6]
    dmax = 10.0 ** (-8.8 - 2.0 * 0.5)
    dev = pruning.run_pruning_to_counts(splats, cams, targets, counts, dmax)
    monkeypatch.setattr(pruning, "compute_delta_mse",
                        lambda *a, **k: R.compute_delta_mse(*a, **k))
    host = pruning.run_pruning_to_counts(splats, cams, targets, counts, dmax)
    assert len(dev) == len(host) == len(counts)
    for a_, b_ in zip(dev, host):
        assert np.array_equal(a_, b_)
    assert len(dev[-1]) == 0 and len(dev[1]) == len(splats.positions) - 500


def test_sh_recompute(C):
    splats, cams = sh_scene()
    g = golden("sh_scene")
    ci = g["camera_importance"]
    for i, lam in enumerate(g["lambdas"]):
        cfg = C.CompactionConfig(float(lam), 0.8175744761936437, 0.5 / 51.0)
        out, yc, rep = C.compact_scene(splats, cams, ci, cfg)
        ref = g[f"ycocg_{i}"]
        assert np.array_equal(yc == 0.0, ref == 0.0)
        np.testing.assert_allclose(yc, ref, rtol=0, atol=1e-9)
        np.testing.assert_allclose(out.sh, g[f"rgb_{i}"], rtol=0, atol=1e-9)
        assert rep["fallback_dc_only"] == int(g[f"fallback_{i}"])
        assert rep["failed"] == list(g[f"failed_{i}"])
        assert abs(C.ac_sparsity(yc) - float(g[f"sparsity_{i}"])) <= 1e-4


def test_sh_recompute_vs_oracle_with_device_importance(R, C, oracle):
    """compute_importance keeps (S, N) in HBM; compact_scene reads it there."""
    from paper_2601_14821_b200.fixture import make_fixture
    splats, cams = make_fixture(20000, 10, 2, width=96, height=64)
    imp, ci = R.compute_importance(splats, cams)
    cfg = C.CompactionConfig(1e-8, 0.8175744761936437, 0.5 / 51.0)
    _, yc, rep = C.compact_scene(splats, cams, ci, cfg)
    rgb_o, yc_o, st_o = oracle.compact(splats, cams, np.asarray(ci), 1e-8, 0.8175744761936437,
                                       0.5 / 51.0, threads=8)
    assert np.array_equal(yc, yc_o)
    assert rep["fallback_dc_only"] == int(np.count_nonzero(st_o == 3))


def test_known_answers(R):
    """Known-answer cases of the reference's tests/test_rasterizer.py."""
    from paper_2601_14821_b200.scene import Camera, Splats
    SH_DC = 0.28209479177387814

    def flat(position, opacity, color, scale):
        sh = np.zeros((1, 3, 16))
        sh[0, :, 0] = np.asarray(color) / SH_DC
        return Splats(np.array([position], dtype=np.float64), sh,
                      np.array([opacity], dtype=np.float64), np.full((1, 3), scale),
                      np.array([[1.0, 0, 0, 0]]))

    def stack(*ss):
        return Splats(*(np.concatenate([getattr(s, f) for s in ss]) for f in
                        ("positions", "sh", "opacities", "scales", "rotations")))

    cam = Camera(eye=np.zeros(3), rotation=np.eye(3), fx=100.0, fy=100.0, cx=8, cy=8,
                 width=16, height=16)
    p = R.project_splats(flat([0, 0, 1.0], 0.5, [1, 1, 1], 0.01), cam)
    assert p.valid[0] and np.allclose(p.mean2d[0], [8.0, 8.0], atol=1e-9)
    assert p.cov2d[0, 0] == pytest.approx(1.3, abs=1e-9)
    assert not R.project_splats(flat([0, 0, 0.009], 0.5, [1, 1, 1], 0.01), cam).valid[0]
    rec = R.render_with_records(flat([0, 0, 1.0], 0.5, [1, 1, 1], 50.0), cam)
    assert rec.image[8, 8, 0] == pytest.approx(0.5, abs=1e-6)
    (sid, alpha, t), = rec.pixel_record(8, 8)
    assert sid == 0 and t == 1.0
    front = flat([0, 0, 1.0], 0.5, [1, 1, 1], 50.0)
    back = flat([0, 0, 2.0], 0.5, [1, 1, 1], 100.0)
    img = R.render_image(stack(back, front), cam)
    assert img[8, 8, 0] == pytest.approx(0.75, abs=1e-6)
    both = stack(front, back)
    targets = R.render_targets(both, [cam])
    st = R.compute_delta_mse(both, [cam], targets)
    rec = R.render_with_records(both, cam)
    covered = np.unique(rec.pixels[rec.splat_ids == 0])
    assert st.delta_mse[0] == pytest.approx(0.0625 * len(covered) / 256, rel=1e-3)
    assert st.mse == 0.0
    neg = flat([0, 0, 1.0], 0.5, [1, 1, 1], 50.0)
    neg.sh[0, 2, 0] = -2.0 / SH_DC
    assert R.render_image(neg, cam)[8, 8, 2] == 0.0
    with pytest.raises(ValueError, match="shape"):
        R.compute_delta_mse(both, [cam], [np.zeros((4, 4, 3))])
    full = R.forward_stats(flat([0, 0, 1.0], 0.5, [1, 1, 1], 500.0), [cam])
    assert full.importance[0] == pytest.approx(0.5, abs=1e-4)


def test_delta_mse_brute_force(R):
    """ΔMSE equals re-render-without-splat (tests/test_rasterizer.py:242-257)."""
    from paper_2601_14821_b200.fixture import random_scene
    splats, cams = random_scene(11, num_splats=20, num_cameras=2)
    targets = R.render_targets(splats, cams)
    pert = perturbed(splats)
    st = R.compute_delta_mse(pert, cams, targets)
    n = len(pert)
    base = [R.render_image(pert, c) for c in cams]
    brute = np.zeros(n)
    for k in range(n):
        mask = np.ones(n, dtype=bool)
        mask[k] = False
        for s, cam in enumerate(cams):
            wo = R.render_image(pert.subset(mask), cam)
            brute[k] += np.mean((wo - targets[s]) ** 2) - np.mean((base[s] - targets[s]) ** 2)
    brute /= len(cams)
    assert np.abs(brute - st.delta_mse).max() <= 1e-9


def test_empty_and_degenerate(R, C):
    from paper_2601_14821_b200.fixture import make_fixture
    splats, cams = make_fixture(100, 2, 0, 32)
    empty = splats.subset(np.zeros(100, dtype=bool))
    img = R.render_image(empty, cams[0])
    assert img.shape == (32, 32, 3) and not img.any()
    targets = R.render_targets(splats, cams)
    st = R.compute_delta_mse(empty, cams, targets)
    assert st.delta_mse.shape == (0,)
    assert st.mse == pytest.approx(np.mean([np.mean(t ** 2) for t in targets]), rel=1e-12)
    # ragged: non-square, non-multiple-of-16 images
    sp, cs = make_fixture(3000, 3, 4, width=37, height=21)
    from oracle import oracle as O
    tg = [O.render(sp, c)[0] for c in cs]
    st = R.compute_delta_mse(perturbed(sp), cs, tg)
    imp, _, dm, mse = O.forward_stats(perturbed(sp), cs, tg)
    np.testing.assert_allclose(st.delta_mse, dm, rtol=1e-9, atol=1e-22)
    np.testing.assert_allclose(st.importance, imp, rtol=1e-12, atol=1e-20)


def test_c_abi_argument_errors(R):
    """Bad arguments come back as POTR_E_ARG (ValueError in Python), never a
    crash: NULL outputs, NULL per-view pointers, bad image sizes, unknown
    options."""
    import ctypes
    import torch
    from paper_2601_14821_b200 import _native, device as D
    splats, cams = small_scene()
    ctx = D.context()
    dev = D.current_device()
    ds = D.DeviceSplats.from_host(splats, dev)
    n, S = ds.n, len(cams)
    buf = torch.zeros((S, n), dtype=torch.float64, device=dev)
    one = torch.zeros(n, dtype=torch.float64, device=dev)
    cam_arr = _native.camera_array(cams)
    nulls = (ctypes.c_void_p * S)()
    with pytest.raises(ValueError):  # targets without row outputs
        ctx.call("potr_score_views_rows", ctypes.byref(ds.struct()), S, cam_arr,
                 (ctypes.c_void_p * S)(*[buf.data_ptr()] * S), D.ptr(buf), None, None)
    with pytest.raises(ValueError):  # no camera_importance output
        ctx.call("potr_score_views_rows", ctypes.byref(ds.struct()), S, cam_arr, None, None,
                 None, None)
    with pytest.raises(ValueError):  # NULL image pointers
        ctx.call("potr_score_views_self", ctypes.byref(ds.struct()), S, cam_arr, nulls,
                 D.ptr(one), None, D.ptr(one), D.ptr(one))
    with pytest.raises(ValueError):
        ctx.call("potr_image_compare", 0, 5, D.ptr(one), D.ptr(one), None, None)
    with pytest.raises(ValueError):
        ctx.call("potr_set_option", 99, 1)
    with pytest.raises(ValueError):
        ctx.call("potr_set_option", _native.OPT_RAW_DEPTH_KEYS, 3)
    with pytest.raises(ValueError):
        ctx.call("potr_set_option", _native.OPT_VIEW_BATCH, 0)
    # the context is still usable afterwards
    st = R.compute_delta_mse(splats, cams, R.render_targets(splats, cams))
    assert np.all(np.isfinite(st.delta_mse))


def test_host_c_abi(R, oracle):
    """potr_forward_stats_host: the reference-facing C entry with host buffers."""
    import ctypes
    from paper_2601_14821_b200 import _native, device
    splats, cams = small_scene()
    g = golden("small_scene")
    sp = perturbed(splats)
    ctx = device.context()
    n, S = len(sp), len(cams)
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in
            (sp.positions, sp.sh, sp.opacities, sp.scales, sp.rotations)]
    tg = [np.ascontiguousarray(t) for t in g["targets"]]
    tptr = (ctypes.c_void_p * S)(*[t.ctypes.data for t in tg])
    imp, ci, dm = np.empty(n), np.empty((S, n)), np.empty(n)
    mse = np.empty(1)
    ctx.call("potr_forward_stats_host", ctypes.c_int64(n),
             *[a.ctypes.data_as(ctypes.c_void_p) for a in arrs], S,
             _native.camera_array(cams), tptr, imp.ctypes.data_as(ctypes.c_void_p),
             ci.ctypes.data_as(ctypes.c_void_p), dm.ctypes.data_as(ctypes.c_void_p),
             mse.ctypes.data_as(ctypes.c_void_p))
    np.testing.assert_allclose(dm, g["pert_delta_mse"], rtol=1e-9, atol=1e-22)
    np.testing.assert_allclose(ci, g["pert_camera_importance"], rtol=1e-12, atol=1e-20)
    assert mse[0] == pytest.approx(float(g["pert_mse"]), rel=1e-12)


def _stress_scene(seed=0):
    """Edge cases in one scene: a 1500-deep stack on a few tiles (long tile
    lists, termination), huge footprints, splats behind / at the near plane,
    off-screen, opacity extremes, and a plain random population."""
    from paper_2601_14821_b200.fixture import random_scene
    from paper_2601_14821_b200.scene import Splats
    rng = np.random.default_rng(seed)
    base, cams = random_scene(seed, num_splats=400, num_cameras=3, resolution=40)
    n_stack = 1500
    eye, fwd = cams[0].eye, cams[0].rotation[2]
    stack_pos = eye + fwd[None, :] * rng.uniform(1.0, 3.0, n_stack)[:, None] \
        + 0.01 * rng.standard_normal((n_stack, 3))
    extra_pos = np.stack([eye + 0.005 * fwd, eye - 1.0 * fwd, eye + 0.0101 * fwd,
                          eye + 2.0 * fwd, eye + 50.0 * cams[0].rotation[0]])
    pos = np.concatenate([base.positions, stack_pos, extra_pos])
    n = len(pos)
    sh = np.concatenate([base.sh, 0.3 * rng.standard_normal((n - len(base.sh), 3, 16))])
    sh[len(base.sh):, :, 0] += 1.5
    op = np.concatenate([base.opacities, rng.uniform(0.05, 0.99, n_stack),
                         np.array([0.9, 0.9, 0.9, 1.0 - 1e-9, 0.5])])
    op[5] = 1e-9  # never reaches the alpha floor
    sc = np.concatenate([base.scales, rng.uniform(0.005, 0.05, (n_stack, 3)),
                         np.array([[0.01] * 3, [0.5] * 3, [0.01] * 3, [3.0, 3.0, 0.01],
                                   [0.01] * 3])])
    q = np.concatenate([base.rotations, rng.standard_normal((n - len(base.rotations), 4))])
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    q[q[:, 0] < 0] *= -1.0
    return Splats(pos, sh, op, sc, q), cams


def test_stress_edge_cases_vs_oracle(R, oracle):
    from paper_2601_14821_b200 import binning
    splats, cams = _stress_scene()
    targets = [oracle.render(splats, c)[0] for c in cams]
    gt = R.render_targets(splats, cams)
    for a, b in zip(gt, targets):
        np.testing.assert_allclose(a, b, rtol=0, atol=1e-13)
    pert = perturbed(splats)
    st = R.compute_delta_mse(pert, cams, targets)
    imp, ci, dm, mse = oracle.forward_stats(pert, cams, targets)
    np.testing.assert_allclose(st.importance, imp, rtol=1e-11, atol=1e-20)
    np.testing.assert_allclose(np.asarray(st.camera_importance), ci, rtol=1e-11, atol=1e-20)
    np.testing.assert_allclose(st.delta_mse, dm, rtol=1e-8, atol=1e-22)
    assert st.mse == pytest.approx(mse, rel=1e-12)
    for cam in cams:
        order, off, lst = binning.tile_lists(splats, cam)
        assert np.array_equal(order, oracle.depth_order(splats, cam))
        o2, l2 = oracle.tile_lists(splats, cam)
        assert np.array_equal(off, o2) and np.array_equal(lst, l2)
    assert np.diff(off).max() > 16 * 32  # tile lists longer than the kept pass-1 masks


def test_image_metrics_vs_reference(R):
    """psnr / ssim / compute_metrics on the device against the reference's
    own values (tests/golden/metrics.npz): clamping, the SSIM window and
    crop, an image too small for the crop (NaN), identical images (99 dB)."""
    from paper_2601_14821_b200 import metrics as M
    from paper_2601_14821_b200.fixture import make_fixture
    from tests.conftest import fingerprint
    g = golden("metrics")
    mse, ss = M.compare_device(g["a"], g["b"])
    assert M.psnr(g["a"], g["b"]) == float(g["psnr_ab"])
    assert M.psnr_from_mse(mse) == pytest.approx(float(g["psnr_ab"]), rel=1e-13)
    assert ss == pytest.approx(float(g["ssim_ab"]), abs=1e-13)
    assert M.ssim(g["a"], g["a"]) == pytest.approx(float(g["ssim_same"]), abs=1e-15)
    assert M.psnr_from_mse(M.compare_device(g["a"], g["a"])[0]) == float(g["psnr_same"])
    mse_t, ss_t = M.compare_device(g["tiny_a"], g["tiny_b"])
    assert np.isnan(ss_t) and np.isnan(float(g["ssim_tiny"]))
    assert M.psnr_from_mse(mse_t) == pytest.approx(float(g["psnr_tiny"]), rel=1e-13)
    splats, cams = make_fixture(3000, 3, 1, 48)
    assert fingerprint(splats, cams) == str(g["fingerprint"])
    rep = M.compute_metrics(splats, perturbed(splats), cams)
    np.testing.assert_allclose(rep.psnr_per_camera, g["model_psnr"], rtol=0, atol=1e-8)
    np.testing.assert_allclose(rep.ssim_per_camera, g["model_ssim"], rtol=0, atol=1e-12)
    assert rep.splat_count == int(g["model_count"])
    with pytest.raises(ValueError):
        M.compare_device(g["a"], g["tiny_b"])


def test_sh_sweep_matches_per_point_compaction(R, C):
    """compaction.sweep (normal equations accumulated once, solves / renders /
    errors per grid point on the device) == the reference's loop of
    compact_scene + render_image + numpy means (compaction.py:258-278)."""
    splats, cams = sh_scene()
    targets = R.render_targets(splats, cams)
    _, ci = R.compute_importance(splats, cams)
    lambdas, alphas = [10.0 ** -0.5, 1e-7], [0.8175744761936437, 0.95]
    rows = C.sweep(splats, cams, targets, ci, lambdas, alphas, 0.5 / 51.0)
    k = 0
    for alpha in alphas:
        for lam in lambdas:
            cfg = C.CompactionConfig(lam, alpha, 0.5 / 51.0)
            comp, yc, _ = C.compact_scene(splats, cams, ci, cfg)
            mse = 0.0
            for s_, cam in enumerate(cams):
                mse += float(np.mean((R.render_image(comp, cam) - targets[s_]) ** 2))
            ref = (lam, alpha, C.ac_sparsity(yc), C.mean_abs_nonzero_ac(yc), mse / len(cams))
            got = rows[k]
            assert got[:3] == ref[:3]
            assert got[3] == pytest.approx(ref[3], rel=1e-12, abs=0)
            assert got[4] == pytest.approx(ref[4], rel=1e-12, abs=0)
            k += 1
    assert k == len(rows)


def _depth_tie_scene(n_long):
    """random_scene plus splats whose depths tie in the high bits of the
    depth key: groups a few hundred ulps apart (stored in reverse depth order,
    so the stable hi sort alone would be wrong), exact duplicates, and
    n_long identical splats (a run longer than the fixup bound when > 64)."""
    from paper_2601_14821_b200.fixture import random_scene
    from paper_2601_14821_b200.scene import Splats
    base, cams = random_scene(3, num_splats=300, num_cameras=4, resolution=48)
    eye, fwd = cams[0].eye, cams[0].rotation[2]
    rows = []
    for g in range(12):
        p0 = base.positions[g]
        d0 = float(np.dot(p0 - eye, fwd))
        for k in range(6, -1, -1):  # reverse depth order in the array
            rows.append((p0 + fwd * (d0 * 2.0 ** -44 * k), g))
        rows.append((p0.copy(), g))  # exact duplicate of the group's first
    rows += [(base.positions[20].copy(), 20)] * n_long
    src = np.array([g for _, g in rows])
    pos = np.concatenate([base.positions, np.stack([p for p, _ in rows])])
    pick = lambda a: np.concatenate([a, a[src]])
    return Splats(pos, pick(base.sh), pick(base.opacities), pick(base.scales),
                  pick(base.rotations)), cams


@pytest.mark.parametrize("n_long", [3, 90])
def test_depth_key_ties_vs_oracle(R, oracle, n_long):
    """Near-equal and equal depths keep the reference's (depth, id) order
    through the split-key sort, its run fixup and its long-run fallback, in
    the per-view binning and in the batched scoring path."""
    from paper_2601_14821_b200 import binning
    splats, cams = _depth_tie_scene(n_long)
    for cam in cams:
        order, off, lst = binning.tile_lists(splats, cam)
        assert np.array_equal(order, oracle.depth_order(splats, cam))
        o2, l2 = oracle.tile_lists(splats, cam)
        assert np.array_equal(off, o2) and np.array_equal(lst, l2)
    targets = [oracle.render(splats, c)[0] for c in cams]
    st = R.compute_delta_mse(perturbed(splats), cams, targets)
    imp, ci, dm, mse = oracle.forward_stats(perturbed(splats), cams, targets)
    np.testing.assert_allclose(st.importance, imp, rtol=1e-11, atol=1e-20)
    np.testing.assert_allclose(st.delta_mse, dm, rtol=1e-8, atol=1e-22)


def test_tile_cull_bit_identical(R):
    """Culling (tile, splat) pairs by the prefilter ellipse never changes a
    bit of the renders or contribution records (no composited sample is
    dropped); the scores move only by the changed add order inside the
    per-(tile, splat) sums (chunk boundaries shift)."""
    from paper_2601_14821_b200 import _native, device
    from paper_2601_14821_b200.fixture import make_fixture
    ctx = device.context()
    scenes = [small_scene(), _stress_scene(), _depth_tie_scene(3),
              make_fixture(20000, 3, 2, width=160, height=120)]
    for splats, cams in scenes:
        out = []
        for cull in (1, 0):
            ctx.call("potr_set_option", _native.OPT_TILE_CULL, cull)
            try:
                tg = R.render_targets(splats, cams)
                st = R.compute_delta_mse(perturbed(splats), cams, tg)
                rec = R.render_with_records(splats, cams[0])
            finally:
                ctx.call("potr_set_option", _native.OPT_TILE_CULL, 1)
            out.append((tg, st, rec))
        (t1, s1, r1), (t0, s0, r0) = out
        for a, b in zip(t1, t0):
            assert np.array_equal(a, b)
        np.testing.assert_allclose(s1.importance, s0.importance, rtol=1e-12, atol=1e-30)
        np.testing.assert_allclose(s1.delta_mse, s0.delta_mse, rtol=1e-9, atol=1e-24)
        np.testing.assert_allclose(np.asarray(s1.camera_importance),
                                   np.asarray(s0.camera_importance), rtol=1e-12, atol=1e-30)
        assert s1.mse == s0.mse
        for f in ("splat_ids", "pixels", "alphas", "trans_at", "partials", "colors"):
            assert np.array_equal(getattr(r1, f), getattr(r0, f))


@pytest.mark.slow
def test_large_scene_views_vs_oracle(R, oracle):
    """300k splats at 800x800 (the C2 shape), two views, against the oracle."""
    from paper_2601_14821_b200.fixture import make_fixture
    splats, cams = make_fixture(300_000, 100, 0, 800)
    cams = cams[:2]
    targets = R.render_targets(splats, cams)
    pert = perturbed(splats)
    st = R.compute_delta_mse(pert, cams, targets)
    imp, ci, dm, mse = oracle.forward_stats(pert, cams, [np.asarray(t) for t in targets],
                                            threads=2)
    np.testing.assert_allclose(st.importance, imp, rtol=1e-10, atol=1e-22)
    assert score_close(st.delta_mse, dm, rel=1e-6, floor=1e-24)
    assert st.mse == pytest.approx(mse, rel=1e-11)


def _codec_cases():
    """Inputs of oracle/gen_golden.py's codec fixture, regenerated here."""
    from paper_2601_14821_b200.fixture import make_fixture
    from paper_2601_14821_b200.scene import Splats
    rng = np.random.default_rng(11)
    cases = []
    s, c = make_fixture(3000, 6, 5, 32)
    cases.append((s, c, 24, None, False))
    s2, c2 = make_fixture(800, 4, 6, 32)
    pos = s2.positions.copy()
    pos[100:140] = pos[99]
    pos[200:203] = pos[500]
    s2 = Splats(pos, s2.sh, s2.opacities, s2.scales, s2.rotations)
    cases.append((s2, c2, 24, None, True))
    cases.append((s2, c2, 5, None, False))
    cases.append((s, c, 24, (np.array([0.01, -0.02, 0.03]), 1.3), True))
    cases.append((s.subset(np.arange(1)), c, 24, None, False))
    s3, c3 = make_fixture(500, 3, 7, 32)
    rot = s3.rotations.copy()
    rot[::3] *= -1.0
    s3 = Splats(s3.positions, s3.sh * 3.0, s3.opacities,
                s3.scales * rng.uniform(0.5, 2.0, (500, 1)), rot)
    cases.append((s3, c3, 24, None, False))
    return cases


def test_codec_bytes_match_reference(C):
    """The device codec back end reproduces the reference's bytes exactly:
    octree stream and DFS order (multi-splat leaves at the depth limit, a
    shallow depth limit, a pinned root cube, a single splat), the 55
    attribute streams (negative rotation real parts, values past the
    quantiser's usual range) and the whole zstd container."""
    from paper_2601_14821_b200 import codec
    from tests.conftest import fingerprint
    g = golden("codec")
    params = codec.QuantParams(51.0, 101.0, 201.0, 2001.0)
    q, beta, gamma = 0.5, 7e-05, 1.5811388300841894e-05
    for i, (s, c, md, rc, with_yc) in enumerate(_codec_cases()):
        assert fingerprint(s, c) == str(g[f"fingerprint_{i}"])
        eyes = [cam.eye for cam in c]
        yc = C.coeffs_rgb_to_ycocg(s.sh) * 0.5 if with_yc else None
        octree, order, center, half = codec.octree_stream(s.positions, eyes, beta, gamma,
                                                          max_depth=md, root_cube_=rc)
        assert octree == g[f"octree_{i}"].tobytes(), f"case {i}: octree stream"
        assert np.array_equal(order, g[f"order_{i}"])
        assert np.array_equal(center, g[f"center_{i}"]) and half == float(g[f"half_{i}"])
        streams = codec.encode_attribute_streams(s.subset(order), params,
                                                 sh_ycocg=None if yc is None else yc[order])
        assert [len(x) for x in streams] == list(g[f"stream_lengths_{i}"]), f"case {i}"
        assert b"".join(streams) == g[f"streams_{i}"].tobytes(), f"case {i}: streams"
        data, order2 = codec.encode_container(s, params, q, beta, gamma, zstd_level=3,
                                              max_depth=md, root_cube=rc, sh_ycocg=yc,
                                              camera_eyes=eyes)
        assert np.array_equal(order2, order)
        assert data == g[f"container_{i}"].tobytes(), f"case {i}: container"


def test_full_size_properties(R, oracle):
    """At the C3 shape (3M splats, 1237x822 views): depth order and tile lists
    equal the oracle's; per-camera importance telescopes to the rendered
    coverage (sum_k I_k(s) = mean over pixels of 1 - T_final); self-target
    scores are non-negative with zero MSE; and the spatial record layout
    changes no bit."""
    from paper_2601_14821_b200 import _native, binning, device
    splats, cams = c3_scene()
    views = [cams[0], cams[101]]
    order, off, lst = binning.tile_lists(splats, views[0])
    assert np.array_equal(order, oracle.depth_order(splats, views[0]))
    o_off, o_lst = oracle.tile_lists(splats, views[0])
    assert np.array_equal(off, o_off) and np.array_equal(lst, o_lst)

    ctx = device.context()
    dev = device.current_device()
    ds = device.DeviceSplats.from_host(splats, dev)
    imp, ci, _, _ = R.forward_stats_device(ds, views, None)
    for s, cam in enumerate(views):
        _, trans = R._render_device(ds, cam, ctx, dev, with_trans=True)
        coverage = float((1.0 - trans).mean())
        assert abs(float(ci[s].sum()) - coverage) <= 1e-10 * coverage

    imgs, imp2, ci2, dm, mse = R.render_and_score_device(ds, views)
    assert float(mse.item()) == 0.0
    assert bool((dm >= 0).all())
    assert np.array_equal(imp.cpu().numpy(), imp2.cpu().numpy())

    try:
        ctx.call("potr_set_option", _native.OPT_SPATIAL_RECORDS, 0)
        imp3, ci3, _, _ = R.forward_stats_device(ds, views, None)
    finally:
        ctx.call("potr_set_option", _native.OPT_SPATIAL_RECORDS, 1)
    assert np.array_equal(imp.cpu().numpy(), imp3.cpu().numpy())
    assert np.array_equal(ci.cpu().numpy(), ci3.cpu().numpy())


def test_full_size_sh_recompute_vs_oracle(R, C, oracle):
    """SH recompute at the C4 shape (3M splats, 200 views at 1237x822): the
    device's coefficients for a random sample of 1500 splats equal the
    oracle's bit for bit (the normal equations run on the fp64 tensor cores,
    whose MMA rounds as the oracle's fma chain) from the same camera-importance
    columns, at three lambdas down to the bench's 1e-12."""
    from paper_2601_14821_b200.scene import Splats
    splats, cams = c3_scene()
    imp, ci = R.compute_importance(splats, cams)
    rng = np.random.default_rng(11)
    idx = np.sort(rng.choice(len(splats.positions), 1500, replace=False))
    sub = Splats(*(np.ascontiguousarray(np.asarray(getattr(splats, f))[idx]) for f in
                   ("positions", "sh", "opacities", "scales", "rotations")))
    ci_sub = np.ascontiguousarray(np.asarray(ci)[:, idx])
    for lam in (1e-7, 1e-9, 1e-12):
        cfg = C.CompactionConfig(lam, 0.8175744761936437, 0.5 / 51.0)
        _, yc, rep = C.compact_scene(splats, cams, ci, cfg)
        _, yc_o, st_o = oracle.compact(sub, cams, ci_sub, lam, 0.8175744761936437, 0.5 / 51.0,
                                       threads=8)
        assert np.array_equal(yc[idx] == 0.0, yc_o == 0.0)
        assert np.array_equal(yc[idx], yc_o)


def test_full_size_delta_mse_vs_oracle(R, oracle):
    """The removal-effect scores of one full C3 view (3M splats, 1237x822,
    opacities x 0.97 against the unperturbed render) equal the oracle's for
    every splat: importance to 1e-12, dMSE to 1e-9 relative."""
    splats, cams = c3_scene()
    view = [cams[57]]
    targets = R.render_targets(splats, view)
    pert = splats.copy()
    pert.opacities = pert.opacities * 0.97
    st = R.compute_delta_mse(pert, view, targets)
    imp, ci, dm, mse = oracle.forward_stats(pert, view, [np.asarray(t) for t in targets])
    np.testing.assert_allclose(st.importance, imp, rtol=1e-12, atol=1e-20)
    np.testing.assert_allclose(st.delta_mse, dm, rtol=1e-9, atol=1e-22)
    assert abs(st.mse - mse) <= 1e-12 * abs(mse)
