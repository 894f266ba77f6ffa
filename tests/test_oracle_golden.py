"""Pin the CPU oracle (oracle/potr_oracle.c) against golden vectors produced
by the reference itself (oracle/gen_golden.py).  No GPU needed."""

import numpy as np
import pytest

from tests.conftest import (fingerprint, golden, oracle_scene, perturbed, sh_scene, small_scene)


def test_fixture_fingerprints():
    g = golden("small_scene")
    assert fingerprint(*small_scene()) == str(g["fingerprint"])
    from paper_2601_14821_b200.fixture import make_fixture
    assert fingerprint(*make_fixture(10000, 8, 0, 128)) == str(golden("c1")["fingerprint"])
    assert fingerprint(*make_fixture(600, 6, 5, 48)) == str(golden("sh_scene")["fingerprint_base"])
    o = golden("oracle_scenes")
    for seed in range(20):
        assert fingerprint(*oracle_scene(seed)) == str(o[f"s{seed}_fingerprint"])


def test_projection_bit_exact(oracle):
    splats, cams = small_scene()
    g = golden("small_scene")
    p = oracle.project(splats, cams[0])
    # the projection restates OpenBLAS's FMA order for (mu - eye) @ W^T, so
    # every field is bit-identical to the reference
    assert np.array_equal(p["valid"], g["proj_valid"])
    assert np.array_equal(p["mean2d"], g["proj_mean2d"])
    assert np.array_equal(p["cov2d"], g["proj_cov2d"])
    assert np.array_equal(p["view_depth"], g["proj_depth"])
    assert np.array_equal(p["radius"], g["proj_radius"])
    ids = g["colors0_ids"]
    np.testing.assert_allclose(p["colors"][ids], g["colors0"], rtol=0, atol=1e-15)


def test_depth_order_and_tile_lists_bit_exact(oracle):
    splats, cams = small_scene()
    g = golden("small_scene")
    for c in (0, 1):
        assert np.array_equal(oracle.depth_order(splats, cams[c]), g[f"order{c}"])
        off, lst = oracle.tile_lists(splats, cams[c])
        assert np.array_equal(off, g[f"tile_offsets{c}"])
        assert np.array_equal(lst, g[f"tile_splats{c}"])


def test_render_matches_reference_targets(oracle):
    splats, cams = small_scene()
    g = golden("small_scene")
    for s, cam in enumerate(cams):
        img, _ = oracle.render(splats, cam)
        np.testing.assert_allclose(img, g["targets"][s], rtol=0, atol=1e-14)


def test_forward_stats_matches_reference(oracle):
    splats, cams = small_scene()
    g = golden("small_scene")
    targets = list(g["targets"])
    imp, ci, dm, mse = oracle.forward_stats(perturbed(splats), cams, targets, threads=4)
    np.testing.assert_allclose(imp, g["pert_importance"], rtol=1e-12, atol=1e-20)
    np.testing.assert_allclose(ci, g["pert_camera_importance"], rtol=1e-12, atol=1e-20)
    np.testing.assert_allclose(dm, g["pert_delta_mse"], rtol=1e-9, atol=1e-22)
    assert mse == pytest.approx(float(g["pert_mse"]), rel=1e-12)
    imp0, _, dm0, mse0 = oracle.forward_stats(splats, cams, targets, threads=1)
    np.testing.assert_allclose(dm0, g["it1_delta_mse"], rtol=1e-9, atol=1e-22)
    assert mse0 < 1e-28 and float(g["it1_mse"]) < 1e-28
    imp1, ci1, _, _ = oracle.forward_stats(splats, cams, None)
    np.testing.assert_allclose(ci1, g["camera_importance"], rtol=1e-12, atol=1e-20)


def test_forward_stats_thread_invariant(oracle):
    splats, cams = small_scene()
    g = golden("small_scene")
    targets = list(g["targets"])
    a = oracle.forward_stats(perturbed(splats), cams, targets, threads=1)
    b = oracle.forward_stats(perturbed(splats), cams, targets, threads=6)
    for x, y in zip(a[:3], b[:3]):
        assert np.array_equal(x, y)


def test_oracle_scenes(oracle):
    o = golden("oracle_scenes")
    for seed in range(20):
        splats, cams = oracle_scene(seed)
        img0, _ = oracle.render(splats, cams[0])
        np.testing.assert_allclose(img0, o[f"s{seed}_image0"], rtol=0, atol=1e-14)
        targets = [oracle.render(splats, c)[0] for c in cams]
        imp, _, dm, mse = oracle.forward_stats(perturbed(splats), cams, targets)
        np.testing.assert_allclose(imp, o[f"s{seed}_importance"], rtol=1e-12, atol=1e-20)
        np.testing.assert_allclose(dm, o[f"s{seed}_delta_mse"], rtol=1e-9, atol=1e-22)
        assert mse == pytest.approx(float(o[f"s{seed}_mse"]), rel=1e-10)


def test_records(oracle):
    from paper_2601_14821_b200.fixture import random_scene
    g = golden("records")
    splats, cams = random_scene(4, num_splats=20)
    img, tr, rec = oracle.render(splats, cams[0], records=True)
    assert np.array_equal(rec["splat_ids"], g["splat_ids"])
    assert np.array_equal(rec["pixels"], g["pixels"])
    np.testing.assert_allclose(rec["alphas"], g["alphas"], rtol=1e-14, atol=0)
    np.testing.assert_allclose(rec["trans_at"], g["trans_at"], rtol=1e-13, atol=0)
    np.testing.assert_allclose(rec["partials"], g["partials"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(tr, g["transmittance"], rtol=1e-13, atol=0)


def test_c1(oracle):
    from paper_2601_14821_b200.fixture import make_fixture
    g = golden("c1")
    splats, cams = make_fixture(10000, 8, 0, 128)
    targets = [oracle.render(splats, c)[0] for c in cams]
    imp, _, dm, mse = oracle.forward_stats(perturbed(splats), cams, targets, threads=8)
    np.testing.assert_allclose(imp, g["pert_importance"], rtol=1e-11, atol=1e-20)
    np.testing.assert_allclose(dm, g["pert_delta_mse"], rtol=1e-8, atol=1e-20)
    assert mse == pytest.approx(float(g["pert_mse"]), rel=1e-10)


def test_sh_compaction_matches_reference(oracle):
    splats, cams = sh_scene()
    g = golden("sh_scene")
    ci = g["camera_importance"]
    for i, lam in enumerate(g["lambdas"]):
        rgb, yc, status = oracle.compact(splats, cams, ci, float(lam), 0.8175744761936437,
                                         0.5 / 51.0, threads=4)
        ref = g[f"ycocg_{i}"]
        assert np.array_equal(yc == 0.0, ref == 0.0), f"zero pattern differs at lambda {lam}"
        np.testing.assert_allclose(yc, ref, rtol=0, atol=1e-9)
        np.testing.assert_allclose(rgb, g[f"rgb_{i}"], rtol=0, atol=1e-9)
        assert np.count_nonzero(status == 3) == int(g[f"fallback_{i}"])
        assert np.array_equal(np.nonzero(status == 2)[0], g[f"failed_{i}"])
        sp = float(np.mean(yc[:, :, 1:] == 0.0))
        assert abs(sp - float(g[f"sparsity_{i}"])) <= 1e-12
