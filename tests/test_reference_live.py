"""Oracle and fixtures against the live reference (development container
only; skipped where /root/reference is absent, e.g. on the GPU box)."""

import numpy as np
import pytest


def test_fixture_generators_bit_identical(reference):
    from potr import fixture as RF
    from paper_2601_14821_b200 import fixture as F
    a, ca = RF.make_fixture(3000, 5, 7, 40)
    b, cb = F.make_fixture(3000, 5, 7, 40)
    for f in ("positions", "sh", "opacities", "scales", "rotations"):
        assert np.array_equal(getattr(a, f), getattr(b, f))
    for x, y in zip(ca, cb):
        assert np.array_equal(x.eye, y.eye) and np.array_equal(x.rotation, y.rotation)
        assert (x.fx, x.fy, x.cx, x.cy, x.width, x.height) == (y.fx, y.fy, y.cx, y.cy, y.width,
                                                               y.height)
    for seed in (0, 5):
        ra, rca = RF.random_scene(seed)
        rb, rcb = F.random_scene(seed)
        assert np.array_equal(ra.sh, rb.sh) and np.array_equal(rca[0].eye, rcb[0].eye)


@pytest.mark.parametrize("seed", [21, 22, 23])
def test_oracle_vs_live_reference(reference, oracle, seed):
    from potr import rasterizer as R
    from potr.fixture import random_scene
    splats, cams = random_scene(seed, num_splats=60, num_cameras=3)
    targets = R.render_targets(splats, cams)
    pert = splats.copy()
    pert.opacities = pert.opacities * 0.9
    st = R.compute_delta_mse(pert, cams, targets)
    imp, ci, dm, mse = oracle.forward_stats(pert, cams, targets)
    np.testing.assert_allclose(imp, st.importance, rtol=1e-12, atol=1e-20)
    np.testing.assert_allclose(dm, st.delta_mse, rtol=1e-9, atol=1e-22)
    for cam in cams:
        p = R.project_splats(pert, cam)
        ids = np.nonzero(p.valid)[0]
        order = ids[np.argsort(p.view_depth[ids], kind="stable")]
        assert np.array_equal(order, oracle.depth_order(pert, cam))


def test_install_patches_every_import_site(reference):
    import potr.pruning
    import potr.pipeline
    import potr.compaction
    import potr.rasterizer
    from paper_2601_14821_b200 import install as I
    import potr.bitstream
    from paper_2601_14821_b200 import rasterizer, compaction, codec
    before = potr.pruning.compute_delta_mse
    undo = I.install()
    try:
        assert potr.pruning.compute_delta_mse is rasterizer.compute_delta_mse
        assert potr.pipeline.compact_scene is compaction.compact_scene
        assert potr.pipeline.compute_importance is rasterizer.compute_importance
        assert potr.compaction.render_image is rasterizer.render_image
        assert potr.rasterizer.forward_stats is rasterizer.forward_stats
        assert potr.pipeline.encode_container is codec.encode_container
        assert potr.bitstream.encode_container is codec.encode_container
        # decode: one wrapper (reference exception classes) bound at both sites
        assert potr.bitstream.decode_container is potr.pipeline.decode_container
        assert potr.bitstream.decode_container.__doc__ == codec.decode_container.__doc__
    finally:
        undo()
    assert potr.pruning.compute_delta_mse is before
    assert potr.bitstream.decode_container.__module__ == "potr.bitstream"
