"""The whole encoder through the B200 path, step for step as
potr.pipeline.encode_pipeline (pipeline.py:31-101) runs it: targets, the
pruning iterations, importance, SH compaction (after pruning, or interleaved
at iteration 20), container -- against the
reference's own encode_pipeline output on the same scene
(tests/golden/pipeline.npz, oracle/gen_golden.py gen_pipeline).  The
container must come out byte for byte, the DFS order of the kept splats
index for index; decode_container (pipeline.py:104-107) closes the loop."""

import numpy as np
from scipy.special import expit
import pytest

from tests.conftest import fingerprint, golden

pytestmark = pytest.mark.gpu

Q = 0.5


@pytest.mark.parametrize("compact_at", [None, 20])
def test_encode_pipeline_matches_reference(cuda, compact_at):
    from paper_2601_14821_b200 import codec, compaction as C, pruning as PR
    from paper_2601_14821_b200 import rasterizer as R
    from paper_2601_14821_b200.fixture import make_fixture
    g = golden("pipeline")
    splats, cams = make_fixture(num_splats=2500, num_cameras=6, seed=13, resolution=48)
    assert fingerprint(splats, cams) == str(g["fingerprint"])
    # config_from_q(0.5, zstd_level=3, delta_mse_max=1e-7, lambda_y=1e-9) (config.py:59-74)
    sf_sh = 1.0 + 100.0 * Q
    prune_cfg = PR.PruneConfig(delta_mse_max=1e-7, a=10.0, iterations=48)
    comp_cfg = C.CompactionConfig(lambda_y=1e-9,
                                  parallel_threshold=float(expit(3.0 * Q)),
                                  zero_threshold=0.5 / sf_sh)
    params = codec.QuantParams(sf_sh, 1.0 + 200.0 * Q, 1.0 + 400.0 * Q, 1.0 + 4000.0 * Q)

    tag = "" if compact_at is None else "_interleaved"
    targets = R.render_targets(splats, cams)
    reports = []
    sink = reports.append
    if compact_at is None:  # pipeline.py:49-60
        pruned, kept, _ = PR.run_pruning(splats, cams, targets, prune_cfg, report_sink=sink)
        _, cam_imp = R.compute_importance(pruned, cams)
        compacted, ycocg, rep = C.compact_scene(pruned, cams, cam_imp, comp_cfg)
    else:  # pipeline.py:61-79
        pruned, kept, _ = PR.run_pruning(splats, cams, targets, prune_cfg, report_sink=sink,
                                         last_iteration=compact_at)
        _, cam_imp = R.compute_importance(pruned, cams)
        mid, ycocg, rep = C.compact_scene(pruned, cams, cam_imp, comp_cfg)
        compacted, kept_rel, _ = PR.run_pruning(mid, cams, targets, prune_cfg, report_sink=sink,
                                                first_iteration=compact_at + 1)
        kept = kept[kept_rel]
        ycocg = ycocg[kept_rel]
    assert [r["removed"] if isinstance(r, dict) else r.removed for r in reports] == \
        g["removed" + tag].tolist()
    assert len(rep["failed"]) == int(g["compaction_failures" + tag])
    assert rep["fallback_dc_only"] == int(g["fallback_dc" + tag])
    assert C.ac_sparsity(ycocg) == float(g["ac_sparsity" + tag])
    container, order = codec.encode_container(
        compacted, params, Q, 1.4e-4 * Q, 5.0 * 10.0 ** (-3.0 - 5.0 * Q), zstd_level=3,
        sh_ycocg=ycocg, camera_eyes=[c.eye for c in cams])
    assert len(compacted.positions) == int(g["splats_out" + tag])
    assert np.array_equal(kept[order], g["dfs_order" + tag])
    assert container == g["container" + tag].tobytes()

    dec, header = codec.decode_container(container)
    assert header.splat_count == int(g["splats_out" + tag])
    assert np.array_equal(dec.positions, g["decoded_positions" + tag])
    assert np.array_equal(dec.sh, g["decoded_sh" + tag])
