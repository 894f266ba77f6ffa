"""A small workload through every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per run):

    compute-sanitizer --tool memcheck python tools/sanitize_run.py

C1-sized prune-score pass (score + importance + self-target modes), renders,
records, binning, the SH recompute (all size classes + the DC fallback), the
device controller's removal order, image metrics, the codec, and a scoring
call through the overlapped upload (lookahead sets, deferred colours)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2601_14821_b200 import (binning, codec, compaction, metrics, pruning,  # noqa: E402
                                   rasterizer as R)
from paper_2601_14821_b200.fixture import make_fixture  # noqa: E402

splats, cams = make_fixture(3000, 3, 1, width=96, height=64)
targets = R.render_targets(splats, cams)
pert = splats.copy()
pert.opacities = pert.opacities * 0.97
st = R.compute_delta_mse(pert, cams, targets)
imp, ci = R.compute_importance(pert, cams)
_, st2 = R.render_targets_and_delta_mse(splats, cams)
rec = R.render_with_records(splats, cams[0])
order, off, lst = binning.tile_lists(splats, cams[0])
cfg = compaction.CompactionConfig(1e-8, 0.8175744761936437, 0.5 / 51.0)
out, yc, rep = compaction.compact_scene(pert, cams, ci, cfg)
cps = pruning.run_pruning_to_counts(splats, cams, targets, [100, 400], 10.0 ** -9.8)
_, kept, _ = pruning.run_pruning(splats, cams, targets,
                                 pruning.PruneConfig(delta_mse_max=10.0 ** -9.8, iterations=3))
m = metrics.compute_metrics(splats, pert, cams)
params = codec.QuantParams(51.0, 101.0, 201.0, 2001.0)
data, corder = codec.encode_container(splats, params, 0.5, 7e-05, 1.58e-05, zstd_level=3,
                                      camera_eyes=[c.eye for c in cams])
# the overlapped upload: SH rows over the async threshold, several view
# batches binned ahead with deferred colours
big, bcams = make_fixture(40_000, 20, 2, width=80, height=60)
btg = R.render_targets(big, bcams)
bst = R.compute_delta_mse(big, bcams, btg)
print("ok", float(st.mse), len(rec.splat_ids), len(lst), len(rep["failed"]), len(kept),
      m.mean_psnr, len(data), float(bst.mse))
