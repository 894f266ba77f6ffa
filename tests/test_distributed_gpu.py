"""The view-sharded path through the CUDA kernels: 2 and 3 ranks on the one
B200 of the lease.

NCCL refuses two ranks on one device, so the ranks talk over gloo and the
collectives stage their CUDA tensors through host memory
(distributed._staged); every kernel is the product's own and no kernel waits
on another rank's (the exchange steps are host-driven).  Each rank runs the
public API exactly as the reference pipeline calls it (pipeline.py:42-59,
pruning.py:132) with view sharding enabled and must reproduce the
single-process results bit for bit: importance, delta MSE, MSE, the 48-step
prune mask, and the splat-sharded SH recompute (coefficients, zero patterns,
statuses).
"""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from tests.conftest import ROOT

pytestmark = pytest.mark.gpu

WORKER = r'''
import os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.environ["POTR_ROOT"])
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
out = os.environ["POTR_OUT"]
torch.cuda.set_device(0)
dist.init_process_group("gloo", rank=rank, world_size=world)
from paper_2601_14821_b200 import compaction, distributed, pruning, rasterizer
from paper_2601_14821_b200.fixture import make_fixture

splats, cams = make_fixture(2500, 7, 11, 56)
targets = rasterizer.render_targets(splats, cams)
pert = splats.copy()
pert.opacities = pert.opacities * 0.97
cfg = compaction.CompactionConfig(1e-8, 0.8175744761936437, 0.5 / 51.0)
pcfg = pruning.PruneConfig(delta_mse_max=10.0 ** (-8.8 - 2.0 * 0.5), iterations=12)

def run():
    st = rasterizer.compute_delta_mse(pert, cams, targets)
    _, ci = rasterizer.compute_importance(pert, cams)
    comp, yc, rep = compaction.compact_scene(pert, cams, ci, cfg)
    _, kept, reps = pruning.run_pruning(splats, cams, targets, pcfg)
    return dict(importance=st.importance, delta_mse=st.delta_mse, mse=np.array(st.mse),
                camera_importance=np.asarray(ci), rgb=comp.sh, ycocg=yc,
                failed=np.array(rep["failed"], dtype=np.int64),
                fallback=np.array(rep["fallback_dc_only"]), kept=kept,
                removed=np.array([r.removed for r in reps]))

distributed.enable_view_sharding(True)
assert distributed.sharding_active()
res = run()
# the unordered all-reduce form as well (a few ulps allowed)
st_u = distributed.forward_stats_sharded(pert, cams, targets, ordered=False)
res["importance_unordered"] = st_u.importance
res["delta_mse_unordered"] = st_u.delta_mse
if rank == 0:
    distributed.enable_view_sharding(False)
    single = run()
    for k, v in single.items():
        res["single_" + k] = v
np.savez(out + f".{rank}.npz", **res)
dist.barrier()
dist.destroy_process_group()
'''


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_view_sharded_ranks_on_one_b200_bit_identical(cuda, tmp_path, world):
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    out = str(tmp_path / "res")
    port = _port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK=str(r),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), POTR_ROOT=ROOT,
                   POTR_OUT=out)
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env))
    codes = [p.wait(timeout=600) for p in procs]
    assert codes == [0] * world
    ranks = [np.load(out + f".{r}.npz") for r in range(world)]
    single = {k[7:]: ranks[0][k] for k in ranks[0].files if k.startswith("single_")}
    assert single
    for got in ranks:
        for k, v in single.items():
            assert np.array_equal(got[k], v), f"{k} differs from the single-process result"
        np.testing.assert_allclose(got["importance_unordered"], single["importance"],
                                   rtol=1e-13, atol=0)
        np.testing.assert_allclose(got["delta_mse_unordered"], single["delta_mse"],
                                   rtol=1e-12, atol=1e-30)
    assert single["kept"].size < 2500  # the prune loop removed splats
