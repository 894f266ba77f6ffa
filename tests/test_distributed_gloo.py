"""View sharding + the all-reduce step on world_size 2 over gloo (CPU).

The per-shard scorer is injected: here it is the CPU oracle (test
infrastructure), on the GPU box it is the CUDA path; what is under test is the
host logic -- contiguous view blocks, one fp64 all-reduce of
[importance | dMSE | mse] sums, normalisation by the global camera count.
"""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests.conftest import ROOT


def _oracle_scorer(splats, cams, targets):
    from oracle import oracle as O
    n = len(splats.positions)
    if len(cams) == 0:
        z = torch.zeros(n, dtype=torch.float64)
        return z, torch.zeros((0, n), dtype=torch.float64), torch.zeros(n, dtype=torch.float64), \
            torch.zeros(1, dtype=torch.float64)
    imp, ci, dm, mse = O.forward_stats(splats, cams, targets)
    S = len(cams)
    # un-normalised sums, as potr_score_views produces them
    return (torch.from_numpy(imp * S), torch.from_numpy(ci), torch.from_numpy(dm * S),
            torch.tensor([mse * S], dtype=torch.float64))


def _worker(rank, world, port, out_path):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2601_14821_b200 import distributed
    from paper_2601_14821_b200.fixture import make_fixture
    from oracle import oracle as O
    splats, cams = make_fixture(800, 5, 2, 40)
    targets = [O.render(splats, c)[0] for c in cams]
    pert = splats.copy()
    pert.opacities = pert.opacities * 0.97
    st = distributed.forward_stats_sharded(pert, cams, targets, score_fn=_oracle_scorer)
    lo, hi = distributed.shard_range(len(cams), rank, world)
    assert st.camera_importance.view_range == (lo, hi)
    np.savez(out_path + f".{rank}.npz", importance=st.importance, delta_mse=st.delta_mse,
             mse=st.mse, rows=np.asarray(st.camera_importance))
    dist.destroy_process_group()


def test_shard_range_covers_views():
    from paper_2601_14821_b200.distributed import shard_range
    for S in (1, 5, 8, 200, 201):
        for W in (1, 2, 4, 8):
            blocks = [shard_range(S, r, W) for r in range(W)]
            assert blocks[0][0] == 0 and blocks[-1][1] == S
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(W - 1))


def test_two_rank_gloo_matches_single_process(tmp_path):
    from oracle import oracle as O
    from paper_2601_14821_b200.fixture import make_fixture
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "res")
    mp.start_processes(_worker, args=(2, port, out), nprocs=2, join=True, start_method="spawn")
    splats, cams = make_fixture(800, 5, 2, 40)
    targets = [O.render(splats, c)[0] for c in cams]
    pert = splats.copy()
    pert.opacities = pert.opacities * 0.97
    imp, ci, dm, mse = O.forward_stats(pert, cams, targets)
    r0 = np.load(out + ".0.npz")
    r1 = np.load(out + ".1.npz")
    for r in (r0, r1):
        np.testing.assert_allclose(r["importance"], imp, rtol=1e-13, atol=1e-22)
        np.testing.assert_allclose(r["delta_mse"], dm, rtol=1e-12, atol=1e-24)
        assert float(r["mse"]) == pytest.approx(mse, rel=1e-13)
    np.testing.assert_array_equal(np.concatenate([r0["rows"], r1["rows"]]), ci)
