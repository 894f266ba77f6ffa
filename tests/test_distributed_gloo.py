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


def _oracle_rows(splats, cams, targets):
    """Per-view rows, as potr_score_views_rows produces them."""
    from oracle import oracle as O
    n = len(splats.positions)
    imp, dm, mse = [], [], []
    for c, t in zip(cams, targets):
        i1, _, d1, m1 = O.forward_stats(splats, [c], [t])
        imp.append(i1), dm.append(d1), mse.append(m1)
    L = len(cams)
    f = lambda rows: torch.from_numpy(np.array(rows, dtype=np.float64).reshape(L, n))  # noqa
    return f(imp), f(dm), torch.tensor(mse, dtype=torch.float64).reshape(L)


def _worker_ordered(rank, world, port, out_path):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2601_14821_b200 import distributed
    from paper_2601_14821_b200.fixture import make_fixture
    from oracle import oracle as O
    splats, cams = make_fixture(600, 7, 3, 32)
    targets = [O.render(splats, c)[0] for c in cams]
    pert = splats.copy()
    pert.opacities = pert.opacities * 0.97
    st = distributed.forward_stats_sharded(pert, cams, targets, ordered=True,
                                           rows_fn=_oracle_rows)
    np.savez(out_path + f".{rank}.npz", importance=st.importance, delta_mse=st.delta_mse,
             mse=st.mse)
    dist.destroy_process_group()


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
    st = distributed.forward_stats_sharded(pert, cams, targets, score_fn=_oracle_scorer,
                                           ordered=False)
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
        # camera_importance is a ShardedRows: numpy access gathers the full (S, N)
        np.testing.assert_array_equal(r["rows"], ci)


@pytest.mark.parametrize("world", [2, 3])
def test_ordered_chain_bit_identical_to_camera_order(tmp_path, world):
    """The ordered reduction (send/recv chain + broadcast) gives every rank
    exactly the single-device camera-order sums, for any world size."""
    from oracle import oracle as O
    from paper_2601_14821_b200.fixture import make_fixture
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "res")
    mp.start_processes(_worker_ordered, args=(world, port, out), nprocs=world, join=True,
                       start_method="spawn")
    splats, cams = make_fixture(600, 7, 3, 32)
    targets = [O.render(splats, c)[0] for c in cams]
    pert = splats.copy()
    pert.opacities = pert.opacities * 0.97
    imp_r, dm_r, mse_r = _oracle_rows(pert, cams, targets)
    n = len(pert.positions)
    acc = torch.zeros(2 * n + 1, dtype=torch.float64)
    for v in range(len(cams)):
        acc[:n] += imp_r[v]
        acc[n:2 * n] += dm_r[v]
        acc[2 * n:] += mse_r[v:v + 1]
    ref = torch.div(acc, torch.tensor(float(len(cams)), dtype=torch.float64)).numpy()
    for r in range(world):
        got = np.load(out + f".{r}.npz")
        assert np.array_equal(got["importance"], ref[:n])
        assert np.array_equal(got["delta_mse"], ref[n:2 * n])
        assert float(got["mse"]) == float(ref[2 * n])


def _oracle_solve(splats, cams, ci, cfg):
    from oracle import oracle as O
    return O.compact(splats, cams, np.asarray(ci), cfg.lambda_y, cfg.parallel_threshold,
                     cfg.zero_threshold)


def _sh_scene():
    from paper_2601_14821_b200.fixture import make_fixture
    from oracle import oracle as O
    splats, cams = make_fixture(701, 7, 4, 32)
    _, ci, _, _ = O.forward_stats(splats, cams)
    return splats, cams, ci


def _worker_sh(rank, world, port, out_path):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2601_14821_b200 import distributed
    from paper_2601_14821_b200.compaction import CompactionConfig
    splats, cams, ci = _sh_scene()
    S, n = ci.shape
    lo, hi = distributed.shard_range(S, rank, world)
    rows = distributed.ShardedRows(torch.from_numpy(ci[lo:hi].copy()), (lo, hi), S)
    # the full matrix comes back from the row blocks (collective numpy access)
    assert rows.shape == (S, n)
    assert np.array_equal(np.asarray(rows), ci)
    cfg = CompactionConfig(1e-8, 0.8175744761936437, 0.5 / 51.0)
    res, yc, rep = distributed.compact_scene_sharded(splats, cams, rows, cfg,
                                                     solve_fn=_oracle_solve)
    np.savez(out_path + f".{rank}.npz", rgb=res.sh, yc=yc, failed=np.array(rep["failed"]),
             fallback=rep["fallback_dc_only"])
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sh_splat_shards_bit_identical(tmp_path, world):
    """compact_scene_sharded: the all-to-all turns the ranks' view rows into
    splat shards with every view in camera order, so each splat is solved on
    exactly the single-device inputs and the all-gather reassembles
    coefficients identical bit for bit to one compact_scene."""
    from oracle import oracle as O
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "res")
    mp.start_processes(_worker_sh, args=(world, port, out), nprocs=world, join=True,
                       start_method="spawn")
    splats, cams, ci = _sh_scene()
    rgb, yc, status = O.compact(splats, cams, ci, 1e-8, 0.8175744761936437, 0.5 / 51.0)
    for r in range(world):
        got = np.load(out + f".{r}.npz")
        assert np.array_equal(got["rgb"], rgb)
        assert np.array_equal(got["yc"], yc)
        assert list(got["failed"]) == [int(k) for k in np.nonzero(status == 2)[0]]
        assert int(got["fallback"]) == int(np.count_nonzero(status == 3))


def _worker_subgroup(rank, world, port, out_path):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2601_14821_b200 import distributed
    group = dist.new_group([1, 2])  # group ranks 0, 1 are global ranks 1, 2
    if rank in (1, 2):
        g = rank - 1
        n = 5
        rows = torch.arange(3 * n, dtype=torch.float64).reshape(3, n) * (g + 1) + 0.1
        acc = distributed.ordered_reduce(rows, None, None, n, group)
        np.save(out_path + f".{rank}.npy", acc.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_ordered_reduce_on_a_subgroup(tmp_path):
    """Group-local ranks are mapped to global ranks for send/recv/broadcast."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "res")
    mp.start_processes(_worker_subgroup, args=(3, port, out), nprocs=3, join=True,
                       start_method="spawn")
    n = 5
    acc = torch.zeros(n, dtype=torch.float64)
    for g in range(2):
        rows = torch.arange(3 * n, dtype=torch.float64).reshape(3, n) * (g + 1) + 0.1
        for v in range(3):
            acc += rows[v]
    for r in (1, 2):
        assert np.array_equal(np.load(out + f".{r}.npy"), acc.numpy())
