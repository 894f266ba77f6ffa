"""View-sharded multi-GPU execution.

One process per GPU (torchrun), splats replicated, cameras split into
contiguous blocks [S*r/W, S*(r+1)/W).  Each rank scores its views with the
B200 kernels into un-normalised per-splat sums, then ONE NCCL all-reduce
combines [importance sum (N) | dMSE sum (N) | MSE sum (1)] in fp64 over
NVLink, and every rank normalises by the global camera count exactly as
rasterizer.py:348-352 does.  The SH recompute shards the same way: each rank
accumulates the normal equations of its views (potr_sh_accumulate), one
all-reduce sums them, and the solves run on the reduced system.

The reduction step is the path's only real exchange; nothing else crosses
devices.  Two forms (SURVEY.md 8e "determinism across G"):

* ordered (default): each rank keeps its per-view rows (potr_score_views_rows)
  and the running [importance | dMSE | mse] sums travel rank 0 -> 1 -> ... ->
  W-1 (send/recv, 2N+1 fp64), each rank adding its rows in camera order, then
  one broadcast.  Every element sees exactly the single-GPU sequence of
  additions, so results are bit-identical for any GPU count.  Cost: W-1
  sequential hops of 48 MB at C3 over NVLink plus the row adds (~1 ms).
* unordered: one NCCL all-reduce of the per-rank sums; NCCL's association
  differs from the camera-order sum by a few ulps (the prune mask is
  insensitive to that, SURVEY.md TL;DR 5).
"""

import ctypes

import numpy as np
import torch
import torch.distributed as dist

_enabled = False


def enable_view_sharding(flag=True):
    """Route forward_stats / compact_scene through the sharded path whenever
    torch.distributed is initialised with more than one rank."""
    global _enabled
    _enabled = bool(flag)


def sharding_active():
    return _enabled and dist.is_available() and dist.is_initialized() and \
        dist.get_world_size() > 1


def shard_range(num_views, rank, world):
    """Contiguous, balanced block of view indices owned by `rank`."""
    return (num_views * rank) // world, (num_views * (rank + 1)) // world


def _gpu_score(splats, cameras, targets):
    from . import device as D
    from .rasterizer import _score_device
    ctx = D.context()
    dev = D.current_device()
    ds = D.DeviceSplats.from_host(splats, dev)
    n = ds.n
    tg = D.targets_cache.get(targets, cameras, dev) if targets is not None else None
    imp, cam_imp, dm, mse = _score_device(ds, cameras, tg, ctx, dev)
    return imp[:n], cam_imp[:len(cameras), :n], (dm[:n] if dm is not None else None), mse


def _gpu_score_rows(splats, cameras, targets):
    """Per-view rows of this rank's views: (camera_importance (L, N), dMSE
    rows (L, N) or None, MSE per view (L,) or None), on the device."""
    from . import _native
    from . import device as D
    ctx = D.context()
    dev = D.current_device()
    ds = D.DeviceSplats.from_host(splats, dev)
    n, L = ds.n, len(cameras)
    ci = D.empty((max(L, 1), max(n, 1)), dev)
    dm = mse = tptr = None
    if targets is not None:
        dm = D.empty((max(L, 1), max(n, 1)), dev)
        mse = D.empty(max(L, 1), dev)
        tg = D.targets_cache.get(targets, cameras, dev)
        tptr = (ctypes.c_void_p * max(L, 1))(*[t.data_ptr() for t in tg])
    if L > 0:
        ctx.call("potr_score_views_rows", ctypes.byref(ds.struct()), L,
                 _native.camera_array(cameras), tptr, D.ptr(ci), D.ptr(dm), D.ptr(mse))
    return (ci[:L, :n], dm[:L, :n] if dm is not None else None,
            mse[:L] if mse is not None else None)


def ordered_reduce(imp_rows, dmse_rows, mse_rows, n, group=None):
    """Camera-order accumulation of the per-view rows across the ranks'
    contiguous view blocks: a chain 0 -> 1 -> ... -> W-1 carrying
    [importance | dMSE | mse] sums, then a broadcast from the last rank.
    Returns the (2N+1,) (or (N,) without dMSE) sums on every rank."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    with_dm = dmse_rows is not None
    acc = torch.zeros(2 * n + 1 if with_dm else n, dtype=torch.float64,
                      device=imp_rows.device)
    if rank > 0:
        dist.recv(acc, src=rank - 1, group=group)
    imp = acc[:n]
    for v in range(imp_rows.shape[0]):  # one IEEE add per element, in camera order
        imp += imp_rows[v]
        if with_dm:
            acc[n:2 * n] += dmse_rows[v]
            acc[2 * n:] += mse_rows[v:v + 1]
    if rank < world - 1:
        dist.send(acc, dst=rank + 1, group=group)
    dist.broadcast(acc, src=world - 1, group=group)
    return acc


def finalize_sums(acc, n, num_views, with_dm=True):
    """acc / num_views with IEEE division (rasterizer.py:348-352), in place.
    On the device through potr_finalize_stats: torch's tensor / scalar on
    CUDA multiplies by the reciprocal, which is not the single-GPU result."""
    if acc.is_cuda:
        from . import device as D
        dm = D.ptr(acc[n:2 * n]) if with_dm else None
        ms = D.ptr(acc[2 * n:]) if with_dm else None
        D.context().call("potr_finalize_stats", ctypes.c_int64(n), int(num_views),
                         D.ptr(acc[:n]), dm, ms)
        return acc
    return torch.div(acc, torch.tensor(float(num_views), dtype=torch.float64), out=acc)


def reduce_stats(imp_sum, dmse_sum, mse_sum, num_views, group=None):
    """All-reduce the per-rank sums in one fp64 message and normalise them
    (rasterizer.py:348-352).  Returns host (importance, delta_mse, mse)."""
    n = imp_sum.numel()
    parts = [imp_sum.reshape(-1)]
    if dmse_sum is not None:
        parts += [dmse_sum.reshape(-1), mse_sum.reshape(-1)]
    buf = torch.cat(parts).to(torch.float64)
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    host = (buf / float(num_views)).cpu().numpy()
    if dmse_sum is None:
        return host[:n], None, None
    return host[:n], host[n:2 * n], float(host[2 * n])


def forward_stats_sharded(splats, cameras, targets=None, group=None, score_fn=None,
                          ordered=True, rows_fn=None):
    """forward_stats over this rank's view block + the cross-rank reduction
    (ordered chain by default, else one all-reduce).

    camera_importance of the result holds only this rank's rows
    (cameras[lo:hi]); `.view_range` says which."""
    from .rasterizer import ForwardStats
    from .device import LazyHostArray
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    S = len(cameras)
    lo, hi = shard_range(S, rank, world)
    local_t = targets[lo:hi] if targets is not None else None
    if ordered:
        n = len(splats.positions)
        cam_imp, dm_rows, mse_rows = (rows_fn or _gpu_score_rows)(splats, cameras[lo:hi],
                                                                   local_t)
        acc = ordered_reduce(cam_imp, dm_rows, mse_rows, n, group)
        host = finalize_sums(acc, n, S, dm_rows is not None).cpu().numpy()
        importance = host[:n]
        delta_mse = host[n:2 * n] if dm_rows is not None else None
        mse_v = float(host[2 * n]) if dm_rows is not None else None
    else:
        score = score_fn or _gpu_score
        imp, cam_imp, dm, mse = score(splats, cameras[lo:hi], local_t)
        importance, delta_mse, mse_v = reduce_stats(imp, dm, mse, S, group)
    rows = cam_imp if isinstance(cam_imp, torch.Tensor) else torch.as_tensor(cam_imp)
    lazy = LazyHostArray(rows)
    lazy.view_range = (lo, hi)
    return ForwardStats(importance, lazy, delta_mse, mse_v)


def compact_scene_sharded(splats, cameras, local_camera_importance, config, group=None):
    """compact_scene when each rank holds the camera_importance rows of its
    own view block: accumulate local normal equations, all-reduce them, solve."""
    from . import _native
    from . import device as D
    from .compaction import _splats_ps, STATUS_FAILED, STATUS_DC_FALLBACK
    from .scene import Splats
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    S = len(cameras)
    lo, hi = shard_range(S, rank, world)
    ctx = D.context()
    dev = D.current_device()
    ds = _splats_ps(splats, dev)
    n = ds.n
    neq = torch.zeros((_native.NEQ_STRIDE, max(n, 1)), dtype=torch.float64, device=dev)
    if hi > lo and n > 0:
        ci = D.as_device_matrix(local_camera_importance, (hi - lo, n), dev)
        ctx.call("potr_sh_accumulate", ctypes.byref(ds.struct()), hi - lo,
                 _native.camera_array(cameras[lo:hi]), D.ptr(ci), D.ptr(neq))
    dist.all_reduce(neq, op=dist.ReduceOp.SUM, group=group)
    rgb = D.empty((max(n, 1), 3, 16), dev)
    yc = D.empty((max(n, 1), 3, 16), dev)
    status = D.empty(max(n, 1), dev, torch.int8)
    ctx.call("potr_sh_solve", ctypes.byref(ds.struct()), D.ptr(neq),
             ctypes.c_double(config.lambda_y), ctypes.c_double(config.parallel_threshold),
             ctypes.c_double(config.zero_threshold), D.ptr(rgb), D.ptr(yc), D.ptr(status))
    rgb = rgb[:n].cpu().numpy()
    yc = yc[:n].cpu().numpy()
    status = status[:n].cpu().numpy()
    out = Splats(np.array(splats.positions, dtype=np.float64), rgb,
                 np.array(splats.opacities, dtype=np.float64),
                 np.array(splats.scales, dtype=np.float64),
                 np.array(splats.rotations, dtype=np.float64))
    report = {"failed": [int(k) for k in np.nonzero(status == STATUS_FAILED)[0]],
              "fallback_dc_only": int(np.count_nonzero(status == STATUS_DC_FALLBACK))}
    return out, yc, report
