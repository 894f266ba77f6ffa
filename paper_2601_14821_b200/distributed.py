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
devices.  NCCL's association differs from the single-GPU camera-order sum by
at most a few ulps (the prune mask is insensitive to that, SURVEY.md TL;DR 5).
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


def forward_stats_sharded(splats, cameras, targets=None, group=None, score_fn=None):
    """forward_stats over this rank's view block + one all-reduce.

    camera_importance of the result holds only this rank's rows
    (cameras[lo:hi]); `.view_range` says which."""
    from .rasterizer import ForwardStats
    from .device import LazyHostArray
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    S = len(cameras)
    lo, hi = shard_range(S, rank, world)
    local_t = targets[lo:hi] if targets is not None else None
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
