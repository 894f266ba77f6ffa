"""View-sharded multi-GPU execution.

One process per GPU (torchrun), splats replicated, cameras split into
contiguous blocks [S*r/W, S*(r+1)/W).  Each rank scores its own views with
the B200 kernels; the path has exactly two exchange steps, and both keep the
single-GPU results bit for bit:

* prune scores (rasterizer.py:338-352) -- ordered chain (default): each rank
  keeps its per-view rows (potr_score_views_rows) and the running
  [importance | dMSE | mse] sums (2N+1 fp64, 48 MB at C3) travel rank 0 -> 1
  -> ... -> W-1, each rank adding its rows in camera order, then one
  broadcast.  Every element sees exactly the single-GPU sequence of IEEE
  additions, so importance, dMSE, MSE and the prune mask are bit-identical
  for any GPU count.  `ordered=False` uses one NCCL all-reduce of the per-rank
  sums instead (a few ulps from the camera-order result).
* SH recompute (compaction.py:195-243, split by splat span at :219-226) --
  the per-camera importance rows are transposed into splat shards by one
  all-to-all (rank q receives columns [N*q/W, N*(q+1)/W) of every view, in
  camera order), each rank accumulates and solves only its own splats, and
  one all-gather returns every splat's coefficients to every rank.  The
  normal equations of a splat are summed over the same views in the same
  order as on one GPU, so coefficients, zero patterns and statuses are
  bit-identical; nothing of size (185, N) is ever reduced.

NCCL carries CUDA tensors directly.  Under gloo (CPU tests, or several ranks
sharing one GPU where NCCL refuses to run) the tensors are staged through host
memory; the arithmetic is unchanged.  `group` may be any process group: peer
ranks are mapped to global ranks for the point-to-point calls.
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


def shard_range(num_items, rank, world):
    """Contiguous, balanced block of item indices (views or splats) owned by `rank`."""
    return (num_items * rank) // world, (num_items * (rank + 1)) // world


# ---------------------------------------------------------------------------
# collective plumbing


def _global(group, r):
    """Global rank of group rank r (send/recv/broadcast take global ranks)."""
    return r if group is None else dist.get_global_rank(group, r)


def _staged(group):
    """True when CUDA tensors must cross through host memory (gloo)."""
    return dist.get_backend(group) == "gloo"


def _send(t, dst, group):
    dist.send(t.cpu() if (t.is_cuda and _staged(group)) else t, dst=_global(group, dst),
              group=group)


def _recv(t, src, group):
    if t.is_cuda and _staged(group):
        h = torch.empty(t.shape, dtype=t.dtype)
        dist.recv(h, src=_global(group, src), group=group)
        t.copy_(h)
    else:
        dist.recv(t, src=_global(group, src), group=group)


def _broadcast(t, src, group):
    if t.is_cuda and _staged(group):
        h = t.cpu()
        dist.broadcast(h, src=_global(group, src), group=group)
        t.copy_(h)
    else:
        dist.broadcast(t, src=_global(group, src), group=group)


def all_reduce(t, op=None, group=None):
    """dist.all_reduce that also works for CUDA tensors under gloo (staged)."""
    op = dist.ReduceOp.SUM if op is None else op
    if t.is_cuda and _staged(group):
        h = t.cpu()
        dist.all_reduce(h, op=op, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op, group=group)
    return t


def _all_to_all(out, inp, out_splits, in_splits, group):
    if inp.is_cuda and _staged(group):
        h = torch.empty(out.shape, dtype=out.dtype)
        dist.all_to_all_single(h, inp.cpu(), out_splits, in_splits, group=group)
        out.copy_(h)
    else:
        dist.all_to_all_single(out, inp, out_splits, in_splits, group=group)


def _all_gather(out, inp, group):
    """out (W * len(inp),) <- every rank's inp, in rank order."""
    if inp.is_cuda and _staged(group):
        h = torch.empty(out.shape, dtype=out.dtype)
        dist.all_gather_into_tensor(h, inp.cpu().contiguous(), group=group)
        out.copy_(h)
    else:
        dist.all_gather_into_tensor(out, inp.contiguous(), group=group)


# ---------------------------------------------------------------------------
# prune scores


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
        _recv(acc, rank - 1, group)
    imp = acc[:n]
    for v in range(imp_rows.shape[0]):  # one IEEE add per element, in camera order
        imp += imp_rows[v]
        if with_dm:
            acc[n:2 * n] += dmse_rows[v]
            acc[2 * n:] += mse_rows[v:v + 1]
    if rank < world - 1:
        _send(acc, rank + 1, group)
    _broadcast(acc, world - 1, group)
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
    if buf.is_cuda and _staged(group):
        h = buf.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
        buf = h
    else:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    host = torch.div(buf.cpu(), torch.tensor(float(num_views), dtype=torch.float64)).numpy()
    if dmse_sum is None:
        return host[:n], None, None
    return host[:n], host[n:2 * n], float(host[2 * n])


class ShardedRows:
    """camera_importance of a view-sharded forward_stats: this rank holds the
    rows of its own view block (`rows`, on the device).  Its shape is the
    full (S, N).  compact_scene consumes it without gathering (the splat-shard
    all-to-all); any numpy use all-gathers the full matrix, which is a
    collective: every rank must touch it the same way (as the reference
    pipeline's symmetric code does)."""

    def __init__(self, rows, view_range, num_views, group=None):
        self.rows = rows
        self.view_range = tuple(view_range)
        self.num_views = int(num_views)
        self.group = group
        self._host = None

    @property
    def shape(self):
        return (self.num_views, int(self.rows.shape[1]))

    @property
    def dtype(self):
        return np.dtype(np.float64)

    @property
    def ndim(self):
        return 2

    def __len__(self):
        return self.num_views

    def local_rows(self):
        return self.rows

    def numpy(self):
        if self._host is None:
            self._host = gather_rows(self.rows, self.num_views, self.group).numpy()
        return self._host

    def __array__(self, dtype=None, copy=None):
        a = self.numpy()
        if dtype is not None and a.dtype != dtype:
            return a.astype(dtype)
        return a.copy() if copy else a

    def __getitem__(self, item):
        return self.numpy()[item]

    def __array_ufunc__(self, ufunc, method, *inputs, **kwargs):
        conv = tuple(np.asarray(x) if isinstance(x, ShardedRows) else x for x in inputs)
        return getattr(ufunc, method)(*conv, **kwargs)

    def __repr__(self):
        return (f"ShardedRows(shape={self.shape}, local views {self.view_range}, "
                f"device={self.rows.device})")


def gather_rows(rows, num_views, group=None):
    """The full (S, N) matrix from every rank's contiguous row block (host)."""
    world = dist.get_world_size(group)
    n = int(rows.shape[1])
    Lmax = max(shard_range(num_views, r, world)[1] - shard_range(num_views, r, world)[0]
               for r in range(world))
    pad = torch.zeros((max(Lmax, 1), n), dtype=torch.float64, device=rows.device)
    pad[:rows.shape[0]] = rows
    out = torch.empty((world * max(Lmax, 1) * n,), dtype=torch.float64, device=rows.device)
    _all_gather(out, pad.reshape(-1), group)
    out = out.reshape(world, max(Lmax, 1), n).cpu()
    parts = []
    for r in range(world):
        lo, hi = shard_range(num_views, r, world)
        parts.append(out[r, :hi - lo])
    return torch.cat(parts) if parts else torch.zeros((0, n), dtype=torch.float64)


def forward_stats_sharded(splats, cameras, targets=None, group=None, score_fn=None,
                          ordered=True, rows_fn=None):
    """forward_stats over this rank's view block + the cross-rank reduction
    (ordered chain by default, else one all-reduce).

    camera_importance of the result is a ShardedRows: this rank's rows
    (cameras[lo:hi], `.view_range`), shaped as the full (S, N) matrix."""
    from .rasterizer import ForwardStats
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
    return ForwardStats(importance, ShardedRows(rows, (lo, hi), S, group), delta_mse, mse_v)


# ---------------------------------------------------------------------------
# SH recompute, splat-sharded


def transpose_to_splat_shard(rows, num_views, n, group=None):
    """All-to-all: this rank's (L, N) camera_importance rows of views [lo, hi)
    -> the (S, N_r) columns of its splat shard [N*r/W, N*(r+1)/W), every view
    in camera order."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    L = int(rows.shape[0])
    cs = [shard_range(n, q, world) for q in range(world)]
    vs = [shard_range(num_views, p, world) for p in range(world)]
    my_n = cs[rank][1] - cs[rank][0]
    send = torch.cat([rows[:, c0:c1].reshape(-1) for c0, c1 in cs]) if L * n > 0 else \
        torch.zeros(0, dtype=torch.float64, device=rows.device)
    in_splits = [L * (c1 - c0) for c0, c1 in cs]
    out_splits = [(v1 - v0) * my_n for v0, v1 in vs]
    recv = torch.empty(sum(out_splits), dtype=torch.float64, device=rows.device)
    _all_to_all(recv, send, out_splits, in_splits, group)
    return recv.reshape(num_views, my_n)  # blocks arrive in rank = camera order


def compact_scene_sharded(splats, cameras, camera_importance, config, group=None,
                          solve_fn=None):
    """compact_scene (compaction.py:195-243) with the splats split into
    per-rank spans (as the reference's own thread split, :219-226).

    camera_importance: a ShardedRows (this rank's view rows), or the full
    (S, N) matrix (host or device), of which this rank uses its view block.
    solve_fn(splats_shard, cameras, ci_shard (S, n_r), config) -> (rgb, ycocg,
    status) on the shard; default the B200 kernel (compaction.compact_device).
    Returns what compact_scene returns, on every rank."""
    from . import device as D
    from .compaction import STATUS_FAILED, STATUS_DC_FALLBACK
    from .scene import Splats
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    S = len(cameras)
    n = len(splats.positions)
    lo, hi = shard_range(S, rank, world)
    on_gpu = solve_fn is None
    dev = D.current_device() if on_gpu else torch.device("cpu")
    if isinstance(camera_importance, ShardedRows):
        if camera_importance.view_range != (lo, hi) or camera_importance.num_views != S:
            raise ValueError("camera_importance rows do not match this rank's view block")
        rows = camera_importance.local_rows()
    elif isinstance(camera_importance, D.LazyHostArray):
        rows = camera_importance.device_tensor[lo:hi]
    elif isinstance(camera_importance, torch.Tensor):
        rows = camera_importance.reshape(S, n)[lo:hi]
    else:
        rows = torch.from_numpy(np.ascontiguousarray(
            np.asarray(camera_importance, dtype=np.float64).reshape(S, n)[lo:hi]))
    rows = rows.to(device=dev, dtype=torch.float64).contiguous()
    ci = transpose_to_splat_shard(rows, S, n, group)
    c0, c1 = shard_range(n, rank, world)
    idx = np.arange(c0, c1)
    shard = Splats(*(np.asarray(getattr(splats, f))[idx] for f in
                     ("positions", "sh", "opacities", "scales", "rotations")))
    if on_gpu:
        from .compaction import compact_device
        rgb, yc, status = compact_device(shard, cameras, ci, config)
    else:
        rgb, yc, status = solve_fn(shard, cameras, ci, config)
        rgb, yc, status = (torch.as_tensor(np.asarray(x)) for x in (rgb, yc, status))
    # all-gather the shards (padded to the largest span) in rank = splat order
    nmax = max(shard_range(n, r, world)[1] - shard_range(n, r, world)[0] for r in range(world))
    nmax = max(nmax, 1)
    pack = torch.zeros((nmax, 97), dtype=torch.float64, device=dev)
    m = c1 - c0
    if m:
        pack[:m, :48] = rgb.reshape(m, 48).to(dev, torch.float64)
        pack[:m, 48:96] = yc.reshape(m, 48).to(dev, torch.float64)
        pack[:m, 96] = status.reshape(m).to(dev, torch.float64)
    out = torch.empty((world * nmax * 97,), dtype=torch.float64, device=dev)
    _all_gather(out, pack.reshape(-1), group)
    out = D.to_host(out) if out.is_cuda else out.numpy()
    out = out.reshape(world, nmax, 97)
    parts = [out[r, :shard_range(n, r, world)[1] - shard_range(n, r, world)[0]]
             for r in range(world)]
    full = np.concatenate(parts) if parts else np.zeros((0, 97))
    rgb_h = np.ascontiguousarray(full[:, :48]).reshape(n, 3, 16)
    yc_h = np.ascontiguousarray(full[:, 48:96]).reshape(n, 3, 16)
    status_h = full[:, 96].astype(np.int8)
    res = Splats(np.array(splats.positions, dtype=np.float64, copy=True), rgb_h,
                 np.array(splats.opacities, dtype=np.float64, copy=True),
                 np.array(splats.scales, dtype=np.float64, copy=True),
                 np.array(splats.rotations, dtype=np.float64, copy=True))
    report = {"failed": [int(k) for k in np.nonzero(status_h == STATUS_FAILED)[0]],
              "fallback_dc_only": int(np.count_nonzero(status_h == STATUS_DC_FALLBACK))}
    return res, yc_h, report
