"""Drop-in for potr.rasterizer on B200 (reference: potr/rasterizer.py).

Same functions, signatures, dataclasses and exceptions as the reference; the
work runs in libpotr_b200.so (kernels (a)-(d), see csrc/raster.cu) on the
current CUDA device.  `threads` is accepted and ignored (results never depend
on it, as in the reference).  Everything is float64, and results are
bit-reproducible run to run.

When torch.distributed is initialised with more than one rank and view
sharding is enabled (paper_2601_14821_b200.distributed.enable_view_sharding),
forward_stats scores only this rank's cameras and all-reduces the per-splat
sums over NCCL.
"""

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from . import device as D

# rasterizer.py:22-26
ALPHA_FLOOR = 1.0 / 255.0
ALPHA_CAP = 0.999
T_TERMINATE = 1e-4
NEAR_CLIP = 0.01
COV_DILATION = 0.3


@dataclass
class Projection:
    """Screen-space footprints of every splat for one camera (:29-37)."""

    mean2d: np.ndarray
    cov2d: np.ndarray
    view_depth: np.ndarray
    radius: np.ndarray
    valid: np.ndarray


@dataclass
class RenderRecord:
    """One camera's image plus its contribution log (:206-243)."""

    image: np.ndarray
    transmittance: np.ndarray
    splat_ids: np.ndarray
    pixels: np.ndarray
    alphas: np.ndarray
    trans_at: np.ndarray
    partials: np.ndarray
    colors: np.ndarray
    width: int
    height: int

    def pixel_record(self, x, y):
        """Ordered (splat_id, alpha, T) contributions of one pixel."""
        mask = self.pixels == y * self.width + x
        return list(zip(self.splat_ids[mask], self.alphas[mask], self.trans_at[mask]))

    def camera_importance(self, num_splats):
        """Fraction of this image coming from each splat (:226-230)."""
        w = self.trans_at * self.alphas
        acc = np.bincount(self.splat_ids, weights=w, minlength=num_splats)
        return acc / (self.width * self.height)

    def prune_deltas(self):
        """Per-contribution colour change of removing its splat (:232-243)."""
        pk = self.image.reshape(-1, 3)[self.pixels]
        a = self.alphas[:, None]
        csplat = self.colors[self.splat_ids]
        return a / (1.0 - a) * (pk - self.partials - self.trans_at[:, None] * csplat)


@dataclass
class ForwardStats:
    """Aggregated products of one instrumented pass (:294-301).

    camera_importance is a LazyHostArray: it stays in HBM (where
    compact_scene reads it) until numpy touches it."""

    importance: np.ndarray
    camera_importance: object
    delta_mse: np.ndarray | None
    mse: float | None


def quat_to_rotmat(q):
    """(N, 4) wxyz unit quaternions to (N, 3, 3) rotation matrices (:40-53).
    Host helper kept for API completeness; the kernels inline it."""
    q = np.asarray(q, dtype=np.float64)
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    R = np.empty((q.shape[0], 3, 3), dtype=np.float64)
    R[:, 0, 0] = 1 - 2 * (y * y + z * z)
    R[:, 0, 1] = 2 * (x * y - w * z)
    R[:, 0, 2] = 2 * (x * z + w * y)
    R[:, 1, 0] = 2 * (x * y + w * z)
    R[:, 1, 1] = 1 - 2 * (x * x + z * z)
    R[:, 1, 2] = 2 * (y * z - w * x)
    R[:, 2, 0] = 2 * (x * z - w * y)
    R[:, 2, 1] = 2 * (y * z + w * x)
    R[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def _project_device(splats, camera):
    ctx = D.context()
    dev = D.current_device()
    ds = D.DeviceSplats.from_host(splats, dev)
    n = ds.n
    mean2d = D.empty((max(n, 1), 2), dev)
    cov2d = D.empty((max(n, 1), 3), dev)
    depth = D.empty(max(n, 1), dev)
    radius = D.empty(max(n, 1), dev)
    valid = D.empty(max(n, 1), dev, torch.uint8)
    colors = D.empty((max(n, 1), 3), dev)
    cam = _native.camera_struct(camera)
    ctx.call("potr_project", ctypes.byref(ds.struct()), ctypes.byref(cam), D.ptr(mean2d),
             D.ptr(cov2d), D.ptr(depth), D.ptr(radius), D.ptr(valid), D.ptr(colors))
    return (mean2d[:n], cov2d[:n], depth[:n], radius[:n], valid[:n], colors[:n])


def project_splats(splats, camera) -> Projection:
    """EWA projection of all splats into one camera (:56-97)."""
    mean2d, cov2d, depth, radius, valid, _ = _project_device(splats, camera)
    return Projection(mean2d.cpu().numpy(), cov2d.cpu().numpy(), depth.cpu().numpy(),
                      radius.cpu().numpy(), valid.cpu().numpy().astype(bool))


def splat_colors(splats, camera):
    """Per-splat colours for one camera, clamped at zero (:100-110)."""
    return _project_device(splats, camera)[5].cpu().numpy()


def render_with_records(splats, camera) -> RenderRecord:
    """Render one camera and log every composited sample (:246-267).
    The log lives on the host, so this is for small scenes (tests, probes)."""
    ctx = D.context()
    dev = D.current_device()
    ds = D.DeviceSplats.from_host(splats, dev)
    n = ds.n
    h, w = int(camera.height), int(camera.width)
    image = D.empty((h, w, 3), dev)
    trans = D.empty((h, w), dev)
    colors = D.empty((max(n, 1), 3), dev)
    cam = _native.camera_struct(camera)
    m = ctypes.c_int64(0)
    args = (ctypes.byref(ds.struct()), ctypes.byref(cam), D.ptr(image), D.ptr(trans),
            D.ptr(colors))
    ctx.call("potr_render_records", *args, ctypes.c_int64(0), ctypes.byref(m), None, None, None,
             None, None)
    cnt = m.value
    ids = D.empty(max(cnt, 1), dev, torch.int64)
    pix = D.empty(max(cnt, 1), dev, torch.int64)
    al = D.empty(max(cnt, 1), dev)
    ta = D.empty(max(cnt, 1), dev)
    pa = D.empty((max(cnt, 1), 3), dev)
    ctx.call("potr_render_records", *args, ctypes.c_int64(max(cnt, 1)), ctypes.byref(m),
             D.ptr(ids), D.ptr(pix), D.ptr(al), D.ptr(ta), D.ptr(pa))
    return RenderRecord(image.cpu().numpy(), trans.cpu().numpy(), ids[:cnt].cpu().numpy(),
                        pix[:cnt].cpu().numpy(), al[:cnt].cpu().numpy(), ta[:cnt].cpu().numpy(),
                        pa[:cnt].cpu().numpy(), colors[:n].cpu().numpy(), w, h)


def _render_device(ds, camera, ctx, dev, with_trans=False):
    h, w = int(camera.height), int(camera.width)
    image = D.empty((h, w, 3), dev)
    trans = D.empty((h, w), dev) if with_trans else None
    cam = _native.camera_struct(camera)
    ctx.call("potr_render", ctypes.byref(ds.struct()), ctypes.byref(cam), D.ptr(image),
             D.ptr(trans))
    return image, trans


def render_image(splats, camera) -> np.ndarray:
    """Composited (H, W, 3) image, unclamped, black background (:270-271)."""
    ctx = D.context()
    dev = D.current_device()
    image, _ = _render_device(D.DeviceSplats.from_host(splats, dev), camera, ctx, dev)
    return D.to_host(image)


def prune_difference(record: RenderRecord, x, y, splat_id):
    """Literal partial-colour form of the removal difference at one pixel
    (:274-291); a host utility over a RenderRecord."""
    mask = record.pixels == y * record.width + x
    sids = record.splat_ids[mask]
    hit = np.nonzero(sids == splat_id)[0]
    if len(hit) == 0:
        return np.zeros(3)
    i = int(hit[0])
    terms = (record.trans_at[mask, None] * record.alphas[mask, None] * record.colors[sids])
    partials = np.vstack([np.zeros(3), np.cumsum(terms, axis=0)])
    p_k = partials[-1]
    a = record.alphas[mask][i]
    return partials[i] - partials[i + 1] / (1.0 - a) + a * p_k / (1.0 - a)


def _score_device(ds, cameras, dev_targets, ctx, dev, want_cam_imp=True):
    """potr_score_views over `cameras` into fresh device sums."""
    n, S = ds.n, len(cameras)
    imp = torch.zeros(max(n, 1), dtype=torch.float64, device=dev)
    cam_imp = D.empty((max(S, 1), max(n, 1)), dev) if want_cam_imp else None
    dm = mse = None
    tptr = None
    if dev_targets is not None:
        dm = torch.zeros(max(n, 1), dtype=torch.float64, device=dev)
        mse = torch.zeros(1, dtype=torch.float64, device=dev)
        tptr = (ctypes.c_void_p * max(S, 1))(*[t.data_ptr() for t in dev_targets])
    cams = _native.camera_array(cameras)
    ctx.call("potr_score_views", ctypes.byref(ds.struct()), S, cams, tptr, D.ptr(imp),
             D.ptr(cam_imp), D.ptr(dm), D.ptr(mse))
    return imp, cam_imp, dm, mse


def forward_stats_device(ds, cameras, dev_targets, want_cam_imp=True):
    """forward_stats on device-resident splats and targets.  Returns device
    tensors (importance (N,), camera_importance (S, N) or None, delta_mse (N,)
    or None, mse (1,) or None), normalised by the camera count."""
    ctx = D.context()
    dev = ds.device
    n, S = ds.n, len(cameras)
    imp, cam_imp, dm, mse = _score_device(ds, cameras, dev_targets, ctx, dev, want_cam_imp)
    ctx.call("potr_finalize_stats", ctypes.c_int64(n), S, D.ptr(imp), D.ptr(dm), D.ptr(mse))
    return (imp[:n], cam_imp[:S, :n] if cam_imp is not None else None,
            dm[:n] if dm is not None else None, mse)


def forward_stats(splats, cameras, targets=None, threads=1) -> ForwardStats:
    """Render every camera once; importance and, with targets, the exact
    removal effect of each splat on the MSE (:311-352)."""
    from . import distributed
    if distributed.sharding_active():
        return distributed.forward_stats_sharded(splats, cameras, targets)
    dev = D.current_device()
    # the SH rows upload while the first view batches are binned
    ds = D.DeviceSplats.from_host(splats, dev, async_sh=len(cameras) > 0)
    n, S = ds.n, len(cameras)
    if S == 0:
        if targets is not None:
            raise ZeroDivisionError("float division by zero")
        return ForwardStats(np.full(n, np.nan), np.zeros((0, n)), None, None)
    try:
        dev_targets = D.targets_cache.get(targets, cameras, dev) if targets is not None else None
        imp, cam_imp, dm, mse = forward_stats_device(ds, cameras, dev_targets)
    finally:
        ds.wait_upload()
    cam_imp = D.LazyHostArray(cam_imp)
    if targets is None:
        return ForwardStats(D.to_host(imp), cam_imp, None, None)
    host = D.to_host(torch.cat([imp, dm, mse]))
    return ForwardStats(host[:n], cam_imp, host[n:2 * n], float(host[2 * n]))


def render_and_score_device(ds, cameras, want_cam_imp=True):
    """render_targets + forward_stats against those very targets, in one pass
    (potr_score_views_self): the first scoring of an encode, whose targets are
    the renders of the unmodified model.  Returns device tensors (images,
    importance, camera_importance or None, delta_mse, mse), normalised."""
    ctx = D.context()
    dev = ds.device
    n, S = ds.n, len(cameras)
    imgs = [D.empty((int(c.height), int(c.width), 3), dev) for c in cameras]
    imp = torch.zeros(max(n, 1), dtype=torch.float64, device=dev)
    dm = torch.zeros(max(n, 1), dtype=torch.float64, device=dev)
    mse = torch.zeros(1, dtype=torch.float64, device=dev)
    cam_imp = D.empty((max(S, 1), max(n, 1)), dev) if want_cam_imp else None
    ptrs = (ctypes.c_void_p * max(S, 1))(*[t.data_ptr() for t in imgs])
    ctx.call("potr_score_views_self", ctypes.byref(ds.struct()), S,
             _native.camera_array(cameras), ptrs, D.ptr(imp), D.ptr(cam_imp), D.ptr(dm),
             D.ptr(mse))
    ctx.call("potr_finalize_stats", ctypes.c_int64(n), S, D.ptr(imp), D.ptr(dm), D.ptr(mse))
    return (imgs, imp[:n], cam_imp[:S, :n] if cam_imp is not None else None, dm[:n], mse)


def render_targets_and_delta_mse(splats, cameras):
    """(render_targets(splats, cameras), compute_delta_mse(splats, cameras,
    those targets)) from one pass; bit-identical to the two calls."""
    if not cameras:
        raise ZeroDivisionError("float division by zero")
    dev = D.current_device()
    ds = D.DeviceSplats.from_host(splats, dev)
    n = ds.n
    imgs, imp, cam_imp, dm, mse = render_and_score_device(ds, cameras)
    targets = []
    for image in imgs:
        img = D.to_host(image)
        img.flags.writeable = False
        targets.append(img)
    host = D.to_host(torch.cat([imp, dm, mse]))
    return targets, ForwardStats(host[:n], D.LazyHostArray(cam_imp), host[n:2 * n],
                                 float(host[2 * n]))


def compute_importance(splats, cameras, threads=1):
    """Per-splat importance plus the per-camera breakdown (:355-358)."""
    stats = forward_stats(splats, cameras, targets=None, threads=threads)
    return stats.importance, stats.camera_importance


def compute_delta_mse(splats, cameras, targets, threads=1):
    """Exact MSE change of removing each splat, against fixed targets (:361-368)."""
    for s, cam in enumerate(cameras):
        if targets[s].shape != (cam.height, cam.width, 3):
            raise ValueError(
                f"target {s} has shape {targets[s].shape}, camera expects "
                f"{(cam.height, cam.width, 3)}")
    return forward_stats(splats, cameras, targets=targets, threads=threads)


def render_targets_device(splats, cameras):
    """All views rendered in view batches; device (H, W, 3) tensors."""
    ctx = D.context()
    dev = D.current_device()
    ds = D.DeviceSplats.from_host(splats, dev)
    imgs = [D.empty((int(c.height), int(c.width), 3), dev) for c in cameras]
    if cameras:
        ptrs = (ctypes.c_void_p * len(imgs))(*[t.data_ptr() for t in imgs])
        ctx.call("potr_render_batch", ctypes.byref(ds.struct()), len(cameras),
                 _native.camera_array(cameras), ptrs, None)
    return imgs


def render_targets(splats, cameras, threads=1):
    """Reference renders of the uncompressed model, read-only (:371-377)."""
    imgs = []
    for image in render_targets_device(splats, cameras):
        img = D.to_host(image)
        img.flags.writeable = False
        imgs.append(img)
    return imgs
