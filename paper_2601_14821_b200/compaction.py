"""Drop-in for potr.compaction on B200 (reference: potr/compaction.py).

compact_scene / compact_splat run kernel (e) (csrc/sh.cu): per-splat normal
equations accumulated over the cameras in HBM, then batched fp64 Cholesky
ridge solves with the reference's sparsification, two-pass zeroing, jitter
retry, RidgeError and DC-fallback semantics.  The colour-space helpers are
tiny host conversions kept for API completeness.
"""

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from . import device as D

# compaction.py:19-28
RGB_TO_YCOCG = np.array([
    [0.25, 0.5, 0.25],
    [0.5, 0.0, -0.5],
    [-0.25, 0.5, -0.25],
])
YCOCG_TO_RGB = np.array([
    [1.0, 1.0, -1.0],
    [1.0, 0.0, 1.0],
    [1.0, -1.0, -1.0],
])

STATUS_OK, STATUS_JITTER, STATUS_FAILED, STATUS_DC_FALLBACK = 0, 1, 2, 3
NEQ_STRIDE = 185  # POTR_NEQ_STRIDE: G upper triangle 136 + B 48 + seen count


class RidgeError(RuntimeError):
    """Normal-equations factorization failed even with jitter (:40-41)."""


@dataclass
class CompactionConfig:
    """compaction.py:44-59."""

    lambda_y: float
    parallel_threshold: float
    zero_threshold: float

    def __post_init__(self):
        if self.lambda_y < 0:
            raise ValueError("lambda_y must be >= 0")
        if not 0 < self.parallel_threshold <= 1:
            raise ValueError("parallel_threshold must be in (0, 1]")

    @property
    def lambdas(self):
        """Per-channel ridge strengths; chrominance three times the luminance."""
        return np.array([self.lambda_y, 3.0 * self.lambda_y, 3.0 * self.lambda_y])


def rgb_to_ycocg(c):
    return np.asarray(c, dtype=np.float64) @ RGB_TO_YCOCG.T


def ycocg_to_rgb(c):
    return np.asarray(c, dtype=np.float64) @ YCOCG_TO_RGB.T


def coeffs_rgb_to_ycocg(sh):
    """(..., 3, 16) RGB coefficient blocks to YCoCg."""
    return np.einsum("ij,...jc->...ic", RGB_TO_YCOCG, sh)


def coeffs_ycocg_to_rgb(sh):
    return np.einsum("ij,...jc->...ic", YCOCG_TO_RGB, sh)


def _splats_ps(splats, dev):
    """Device copies of the two arrays the SH path reads."""
    if isinstance(splats, D.DeviceSplats):
        return splats
    n = len(splats.positions)
    pos = D.to_device(splats.positions, dev, (n, 3))
    sh = D.to_device(splats.sh, dev, (n, 3, 16))
    empty = torch.empty(0, dtype=torch.float64, device=dev)
    return D.DeviceSplats(pos, sh, empty, empty, empty)


def compact_device(splats, cameras, camera_importance, config):
    """Kernel (e) on the current device.  Returns device tensors
    (rgb (N,3,16), ycocg (N,3,16), status (N,) int8)."""
    ctx = D.context()
    dev = D.current_device()
    ds = _splats_ps(splats, dev)
    n, S = ds.n, len(cameras)
    ci = D.as_device_matrix(camera_importance, (S, n), dev) if S * n > 0 else None
    rgb = D.empty((max(n, 1), 3, 16), dev)
    yc = D.empty((max(n, 1), 3, 16), dev)
    status = D.empty(max(n, 1), dev, torch.int8)
    cams = _native.camera_array(cameras)
    ctx.call("potr_compact", ctypes.byref(ds.struct()), S, cams, D.ptr(ci),
             ctypes.c_double(config.lambda_y), ctypes.c_double(config.parallel_threshold),
             ctypes.c_double(config.zero_threshold), D.ptr(rgb), D.ptr(yc), D.ptr(status))
    return rgb[:n], yc[:n], status[:n]


def compact_scene(splats, cameras, camera_importance, config: CompactionConfig, threads=1):
    """Replace every splat's coefficients independently (:195-243).

    Returns (new splats, ycocg (N, 3, 16), {"failed": [...],
    "fallback_dc_only": n}); failed splats keep their original coefficients.
    """
    from .scene import Splats
    if len(splats.positions) == 0:
        return (Splats(*(np.asarray(a).copy() for a in (splats.positions, splats.sh,
                                                         splats.opacities, splats.scales,
                                                         splats.rotations))),
                np.zeros((0, 3, 16)), {"failed": [], "fallback_dc_only": 0})
    from . import distributed
    if distributed.sharding_active() or isinstance(camera_importance, distributed.ShardedRows):
        # view-sharded run: splat spans per rank (distributed.compact_scene_sharded)
        return distributed.compact_scene_sharded(splats, cameras, camera_importance, config,
                                                 group=getattr(camera_importance, "group", None))
    rgb, yc, status = compact_device(splats, cameras, camera_importance, config)
    rgb = D.to_host(rgb)
    yc = D.to_host(yc)
    status = D.to_host(status)
    failed = np.nonzero(status == STATUS_FAILED)[0]
    fallback = int(np.count_nonzero(status == STATUS_DC_FALLBACK))
    out = Splats(np.array(splats.positions, dtype=np.float64, copy=True), rgb,
                 np.array(splats.opacities, dtype=np.float64, copy=True),
                 np.array(splats.scales, dtype=np.float64, copy=True),
                 np.array(splats.rotations, dtype=np.float64, copy=True))
    return out, yc, {"failed": [int(k) for k in failed], "fallback_dc_only": fallback}


def compact_splat(splat_index, splats, cameras, camera_importance, config: CompactionConfig):
    """Recompute one splat's coefficients (:169-192); camera_importance is
    that splat's (S,) column.  Raises RidgeError like the reference."""
    from .scene import Splats
    k = int(splat_index)
    one = Splats(np.asarray(splats.positions)[k:k + 1], np.asarray(splats.sh)[k:k + 1],
                 np.asarray(splats.opacities)[k:k + 1], np.asarray(splats.scales)[k:k + 1],
                 np.asarray(splats.rotations)[k:k + 1])
    col = np.asarray(camera_importance, dtype=np.float64).reshape(len(cameras), 1)
    rgb, yc, status = compact_device(one, cameras, col, config)
    if int(status[0].item()) == STATUS_FAILED:
        raise RidgeError("singular system")
    return rgb[0].cpu().numpy(), yc[0].cpu().numpy()


def ac_sparsity(ycocg):
    """Fraction of exactly-zero AC entries in (N, 3, 16) coefficients (:246-249)."""
    ac = np.asarray(ycocg)[:, :, 1:]
    return float(np.mean(ac == 0.0))


def mean_abs_nonzero_ac(ycocg):
    ac = np.asarray(ycocg)[:, :, 1:]
    nz = ac[ac != 0.0]
    return float(np.mean(np.abs(nz))) if len(nz) else 0.0


def sweep(splats, cameras, targets, camera_importance, lambdas, alphas, zero_threshold,
          threads=1):
    """Regularization sweep (:258-278): rows of (lambda, alpha, AC sparsity,
    mean |nonzero AC|, MSE vs targets), one per (lambda, alpha).

    Device-resident: the weighted normal equations do not depend on
    (lambda, alpha), so they are accumulated once (potr_sh_normal_equations) and
    only the solves, the re-renders and the error reductions run per grid
    point; nothing but the row scalars comes back to the host."""
    from .rasterizer import render_targets_device
    ctx = D.context()
    dev = D.current_device()
    ds = D.DeviceSplats.from_host(splats, dev)
    n, S = ds.n, len(cameras)
    rows = []
    if n == 0 or S == 0:
        for alpha in alphas:
            for lam in lambdas:
                compacted, ycocg, _ = compact_scene(splats, cameras, camera_importance,
                                                    CompactionConfig(lam, alpha, zero_threshold))
                mse = 0.0
                from .rasterizer import render_image
                for s_, cam in enumerate(cameras):
                    mse += float(np.mean((render_image(compacted, cam) - targets[s_]) ** 2))
                rows.append((lam, alpha, ac_sparsity(ycocg), mean_abs_nonzero_ac(ycocg),
                             mse / len(cameras)))
        return rows
    ci = D.as_device_matrix(camera_importance, (S, n), dev)
    neq = torch.empty((NEQ_STRIDE, n), dtype=torch.float64, device=dev)
    cams = _native.camera_array(cameras)
    ctx.call("potr_sh_normal_equations", ctypes.byref(ds.struct()), S, cams, D.ptr(ci), D.ptr(neq))
    dev_targets = D.targets_cache.get(targets, cameras, dev)
    rgb = D.empty((n, 3, 16), dev)
    yc = D.empty((n, 3, 16), dev)
    status = D.empty(n, dev, torch.int8)
    for alpha in alphas:
        for lam in lambdas:
            cfg = CompactionConfig(lambda_y=lam, parallel_threshold=alpha,
                                   zero_threshold=zero_threshold)
            ctx.call("potr_sh_solve", ctypes.byref(ds.struct()), D.ptr(neq),
                     ctypes.c_double(cfg.lambda_y), ctypes.c_double(cfg.parallel_threshold),
                     ctypes.c_double(cfg.zero_threshold), D.ptr(rgb), D.ptr(yc), D.ptr(status))
            compacted = D.DeviceSplats(ds.positions, rgb, ds.opacities, ds.scales,
                                       ds.rotations)
            imgs = render_targets_device(compacted, cameras)
            errs = torch.stack([((im - t) ** 2).mean() for im, t in zip(imgs, dev_targets)])
            ac = yc[:, :, 1:]
            nz = ac != 0.0
            n_nz = int(nz.sum().item())
            sparsity = float(ac.numel() - n_nz) / ac.numel()  # == np.mean(ac == 0)
            mean_nz = float(ac.abs()[nz].mean().item()) if n_nz else 0.0
            mse = 0.0
            for e in errs.cpu().numpy():
                mse += float(e)
            rows.append((lam, alpha, sparsity, mean_nz, mse / S))
    return rows
