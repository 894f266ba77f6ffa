"""Pruning controller over GPU scores (reference: potr/pruning.py).

SURVEY.md section 8(f) row 1.  The functions restate the reference's numpy
semantics (stable argsort on the V-shaped priority, sequential cumsum
crossing the budget, zero-importance sweep) and give the bit-exact prune mask.

run_pruning is device-resident when it drives this package's own scorer: the
splats are uploaded once and subset in HBM between iterations, the targets
stay resident, and the O(N log N) removal order is a stable GPU sort of the
same fp64 priorities (bitwise equal to numpy's, -0.0 canonicalised).  The O(N)
budget sum and the cumulative-importance crossing run in numpy on the
downloaded scores, so the mask is bit-identical to the reference's.
"""

from dataclasses import dataclass, field

import numpy as np

from .rasterizer import compute_delta_mse


@dataclass
class PruneConfig:
    """pruning.py:17-29."""

    delta_mse_max: float
    a: float = 10.0
    iterations: int = 48

    def __post_init__(self):
        if self.delta_mse_max <= 0:
            raise ValueError("delta_mse_max must be > 0")
        if self.a <= 0:
            raise ValueError("a must be > 0")
        if self.iterations < 1:
            raise ValueError("iterations must be >= 1")


@dataclass
class PruneIterationReport:
    iteration: int
    budget: float
    removed: int
    removed_importance: float
    cumulative_removed_importance: float
    splats_before: int
    splats_after: int
    mse: float
    removed_ids: np.ndarray = field(repr=False, default=None)

    def to_dict(self):
        return {k: getattr(self, k) for k in (
            "iteration", "budget", "removed", "removed_importance",
            "cumulative_removed_importance", "splats_before", "splats_after", "mse")}


def mapping_m(x, a=10.0):
    """V-shaped removal priority (pruning.py:57-66): identity for x >= 0,
    (sqrt(1 - 2 a x) - 1) / a for x < 0."""
    x = np.asarray(x, dtype=np.float64)
    neg = (np.sqrt(1.0 - 2.0 * a * np.minimum(x, 0.0)) - 1.0) / a
    out = np.where(x >= 0.0, x, neg)
    return float(out) if out.ndim == 0 else out


def compute_budget(delta_mse, importance, delta_mse_max, remaining_iterations):
    """Eligible importance mass spread over the remaining iterations (:69-77)."""
    if remaining_iterations < 1:
        raise ValueError("remaining_iterations must be >= 1")
    delta_mse = np.asarray(delta_mse, dtype=np.float64)
    importance = np.asarray(importance, dtype=np.float64)
    return float(importance[delta_mse < delta_mse_max].sum() / remaining_iterations)


def removal_order(delta_mse, delta_mse_max, a=10.0):
    """All indices by ascending removal score, ties by index (:80-83)."""
    return np.argsort(mapping_m(np.asarray(delta_mse, dtype=np.float64) / delta_mse_max, a),
                      kind="stable")


def select_removal_set(delta_mse, importance, budget, delta_mse_max, a=10.0):
    """One iteration's removal set (:86-111): eligible splats in score order
    until cumulative importance reaches the budget (crossing splat included);
    zero-importance splats are always taken."""
    delta_mse = np.asarray(delta_mse, dtype=np.float64)
    importance = np.asarray(importance, dtype=np.float64)
    cand = np.nonzero(delta_mse < delta_mse_max)[0]
    if len(cand) == 0:
        return np.empty(0, dtype=np.int64)
    cand = cand[np.argsort(mapping_m(delta_mse[cand] / delta_mse_max, a), kind="stable")]
    imp = importance[cand]
    positive = imp > 0.0
    take = ~positive
    if budget > 0.0:
        cum = np.cumsum(np.where(positive, imp, 0.0))
        crossed = np.nonzero(cum >= budget)[0]
        cut = int(crossed[0]) if len(crossed) else len(cand) - 1
        take = take.copy()
        take[:cut + 1] = True
    return np.sort(cand[take])


def _removal_order_device(dm_dev, idx_dev, delta_mse_max, a):
    """idx_dev[stable argsort of m(dm / max)] on the GPU (pruning.py:80-83,
    :99-100): potr_removal_order computes the priorities with numpy's
    operation order and IEEE division and sorts them with the library's
    stable radix sort (ties keep the candidate order)."""
    import ctypes
    import torch
    from . import device as D
    idx = idx_dev.to(torch.int64).contiguous() if idx_dev is not None else None
    n = int(idx.numel()) if idx is not None else int(dm_dev.numel())
    order = torch.empty(max(n, 1), dtype=torch.int64, device=dm_dev.device)
    D.context().call("potr_removal_order", ctypes.c_int64(n), D.ptr(dm_dev.contiguous()),
                     D.ptr(idx), ctypes.c_double(delta_mse_max), ctypes.c_double(a),
                     D.ptr(order))
    return order[:n]


def select_removal_set_device(dm_dev, delta_mse, importance, budget, delta_mse_max, a=10.0):
    """select_removal_set with the candidate ordering sorted on the device."""
    import torch
    from . import device as D
    cand_dev = torch.nonzero(dm_dev < delta_mse_max).squeeze(1)
    if cand_dev.numel() == 0:
        return np.empty(0, dtype=np.int64)
    cand = D.to_host(_removal_order_device(dm_dev, cand_dev, delta_mse_max, a))
    imp = np.asarray(importance, dtype=np.float64)[cand]
    positive = imp > 0.0
    take = ~positive
    if budget > 0.0:
        cum = np.cumsum(np.where(positive, imp, 0.0))
        crossed = np.nonzero(cum >= budget)[0]
        cut = int(crossed[0]) if len(crossed) else len(cand) - 1
        take = take.copy()
        take[:cut + 1] = True
    return np.sort(cand[take])


def _device_scorer_active():
    from . import rasterizer, distributed
    return compute_delta_mse is rasterizer.compute_delta_mse and not distributed.sharding_active()


def _check_targets(cameras, targets):
    for s, cam in enumerate(cameras):
        if targets[s].shape != (cam.height, cam.width, 3):
            raise ValueError(
                f"target {s} has shape {targets[s].shape}, camera expects "
                f"{(cam.height, cam.width, 3)}")


def _to_host_splats(ds):
    from .scene import Splats
    from . import device as D
    return Splats(D.to_host(ds.positions), D.to_host(ds.sh), D.to_host(ds.opacities),
                  D.to_host(ds.scales), D.to_host(ds.rotations))


def _run_pruning_device(splats, cameras, targets, config, report_sink, first_iteration,
                        last_iteration):
    import torch
    from . import device as D
    from .rasterizer import forward_stats_device
    _check_targets(cameras, targets)
    if len(cameras) == 0:
        raise ZeroDivisionError("float division by zero")
    dev = D.current_device()
    ds = D.DeviceSplats.from_host(splats, dev)
    dev_targets = D.targets_cache.get(targets, cameras, dev)
    kept = np.arange(ds.n, dtype=np.int64)
    reports = []
    cum_removed = 0.0
    for it in range(first_iteration, last_iteration + 1):
        imp_d, _, dm_d, mse_d = forward_stats_device(ds, cameras, dev_targets,
                                                     want_cam_imp=False)
        host = D.to_host(torch.cat([imp_d, dm_d, mse_d]))
        n = ds.n
        importance, delta_mse, mse = host[:n], host[n:2 * n], float(host[2 * n])
        if not (delta_mse < config.delta_mse_max).any():
            break
        remaining = config.iterations - it + 1
        budget = compute_budget(delta_mse, importance, config.delta_mse_max, remaining)
        sel = select_removal_set_device(dm_d, delta_mse, importance, budget,
                                        config.delta_mse_max, config.a)
        removed_importance = float(importance[sel].sum())
        cum_removed += removed_importance
        report = PruneIterationReport(it, budget, len(sel), removed_importance, cum_removed,
                                      n, n - len(sel), mse, kept[sel])
        reports.append(report)
        if report_sink is not None:
            report_sink(report.to_dict())
        if len(sel) == 0:
            continue
        mask = np.ones(n, dtype=bool)
        mask[sel] = False
        mask_d = torch.from_numpy(mask).to(dev)
        ds = D.DeviceSplats(ds.positions[mask_d], ds.sh[mask_d], ds.opacities[mask_d],
                            ds.scales[mask_d], ds.rotations[mask_d])
        kept = kept[mask]
    return _to_host_splats(ds), kept, reports


def run_pruning(splats, cameras, targets, config: PruneConfig, threads=1, report_sink=None,
                first_iteration=1, last_iteration=None):
    """The iterative controller (:114-163).  Returns (pruned splats, kept
    original indices, iteration reports)."""
    if last_iteration is None:
        last_iteration = config.iterations
    if _device_scorer_active():
        return _run_pruning_device(splats, cameras, targets, config, report_sink,
                                   first_iteration, last_iteration)
    current = splats
    kept = np.arange(len(splats.positions), dtype=np.int64)
    reports = []
    cum_removed = 0.0
    for it in range(first_iteration, last_iteration + 1):
        stats = compute_delta_mse(current, cameras, targets, threads=threads)
        if not (stats.delta_mse < config.delta_mse_max).any():
            break
        remaining = config.iterations - it + 1
        budget = compute_budget(stats.delta_mse, stats.importance, config.delta_mse_max,
                                remaining)
        sel = select_removal_set(stats.delta_mse, stats.importance, budget,
                                 config.delta_mse_max, config.a)
        removed_importance = float(stats.importance[sel].sum())
        cum_removed += removed_importance
        n_before = len(current.positions)
        report = PruneIterationReport(it, budget, len(sel), removed_importance, cum_removed,
                                      n_before, n_before - len(sel), stats.mse, kept[sel])
        reports.append(report)
        if report_sink is not None:
            report_sink(report.to_dict())
        if len(sel) == 0:
            continue
        mask = np.ones(n_before, dtype=bool)
        mask[sel] = False
        current = current.subset(mask)
        kept = kept[mask]
    return current, kept, reports


def _run_pruning_to_counts_device(splats, cameras, targets, cumulative_counts, delta_mse_max, a):
    import torch
    from . import device as D
    from .rasterizer import forward_stats_device
    _check_targets(cameras, targets)
    if len(cameras) == 0:
        raise ZeroDivisionError("float division by zero")
    dev = D.current_device()
    ds = D.DeviceSplats.from_host(splats, dev)
    n0 = ds.n
    dev_targets = D.targets_cache.get(targets, cameras, dev)
    kept = np.arange(n0, dtype=np.int64)
    checkpoints = []
    removed = 0
    for target in cumulative_counts:
        batch = min(target, n0) - removed
        if batch > 0:
            _, _, dm_d, _ = forward_stats_device(ds, cameras, dev_targets, want_cam_imp=False)
            order = _removal_order_device(dm_d, None, delta_mse_max, a)
            sel = np.sort(D.to_host(order[:batch]))
            mask = np.ones(ds.n, dtype=bool)
            mask[sel] = False
            mask_d = torch.from_numpy(mask).to(dev)
            ds = D.DeviceSplats(ds.positions[mask_d], ds.sh[mask_d], ds.opacities[mask_d],
                                ds.scales[mask_d], ds.rotations[mask_d])
            kept = kept[mask]
            removed = target
        checkpoints.append(kept.copy())
    return checkpoints


def run_pruning_to_counts(splats, cameras, targets, cumulative_counts, delta_mse_max, a=10.0,
                          threads=1):
    """Rate-sweep variant with fixed batch sizes (:166-190); device-resident
    (splats subset in HBM, GPU stable sort of the whole removal order) when it
    drives this package's scorer."""
    if _device_scorer_active():
        return _run_pruning_to_counts_device(splats, cameras, targets, cumulative_counts,
                                             delta_mse_max, a)
    current = splats
    kept = np.arange(len(splats.positions), dtype=np.int64)
    checkpoints = []
    removed = 0
    for target in cumulative_counts:
        batch = min(target, len(splats.positions)) - removed
        if batch > 0:
            stats = compute_delta_mse(current, cameras, targets, threads=threads)
            sel = np.sort(removal_order(stats.delta_mse, delta_mse_max, a)[:batch])
            mask = np.ones(len(current.positions), dtype=bool)
            mask[sel] = False
            current = current.subset(mask)
            kept = kept[mask]
            removed = target
        checkpoints.append(kept.copy())
    return checkpoints


def importance_baseline_keep(importance, remove_count):
    """Drop the remove_count lowest-importance splats in one shot (:193-197)."""
    order = np.argsort(np.asarray(importance, dtype=np.float64), kind="stable")
    return np.sort(order[remove_count:])
