"""The pruning controller (host logic over scores, pruning.py mirror).

Its re-scoring call is pointed at the CPU oracle here (test infrastructure;
the product calls the CUDA path), which pins the controller's bit-exact
mask semantics against the reference's own 48-iteration run."""

import numpy as np
import pytest

from tests.conftest import golden, small_scene


def test_mapping_m_shape():
    from paper_2601_14821_b200.pruning import mapping_m
    assert mapping_m(0.0) == 0.0 and mapping_m(0.5) == 0.5
    xs = np.linspace(-5, 0, 11)
    m = mapping_m(xs)
    assert np.all(m[:-1] > 0) and np.all(np.diff(m) < 0)  # V-shaped: decreasing on negatives
    assert mapping_m(-1.0, a=10.0) == pytest.approx((np.sqrt(21.0) - 1.0) / 10.0)


def test_select_removal_set_rules():
    from paper_2601_14821_b200.pruning import select_removal_set
    dm = np.array([0.5, -1.0, 0.1, 5.0, 0.2])
    imp = np.array([0.3, 0.2, 0.0, 0.9, 0.4])
    sel = select_removal_set(dm, imp, budget=0.25, delta_mse_max=1.0)
    # order by m: 0.1 (id2, zero importance), 0.2 (id4), 0.5 (id0), -1 -> m=0.358 (id1)
    assert list(sel) == [2, 4]
    assert list(select_removal_set(dm, imp, 0.0, 1.0)) == [2]
    assert list(select_removal_set(dm, imp, 1.0, 0.01)) == [1]  # only the improving splat is eligible


def test_run_pruning_matches_reference_kept_set(monkeypatch):
    from oracle import oracle as O
    from paper_2601_14821_b200 import pruning
    from paper_2601_14821_b200.rasterizer import ForwardStats

    def oracle_delta_mse(splats, cams, targets, threads=1):
        imp, ci, dm, mse = O.forward_stats(splats, cams, targets, threads=4)
        return ForwardStats(imp, ci, dm, mse)

    monkeypatch.setattr(pruning, "compute_delta_mse", oracle_delta_mse)
    splats, cams = small_scene()
    g = golden("small_scene")
    targets = list(g["targets"])
    cfg = pruning.PruneConfig(delta_mse_max=10.0 ** (-8.8 - 2.0 * 0.5))
    _, kept, reports = pruning.run_pruning(splats, cams, targets, cfg)
    assert np.array_equal(kept, g["prune_kept"])
    assert [r.removed for r in reports] == list(g["prune_removed"])
