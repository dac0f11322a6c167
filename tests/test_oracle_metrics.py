"""Pins for oracle.metrics (NEXT-4: shot-level alarms, ROC / AUC).

Examples from SPEC.md:420-437 (eval module); the trapezoid AUC is pinned to the
independent Mann-Whitney pair-counting definition and to the AUC invariants."""
import numpy as np
import pytest

from oracle import metrics


def test_shot_score_windows():
    # constant trace; spike 10 steps before the disruption is past the
    # 30 ms cutoff (excluded), 50 steps before counts
    assert metrics.shot_score(np.full(100, 0.3), False) == 0.3
    assert metrics.shot_score(np.full(100, 0.3), True, t_disrupt=99) == 0.3
    tr = np.zeros(100)
    tr[89] = 5.0
    assert metrics.shot_score(tr, True, t_disrupt=99) == 0.0
    assert metrics.shot_score(tr, False) == 5.0        # any alarm in a non-disruptive shot counts
    tr = np.zeros(100)
    tr[49] = 5.0
    assert metrics.shot_score(tr, True, t_disrupt=99) == 5.0
    tr = np.zeros(100)
    tr[69] = 5.0                                      # exactly t_disrupt - 30: still legal
    assert metrics.shot_score(tr, True, t_disrupt=99) == 5.0
    with pytest.raises(ValueError):
        metrics.shot_score(tr, True, t_disrupt=20)


def test_auc_examples():
    # SPEC.md:431-434
    assert metrics.auc_trapezoid([0.9, 0.8, 0.7, 0.1], [1, 0, 1, 0]) == pytest.approx(0.75, abs=1e-15)
    assert metrics.auc_trapezoid([3, 4, 1, 2], [1, 1, 0, 0]) == 1.0
    assert metrics.auc_trapezoid([0.5] * 6, [1, 0, 1, 0, 0, 1]) == 0.5
    with pytest.raises(ValueError):
        metrics.auc_trapezoid([1, 2], [1, 1])


def test_auc_equals_mann_whitney_and_invariants():
    rng = np.random.default_rng(0)
    for _ in range(1000):
        n = int(rng.integers(2, 40))
        s = np.round(rng.normal(size=n), int(rng.integers(0, 3)))   # rounding creates ties
        y = rng.random(n) < 0.4
        if y.all() or not y.any():
            continue
        a = metrics.auc_trapezoid(s, y)
        assert abs(a - metrics.auc_mann_whitney(s, y)) < 1e-12
        assert abs(metrics.auc_trapezoid(np.exp(3 * s), y) - a) < 1e-12      # strictly increasing map
        assert abs(metrics.auc_trapezoid(s, ~y) - (1 - a)) < 1e-12           # flipped labels
        pts = metrics.roc_curve(s, y)
        assert pts[0] == (0.0, 0.0) and pts[-1] == (1.0, 1.0)
        assert all(b[0] >= a_[0] and b[1] >= a_[1] for a_, b in zip(pts[:-1], pts[1:]))
