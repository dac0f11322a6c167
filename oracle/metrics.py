"""Shot-level disruption alarms and ROC / AUC (NEXT-4, the
figure of merit of Figs. 3-4, :123-127).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): used by tests/ and
tools/convergence.py to score what the CUDA path trained; never by the
product path.

PAPER.md:171: "The LSTM outputs a plasma disruptivity signal which is counted
as an alarm when it passes a user-defined threshold.  Calling an alarm at any
point during a non-disruptive shot counts as a false positive (FP).  Calling
an alarm before the 30 ms cutoff during a disruptive shot counts as a true
positive (TP) ... Varying the threshold traces out an ROC curve ... The
validation level area under the ROC curve, or AUC".

Readings (Q27): the ROC is shot-level; a shot's score is the
maximum of its disruptivity trace over the legal alarm window -- every step
for a non-disruptive shot, steps t <= t_disrupt - 30 for a disruptive one
(1 ms sampling, so 30 ms = 30 steps); an alarm is raised iff
score > threshold (strict); thresholds sweep the distinct scores, ties
grouped; AUC by the trapezoid rule over the ROC points.
"""
from __future__ import annotations

import numpy as np

CUTOFF_STEPS = 30  # 30 ms at 1 ms sampling


def shot_score(trace, disruptive: bool, t_disrupt: int = None, cutoff: int = CUTOFF_STEPS) -> float:
    """Max of the trace over the legal alarm window."""
    trace = np.asarray(trace, np.float64)
    if not disruptive:
        return float(np.max(trace))
    last = t_disrupt - cutoff
    if last < 0:
        raise ValueError("no legal alarm window: t_disrupt < cutoff")
    return float(np.max(trace[:last + 1]))


def roc_curve(scores, labels):
    """ROC points (fpr, tpr) from (0, 0) to (1, 1): alarm iff score > threshold,
    thresholds = +inf then every distinct score in decreasing order."""
    s = np.asarray(scores, np.float64)
    y = np.asarray(labels).astype(bool)
    P, Nn = int(y.sum()), int((~y).sum())
    if P == 0 or Nn == 0:
        raise ValueError("ROC needs both classes")
    pts = [(0.0, 0.0)]
    for thr in np.unique(s)[::-1]:
        alarm = s >= thr          # = "score > the next lower threshold": ties grouped
        pts.append((float(np.sum(alarm & ~y)) / Nn, float(np.sum(alarm & y)) / P))
    return pts


def auc_trapezoid(scores, labels) -> float:
    pts = roc_curve(scores, labels)
    a = 0.0
    for (x0, y0), (x1, y1) in zip(pts[:-1], pts[1:]):
        a += (x1 - x0) * (y0 + y1) / 2.0
    return a


def auc_mann_whitney(scores, labels) -> float:
    """Pair-counting definition: P(score_pos > score_neg) + 1/2 P(equal)."""
    s = np.asarray(scores, np.float64)
    y = np.asarray(labels).astype(bool)
    pos, neg = s[y], s[~y]
    gt = (pos[:, None] > neg[None, :]).sum()
    eq = (pos[:, None] == neg[None, :]).sum()
    return float(gt + 0.5 * eq) / (pos.size * neg.size)
