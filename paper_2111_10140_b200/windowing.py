"""Host preprocessing around the hot path (fit's caller side), same semantics as
the reference: population-std z-scoring (data.py:122-150), histogram mutual
information feature ranking (anova.py:20-88) and greedy 3-feature windows
(anova.py:124-135).  O(N d) numpy work done once per fit; not the matvec.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import ShapeError, ValidationError
from .operators import WINDOW_SIZE, WindowSet


@dataclass
class ScalerStats:
    """Per-feature mean and population std of the training rows (zero std -> 1)."""

    means: np.ndarray
    stds: np.ndarray


def zscore_fit(X):
    X = np.atleast_2d(np.asarray(X, dtype=np.float64))
    if X.shape[0] == 0:
        raise ValidationError("cannot fit a scaler on an empty dataset")
    stds = X.std(axis=0)
    return ScalerStats(means=X.mean(axis=0), stds=np.where(stds == 0.0, 1.0, stds))


def zscore_apply(stats, X):
    X = np.atleast_2d(np.asarray(X, dtype=np.float64))
    if X.shape[1] != stats.means.shape[0]:
        raise ValidationError(
            f"matrix has {X.shape[1]} columns, scaler was fitted on {stats.means.shape[0]}")
    return (X - stats.means) / stats.stds


class MisReport:
    """Mutual information scores (nats) and the ranking: descending, ties by index."""

    def __init__(self, scores):
        self.scores = np.asarray(scores, dtype=np.float64)
        self.ranking = np.lexsort((np.arange(self.scores.size), -self.scores)).astype(np.int64)

    def to_dict(self):
        return {"scores": [float(s) for s in self.scores],
                "ranking": [int(i) for i in self.ranking]}


def _labels_pm1(y):
    y = np.asarray(y)
    if y.ndim != 1 or y.size == 0:
        raise ShapeError("labels must form a nonempty vector")
    vals = np.unique(y)
    if not np.all(np.isin(vals, (-1, 1))):
        raise ValidationError(f"labels must be -1 or +1, got values {vals}")
    if vals.size < 2:
        raise ValidationError("both classes must be present")
    return y.astype(np.int64)


def mis_scores(X, y, bins=None):
    """Plug-in histogram I(feature; label) with min(64, ceil(sqrt N)) equal-width bins."""
    X = np.atleast_2d(np.asarray(X, dtype=np.float64))
    if X.ndim != 2 or X.shape[0] == 0:
        raise ShapeError("feature matrix must be a nonempty (N, d) array")
    y = _labels_pm1(y)
    if y.shape[0] != X.shape[0]:
        raise ShapeError("feature matrix and labels must have the same length")
    N = X.shape[0]
    if N < 2:
        raise ValidationError("mutual information needs at least 2 samples")
    bins = min(64, math.ceil(math.sqrt(N))) if bins is None else bins
    pos = y > 0
    npos = int(pos.sum())
    plab = np.array([(N - npos) / N, npos / N])
    scores = np.zeros(X.shape[1])
    for j in range(X.shape[1]):
        col = X[:, j]
        lo, hi = col.min(), col.max()
        if hi == lo:
            continue
        idx = np.minimum((bins * (col - lo) / (hi - lo)).astype(np.int64), bins - 1)
        joint = np.stack([np.bincount(idx[~pos], minlength=bins),
                          np.bincount(idx[pos], minlength=bins)], axis=1) / N
        prod = joint.sum(axis=1)[:, None] * plab[None, :]
        nz = joint > 0
        scores[j] = float(np.sum(joint[nz] * np.log(joint[nz] / prod[nz])))
    return MisReport(scores)


def build_windows(report, threshold=0.0):
    """Keep features scoring >= threshold, chunk them 3 at a time in ranking order."""
    if threshold < 0:
        raise ValidationError("threshold must be nonnegative")
    kept = [int(i) for i in report.ranking if report.scores[i] >= threshold]
    if not kept:
        raise ValidationError(
            f"no feature has a mutual information score >= {threshold}; empty model")
    return WindowSet([tuple(kept[i:i + WINDOW_SIZE]) for i in range(0, len(kept), WINDOW_SIZE)])
