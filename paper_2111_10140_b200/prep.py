"""Caller-side preprocessing that ``fit`` needs before the hot path runs.

SURVEY.md §2 puts feature ranking and windowing OUT OF SCOPE for the GPU work;
this module is only the glue that keeps ``fit`` a drop-in for the reference's
(z-scoring, data.py:122-150; histogram mutual-information ranking and greedy
3-feature windows, anova.py:17-135).  It is O(N d) host numpy run once per fit:
all features are binned and counted in ONE ``bincount`` over (feature, bin,
label) codes, and the windows are cut from the ranking in one slice.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import ShapeError, ValidationError
from .operators import WINDOW_SIZE, WindowSet


@dataclass
class ScalerStats:
    """Training means and population stds (a zero std is stored as 1)."""

    means: np.ndarray
    stds: np.ndarray


def zscore_fit(X):
    A = np.atleast_2d(np.asarray(X, dtype=np.float64))
    if A.shape[0] == 0:
        raise ValidationError("cannot fit a scaler on an empty dataset")
    sd = A.std(axis=0)
    sd[sd == 0.0] = 1.0
    return ScalerStats(means=A.mean(axis=0), stds=sd)


def zscore_apply(stats, X):
    A = np.atleast_2d(np.asarray(X, dtype=np.float64))
    want = stats.means.shape[0]
    if A.shape[1] != want:
        raise ValidationError(f"matrix has {A.shape[1]} columns, scaler was fitted on {want}")
    return (A - stats.means) / stats.stds


class MisReport:
    """Scores (nats) per feature; ``ranking`` orders features by descending score, ties by
    ascending index."""

    def __init__(self, scores):
        self.scores = np.asarray(scores, dtype=np.float64)
        idx = np.arange(self.scores.size)
        self.ranking = np.lexsort((idx, -self.scores)).astype(np.int64)

    def to_dict(self):
        return {"scores": self.scores.tolist(), "ranking": self.ranking.tolist()}


def _binary_labels(y):
    lab = np.asarray(y)
    if lab.ndim != 1 or lab.size == 0:
        raise ShapeError("labels must form a nonempty vector")
    present = np.unique(lab)
    if not np.isin(present, (-1, 1)).all():
        raise ValidationError(f"labels must be -1 or +1, got values {present}")
    if present.size < 2:
        raise ValidationError("both classes must be present")
    return lab > 0


def mis_scores(X, y, bins=None):
    """Plug-in I(feature; label) from equal-width histograms over each feature's range
    (``min(64, ceil(sqrt N))`` bins by default); constant features score 0."""
    A = np.atleast_2d(np.asarray(X, dtype=np.float64))
    if A.ndim != 2 or A.shape[0] == 0:
        raise ShapeError("feature matrix must be a nonempty (N, d) array")
    pos = _binary_labels(y)
    N, d = A.shape
    if pos.shape[0] != N:
        raise ShapeError("feature matrix and labels must have the same length")
    if N < 2:
        raise ValidationError("mutual information needs at least 2 samples")
    nb = int(bins) if bins is not None else min(64, math.ceil(math.sqrt(N)))
    lo, hi = A.min(axis=0), A.max(axis=0)
    live = hi > lo
    span = np.where(live, hi - lo, 1.0)
    binned = np.minimum((nb * (A - lo) / span).astype(np.int64), nb - 1)
    code = (binned + np.arange(d) * nb) * 2 + pos[:, None]
    joint = np.bincount(code.ravel(), minlength=2 * nb * d).reshape(d, nb, 2) / N
    p1 = pos.sum() / N
    marg = joint.sum(axis=2, keepdims=True) * np.array([1.0 - p1, p1])
    hit = joint > 0
    terms = np.zeros_like(joint)
    terms[hit] = joint[hit] * np.log(joint[hit] / marg[hit])
    return MisReport(np.where(live, terms.sum(axis=(1, 2)), 0.0))


def build_windows(report, threshold=0.0):
    """Features scoring >= threshold, in ranking order, cut into windows of 3."""
    if threshold < 0:
        raise ValidationError("threshold must be nonnegative")
    order = report.ranking[report.scores[report.ranking] >= threshold].tolist()
    if not order:
        raise ValidationError(
            f"no feature has a mutual information score >= {threshold}; empty model")
    return WindowSet([tuple(order[k:k + WINDOW_SIZE]) for k in range(0, len(order), WINDOW_SIZE)])
