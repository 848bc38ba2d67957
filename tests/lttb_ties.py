"""LTTB tie accounting (test infrastructure, numpy; never part of the product).

The north star allows an LTTB / MinMaxLTTB pick to differ from the
reference's only where the two best triangle areas of a bucket are within
1e-12 relative.  `near_ties` counts, along a given
sequence of picks (normally the reference's own), the buckets where that
happens; `explain_mismatches` checks that every index where a result differs
from the reference is such a bucket.  Areas use the reference formula
(_kernels.py:375-480): 0.5*|(ax-cx)*(y-ay) - (ax-x)*(cy-ay)|, f64, no FMA
(numpy evaluates each operation separately).
"""
import numpy as np


def lttb_offsets(n, n_out):
    """Bucket offsets of LTTB over the interior points 1..n-2 (algorithms.py:66-79, implicit x)."""
    nb = n_out - 2
    k = np.arange(nb + 1, dtype=np.int64)
    return k * np.int64(n - 2) // np.int64(nb) + 1


def _bucket_areas(x, y, s, e, a, c):
    xs = np.arange(s, e, dtype=np.float64) if x is None else x[s:e].astype(np.float64)
    ys = y[s:e].astype(np.float64)
    ax, ay = a
    cx, cy = c
    return 0.5 * np.abs((ax - cx) * (ys - ay) - (ax - xs) * (cy - ay))


def near_ties(y, picks, off, x=None, rel=1e-12):
    """(number of buckets whose best and second-best area are within rel, list of those buckets)."""
    n = y.shape[0]
    nb = off.shape[0] - 1
    xv = (lambda i: float(i)) if x is None else (lambda i: float(x[i]))
    ties = []
    picks = np.asarray(picks, dtype=np.int64)
    prev = 0
    j = 0  # index into picks[1:-1] (the bucket picks)
    for k in range(nb):
        s, e = int(off[k]), int(off[k + 1])
        if e <= s:
            continue
        if k == nb - 1 or int(off[k + 2]) <= int(off[k + 1]):
            c = (xv(n - 1), float(y[n - 1]))
        else:
            s2, e2 = int(off[k + 1]), int(off[k + 2])
            cx = float(np.sum(np.arange(s2, e2, dtype=np.float64))) if x is None else float(np.sum(x[s2:e2], dtype=np.float64))
            c = (cx / (e2 - s2), float(np.sum(y[s2:e2].astype(np.float64))) / (e2 - s2))
        areas = _bucket_areas(x, y, s, e, (xv(prev), float(y[prev])), c)
        areas = np.where(np.isnan(areas), -1.0, areas)
        if areas.shape[0] >= 2:
            top2 = np.partition(areas, -2)[-2:]
            best, second = float(top2[1]), float(top2[0])
            if best >= 0 and best - second <= rel * best:
                ties.append(k)
        prev = int(picks[1 + j])
        j += 1
    return len(ties), ties


def explain_mismatches(got, want, y, off, x=None, rel=1e-12):
    """Indices where got != want must all lie in near-tie buckets; returns the mismatch count."""
    got, want = np.asarray(got, np.int64), np.asarray(want, np.int64)
    if got.shape == want.shape and np.array_equal(got, want):
        return 0
    assert got.shape == want.shape, "length differs"
    _, ties = near_ties(y, want, off, x=x, rel=rel)
    tie_set = set(ties)
    bad = np.nonzero(got != want)[0]
    for i in bad:
        k = int(np.searchsorted(off, want[i], side="right") - 1)
        assert k in tie_set, f"pick {i} differs outside a near-tie bucket"
    return int(bad.size)
