"""KDE contour construction on the device KDE.

Upstream of the solve: the reference turns a predicted spectrum into circular
contours with its Algorithm 1 (`/root/reference/pkg/src/cieig/contours.py`:
`kde_sparsity` 175-192, `find_cut` 195-227, `construct_contours` 230-320,
types 140-168).  The density G(t) = sum_j exp(-w/(end-start)^2 (t - lambda_j)^2)
is evaluated by `cirr_kde_eval` (one thread per abscissa, eigenvalues staged
through shared memory, summed in index order like the reference's numba loop,
kernels.py:58-67); the cut search and the split / merge bookkeeping are host
control flow on those values, as in the reference.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .contours import Contour
from .errors import CutUndefinedError, EmptyPredictionError, ParameterError

GOLDEN = (np.sqrt(5.0) - 1.0) / 2.0        # contours.py:22
SCAN_POINTS = 2048                          # contours.py:23


@dataclass(frozen=True)
class SpectrumPrediction:
    """Predicted eigenvalues, ascending (contours.py:140-157)."""

    values: np.ndarray
    source: str = "manual"
    problem_id: str = ""

    def __post_init__(self):
        if len(self.values) == 0:
            raise EmptyPredictionError("prediction holds no values")
        if np.any(np.diff(self.values) < 0):
            raise ParameterError("prediction values must ascend")

    @property
    def m(self) -> int:
        return len(self.values)


@dataclass(frozen=True)
class Interval:
    start: float
    end: float
    count: int


@dataclass(frozen=True)
class IntervalPartition:
    intervals: tuple


def kde_eval(ts, eigs, coef: float) -> np.ndarray:
    """sum_j exp(-coef (t_i - eigs_j)^2) for every t_i, on the device."""
    from .solvers import _h2d, _ptr, _stream, _torch
    torch = _torch()
    ts = np.ascontiguousarray(ts, dtype=np.float64)
    eigs = np.ascontiguousarray(eigs, dtype=np.float64)
    if ts.size == 0:
        return np.zeros(0)
    t_d = _h2d(ts)
    e_d = _h2d(eigs) if eigs.size else torch.zeros(1, dtype=torch.float64, device="cuda")
    out = torch.empty(ts.size, dtype=torch.float64, device="cuda")
    _lib.call("cirr_kde_eval", _ptr(t_d), ts.size, _ptr(e_d), eigs.size, float(coef), _ptr(out), _stream())
    return out.cpu().numpy()


def kde_sparsity(start: float, end: float, eigs_in, w: float, t):
    """Gaussian-kernel spectral density on [start, end] (contours.py:175-192)."""
    if end <= start:
        raise ParameterError("degenerate interval")
    if w <= 0:
        raise ParameterError("kernel weight must be positive")
    eigs = np.asarray(eigs_in, dtype=float)
    scalar = np.ndim(t) == 0
    ts = np.atleast_1d(np.asarray(t, dtype=float))
    out = np.zeros_like(ts) if eigs.size == 0 else kde_eval(ts, eigs, w / (end - start) ** 2)
    return float(out[0]) if scalar else out


def find_cut(start: float, end: float, eigs_in, w: float) -> float:
    """Sparsest point of (start, end) (contours.py:195-227): a scan of
    SCAN_POINTS interior abscissae, the first minimum, then golden-section
    refinement of its bracket down to 1e-10 of the width, ties going left."""
    eigs = np.asarray(eigs_in, dtype=float)
    if eigs.size < 2:
        raise CutUndefinedError("need at least 2 eigenvalues to cut")
    width = end - start
    ts = np.linspace(start, end, SCAN_POINTS + 2)[1:-1]
    g = kde_sparsity(start, end, eigs, w, ts)
    i = int(np.argmin(g))
    a = ts[i - 1] if i > 0 else start
    b = ts[i + 1] if i < len(ts) - 1 else end
    coef = w / (end - start) ** 2

    def f(t):
        return float(kde_eval(np.array([t]), eigs, coef)[0])

    c, d = b - GOLDEN * (b - a), a + GOLDEN * (b - a)
    fc, fd = f(c), f(d)
    while (b - a) > 1e-10 * width:
        if fc <= fd:
            b, d, fd = d, c, fc
            c = b - GOLDEN * (b - a)
            fc = f(c)
        else:
            a, c, fc = c, d, fd
            d = a + GOLDEN * (b - a)
            fd = f(d)
    return 0.5 * (a + b)


def construct_contours(pred: SpectrumPrediction, n_min: int = 10, n_max: int = 50, w: float = 10.0,
                       margin: float = 0.5):
    """Adaptive KDE partition into circles (contours.py:230-320): split every
    interval holding more than n_max predictions at its sparsest point, merge
    intervals under n_min into the neighbour across the smaller gap, re-split,
    repeat to a fixed point (at most 10 sweeps); one circle per interval."""
    if n_min < 1 or n_max < n_min:
        raise ParameterError("need 1 <= n_min <= n_max")
    if margin < 0:
        raise ParameterError("margin must be non-negative")
    vals = np.sort(np.asarray(pred.values, dtype=float))
    m = len(vals)
    span = vals[-1] - vals[0]
    if span == 0.0:
        span = max(abs(vals[0]), 1.0) * 1e-6
    ext = margin * span / m
    lo, hi = vals[0] - ext, vals[-1] + ext
    if ext == 0.0:
        pad = 1e-12 * max(span, 1.0)
        lo, hi = lo - pad, hi + pad

    def split(start, end, i0, i1):
        # segments (start, end, first index, one past the last) over the sorted values
        if i1 - i0 <= n_max:
            return [(start, end, i0, i1)]
        cut = find_cut(start, end, vals[i0:i1], w)
        mid = i0 + int(np.searchsorted(vals[i0:i1], cut))
        if mid in (i0, i1):          # the cut missed the owned values: median split
            mid = i0 + (i1 - i0) // 2
            cut = 0.5 * (vals[mid - 1] + vals[mid])
        return split(start, cut, i0, mid) + split(cut, end, mid, i1)

    segs = split(lo, hi, 0, m)
    for _ in range(10):
        changed = False
        k = 0
        while len(segs) > 1 and k < len(segs):
            s0, e0, a0, b0 = segs[k]
            if b0 - a0 >= n_min:
                k += 1
                continue
            gl = gr = np.inf
            if k > 0:
                la, lb = segs[k - 1][2], segs[k - 1][3]
                gl = vals[a0] - vals[lb - 1] if lb > la and b0 > a0 else 0.0
            if k < len(segs) - 1:
                ra, rb = segs[k + 1][2], segs[k + 1][3]
                gr = vals[ra] - vals[b0 - 1] if rb > ra and b0 > a0 else 0.0
            if gl <= gr:
                ps, _, pa, _ = segs[k - 1]
                segs[k - 1:k + 1] = [(ps, e0, pa, b0)]
            else:
                _, ne, _, nb = segs[k + 1]
                segs[k:k + 2] = [(s0, ne, a0, nb)]
            changed = True
        resplit = []
        for s0, e0, a0, b0 in segs:
            if b0 - a0 > n_max:
                resplit.extend(split(s0, e0, a0, b0))
                changed = True
            else:
                resplit.append((s0, e0, a0, b0))
        segs = resplit
        if not changed:
            break
    intervals = tuple(Interval(s0, e0, b0 - a0) for s0, e0, a0, b0 in segs)
    contours = [Contour(shape="circle", center=complex(0.5 * (iv.start + iv.end), 0.0),
                        radius=0.5 * (iv.end - iv.start), expected_count=iv.count, source="kde")
                for iv in intervals]
    return IntervalPartition(intervals=intervals), contours
