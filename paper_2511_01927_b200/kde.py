"""Device KDE density for the reference's contour construction (SURVEY.md
§8(f) row 4).

The contour construction itself (Algorithm 1: `kde_sparsity`, `find_cut`,
`construct_contours`, `/root/reference/pkg/src/cieig/contours.py:175-320`)
stays upstream as the reference's own code, as the north star asks. Its only
numeric kernel is the density

    G(t_i) = sum_j exp(-coef (t_i - lambda_j)^2)

which the reference evaluates with `cieig.kernels.kde_eval` (numba loop,
kernels.py:58-67), imported into `cieig.contours` by name (contours.py:20)
and looked up at call time (contours.py:191). `install(cieig)` swaps that
name for `kde_eval` below, so every 2048-point scan and every golden-section
probe of the unmodified reference evaluates on the device (`cirr_kde_eval`:
one thread per abscissa, eigenvalues staged through shared memory, summed in
index order like the numba loop). `patch.install` calls it.
"""
from __future__ import annotations

import numpy as np

from . import _lib

_ORIG: dict = {}


def kde_eval(ts, eigs, coef: float) -> np.ndarray:
    """sum_j exp(-coef (t_i - eigs_j)^2) for every t_i, on the device
    (same signature and result as cieig.kernels.kde_eval)."""
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


def install(cieig) -> None:
    """Point the reference's contour construction at the device density."""
    import cieig.contours  # noqa: F401

    if "contours.kde_eval" not in _ORIG:
        _ORIG["contours.kde_eval"] = cieig.contours.kde_eval
    cieig.contours.kde_eval = kde_eval


def uninstall(cieig) -> None:
    if "contours.kde_eval" in _ORIG:
        cieig.contours.kde_eval = _ORIG.pop("contours.kde_eval")
