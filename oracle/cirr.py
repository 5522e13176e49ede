"""Numpy/scipy restatement of the reference CIRR stage -- TEST INFRASTRUCTURE.

This module is the parity oracle and the timed CPU baseline.  It is never
imported by the product package.  Each function cites the reference line it
restates (paths relative to /root/reference/pkg/src/cieig/).

Two modes, selected by ``OracleConfig``:

* ``moments="raw", lu="superlu", rr="hermitian"`` -- *reference mode*: the
  reference algorithm as written (uncentred moments S_m = sum w_j z_j^m Y_j,
  SuperLU factorisations, Hermitian-only Rayleigh-Ritz).  Pinned bit-for-bit
  in spirit (to rounding) against outputs of the unmodified reference in
  tests/golden/ref_*.npz.
* ``moments="centred"`` (default) -- the restated oracle with the deltas
  documented in SURVEY.md section 8(c) and DESIGN.md section 3:
    1. centred + radius-scaled moments ((z_j - gamma)/rho)^m  (solvers.py:126-129),
    2. ellipse contours (contours.py:40-66, 327-342 have only circle/rect),
    3. non-Hermitian Rayleigh-Ritz via scipy.linalg.eig when the pencil is not
       Hermitian (solvers.py:150-158 always symmetrises),
    4. dense LAPACK LU (scipy.linalg.lu_factor) in place of SuperLU.
  This is the same algorithm the GPU path runs.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla


class OracleError(Exception):
    pass


class SingularShiftError(OracleError):
    def __init__(self, shift, node_index=None):
        self.shift = shift
        self.node_index = node_index
        super().__init__(f"singular shifted matrix at z={shift!r} (node {node_index})")


class RankZeroError(OracleError):
    pass


class NoEigenvaluesFound(OracleError):
    pass


class ConvergenceError(OracleError):
    def __init__(self, best_residual):
        self.best_residual = best_residual
        super().__init__(f"not converged; best residual {best_residual:.3e}")


class IndefiniteBError(OracleError):
    pass


PIVOT_REL_TOL = 1e-14  # linalg.py:26


@dataclass
class OracleConfig:
    """Mirrors SolverConfig (solvers.py:25-44) plus the oracle's mode switches."""

    n_q: int = 32
    source_cols: int | None = None
    n_moments: int = 4
    max_refine: int = 8
    tol: float = 1e-10
    rank_rel_tol: float = 1e-12
    drop_tol: float = 1e-10
    moments: str = "centred"  # "centred" | "raw"
    lu: str = "dense"  # "dense" | "superlu"
    rr: str = "auto"  # "auto" | "hermitian" | "general"

    def cols_for(self, expected_count: int) -> int:  # solvers.py:41-44
        if self.source_cols is not None:
            return self.source_cols
        return max(8, 2 * expected_count)


# ---------------------------------------------------------------------------
# geometry (contours.py:59-66, 327-363 + ellipse delta)


def _shape(c):
    return getattr(c, "shape")


def contains(c, z: complex) -> bool:
    """Strict interior test (contours.py:59-66); ellipse is the delta."""
    z = complex(z)
    s = _shape(c)
    if s == "circle":
        return abs(z - c.center) < c.radius
    if s == "ellipse":
        dr = (z.real - c.center.real) / c.semi_re
        di = (z.imag - c.center.imag) / c.semi_im
        return dr * dr + di * di < 1.0
    return c.re_min < z.real < c.re_max and c.im_min < z.imag < c.im_max


def quadrature(c, n_q: int):
    """Nodes and weights (contours.py:327-363).  Ellipse (delta):
    z = c + a cos t + i b sin t, w = z'(t)/(i N) = (b cos t + i a sin t)/N."""
    if n_q < 4 or n_q % 2 != 0:
        raise ValueError("n_q must be even and >= 4")
    s = _shape(c)
    if s == "circle":
        j = np.arange(n_q)
        theta = 2.0 * np.pi * (j + 0.5) / n_q
        rot = np.exp(1j * theta)
        return c.center + c.radius * rot, c.radius * rot / n_q
    if s == "ellipse":
        j = np.arange(n_q)
        theta = 2.0 * np.pi * (j + 0.5) / n_q
        ct, st = np.cos(theta), np.sin(theta)
        nodes = c.center + (c.semi_re * ct + 1j * c.semi_im * st)
        weights = (c.semi_im * ct + 1j * c.semi_re * st) / n_q
        return nodes, weights
    if n_q % 4 != 0:
        raise ValueError("rect contours need n_q divisible by 4")
    per_edge = n_q // 4
    gl_x, gl_w = np.polynomial.legendre.leggauss(per_edge)
    corners = [complex(c.re_min, c.im_min), complex(c.re_max, c.im_min),
               complex(c.re_max, c.im_max), complex(c.re_min, c.im_max)]
    nodes, weights = [], []
    for k in range(4):
        p0, p1 = corners[k], corners[(k + 1) % 4]
        half = 0.5 * (p1 - p0)
        mid = 0.5 * (p1 + p0)
        nodes.append(mid + gl_x * half)
        weights.append(gl_w * half / (2.0j * np.pi))
    return np.concatenate(nodes), np.concatenate(weights)


def moment_frame(c):
    """(gamma, rho) of the centred/scaled moments (delta 1)."""
    s = _shape(c)
    if s == "circle":
        return complex(c.center), float(c.radius)
    if s == "ellipse":
        return complex(c.center), float(max(c.semi_re, c.semi_im))
    g = complex(0.5 * (c.re_min + c.re_max), 0.5 * (c.im_min + c.im_max))
    return g, float(max(0.5 * (c.re_max - c.re_min), 0.5 * (c.im_max - c.im_min)))


# ---------------------------------------------------------------------------
# pencil handling


def _dense(m):
    if isinstance(m, np.ndarray):
        return m
    if sp.issparse(m):
        return m.toarray()
    if hasattr(m, "to_dense"):
        return m.to_dense()
    return np.asarray(m)


class Pencil:
    """Dense (A, B) with a Hermitian flag; accepts the reference MatrixPencil."""

    def __init__(self, a, b, hermitian=None):
        self.a = np.asarray(_dense(a))
        self.b = np.asarray(_dense(b))
        if hermitian is None:
            hermitian = _is_hermitian(self.a) and _is_hermitian(self.b)
        self.hermitian = bool(hermitian)
        self.n = self.a.shape[0]

    @classmethod
    def of(cls, p):
        if isinstance(p, Pencil):
            return p
        herm = getattr(p, "hermitian", None)
        a, b = _dense(p.a), _dense(p.b)
        if herm is False:
            herm = None  # the reference flag defaults to False; decide numerically
        return cls(a, b, herm)


def _is_hermitian(m, rel_tol=1e-12):  # sparse.py:83-87
    scale = max(np.abs(m).max() if m.size else 0.0, 1e-300)
    return np.abs(m - m.conj().T).max() <= rel_tol * scale


# ---------------------------------------------------------------------------
# ProjectorContext (solvers.py:97-130, linalg.py:38-71)


class Projector:
    def __init__(self, pencil: Pencil, nodes, weights, cfg: OracleConfig,
                 frame=(0j, 1.0)):
        self.pencil = pencil
        self.nodes = np.asarray(nodes)
        self.weights = np.asarray(weights)
        self.cfg = cfg
        self.frame = frame
        self.facs = []
        a, b = pencil.a, pencil.b
        for j, z in enumerate(self.nodes):
            z = complex(z)
            m = z * b - a  # linalg.py:62
            scale = max(np.abs(m).max() if m.size else 0.0, 1e-300)  # linalg.py:63
            if cfg.lu == "superlu":
                try:
                    lu = spla.splu(sp.csc_matrix(m))  # linalg.py:65
                except RuntimeError as exc:
                    raise SingularShiftError(z, j) from exc
                piv = np.abs(lu.U.diagonal())
                fac = ("splu", lu)
            else:
                lu, ipiv = sla.lu_factor(m, check_finite=False)
                piv = np.abs(np.diag(lu))
                fac = ("dense", (lu, ipiv))
            if piv.size == 0 or piv.min() < PIVOT_REL_TOL * scale:  # linalg.py:68-70
                raise SingularShiftError(z, j)
            self.facs.append(fac)
        self.n_factorizations = len(self.facs)
        self.n_linear_solves = 0

    def _solve(self, fac, rhs):
        kind, f = fac
        if kind == "splu":
            return f.solve(rhs)
        return sla.lu_solve(f, rhs, check_finite=False)

    def apply(self, v, moments=1):
        """S_m = sum_j w_j zeta_j^m Y_j (solvers.py:113-130); zeta_j is z_j
        (raw) or (z_j - gamma)/rho (centred, delta 1)."""
        v = np.asarray(v, dtype=np.complex128)
        if v.ndim == 1:
            v = v[:, None]
        bv = self.pencil.b @ v  # solvers.py:120
        acc = [np.zeros_like(v) for _ in range(moments)]
        gamma, rho = self.frame
        for z, w, fac in zip(self.nodes, self.weights, self.facs):
            y = self._solve(fac, bv) if v.shape[1] else v.copy()
            self.n_linear_solves += v.shape[1]
            zeta = z if self.cfg.moments == "raw" else (z - gamma) / rho
            zp = 1.0 + 0.0j
            for m in range(moments):
                acc[m] += (w * zp) * y
                zp *= zeta
        return acc


def apply_projector(pencil, contour_or_rule, v, cfg: OracleConfig | None = None):
    """solvers.py:133-137: sum_j w_j (z_j B - A)^{-1} B v."""
    cfg = cfg or OracleConfig()
    p = Pencil.of(pencil)
    if isinstance(contour_or_rule, tuple):
        nodes, weights = contour_or_rule
    else:
        nodes, weights = quadrature(contour_or_rule, cfg.n_q)
    return Projector(p, nodes, weights, cfg).apply(v, 1)[0]


# ---------------------------------------------------------------------------
# rank truncation, Rayleigh-Ritz, residuals


def rank_truncate_svd(block, rel_tol=1e-12):  # linalg.py:107-119
    b = np.asarray(block, dtype=np.complex128)
    if b.shape[1] == 0:
        raise RankZeroError("empty block")
    u, s, _ = np.linalg.svd(b, full_matrices=False)
    if s.size == 0 or s[0] == 0.0:
        raise RankZeroError("zero block")
    r = int(np.count_nonzero(s >= rel_tol * s[0]))
    return u[:, :r]


def orthonormalize(block, drop_tol=1e-10):  # linalg.py:79-104
    """Gram-Schmidt with one re-orthogonalisation pass per column; a column
    whose remaining norm is <= drop_tol x its original norm is dropped."""
    b = np.array(block, dtype=np.complex128)
    if b.ndim == 1:
        b = b[:, None]
    if b.shape[1] == 0:
        raise RankZeroError("empty block")
    kept = []
    for j in range(b.shape[1]):
        v = b[:, j]
        orig = np.linalg.norm(v)
        if orig == 0.0:
            continue
        for _ in range(2):
            for q in kept:
                v = v - q * (q.conj() @ v)
        nrm = np.linalg.norm(v)
        if nrm <= drop_tol * orig:
            continue
        kept.append(v / nrm)
    if not kept:
        raise RankZeroError("all columns dropped")
    return np.column_stack(kept)


def rayleigh_ritz(pencil: Pencil, q, mode: str):
    """solvers.py:150-158 + linalg.py:122-145; 'general' is delta 3."""
    aq = pencil.a @ q
    bq = pencil.b @ q
    a_s = q.conj().T @ aq
    b_s = q.conj().T @ bq
    if mode == "general":
        w, s = sla.eig(a_s, b_s)
        order = np.lexsort((w.imag, w.real))
        return w[order], q @ s[:, order]
    a_s = 0.5 * (a_s + a_s.conj().T)
    b_s = 0.5 * (b_s + b_s.conj().T)
    if a_s.size and np.abs(a_s.imag).max() == 0.0 and np.abs(b_s.imag).max() == 0.0:
        a_s, b_s = a_s.real.copy(), b_s.real.copy()
    try:
        np.linalg.cholesky(b_s)
    except np.linalg.LinAlgError as exc:
        raise IndefiniteBError("projected B is not positive definite") from exc
    w, s = sla.eigh(a_s, b_s)
    return w, q @ s


def residuals(pencil: Pencil, lam, x):  # solvers.py:140-147
    ax = pencil.a @ x
    bx = pencil.b @ x
    num = np.linalg.norm(ax - lam[None, :] * bx, axis=0)
    den = np.linalg.norm(ax, axis=0) + np.abs(lam) * np.linalg.norm(bx, axis=0)
    den = np.where(den == 0.0, 1e-300, den)
    return num / den


def _inside(contour, lam, hermitian_rr: bool):  # solvers.py:161-162
    if hermitian_rr:
        return np.array([contains(contour, complex(v, 0.0)) for v in np.real(lam)], dtype=bool)
    return np.array([contains(contour, v) for v in lam], dtype=bool)


@dataclass
class OracleResult:
    eigenvalues: np.ndarray
    eigenvectors: np.ndarray
    residuals: np.ndarray
    contour: object
    iterations: int
    n_linear_solves: int
    n_factorizations: int
    elapsed: float
    ranks: list


def cirr_solve(pencil, contour, cfg: OracleConfig | None = None, seed: int = 0):
    """solvers.py:165-227 with the configured deltas."""
    cfg = cfg or OracleConfig()
    t0 = time.perf_counter()
    p = Pencil.of(pencil)
    nodes, weights = quadrature(contour, cfg.n_q)
    frame = moment_frame(contour)
    ctx = Projector(p, nodes, weights, cfg, frame)
    rng = np.random.default_rng(seed)
    ncols = cfg.cols_for(getattr(contour, "expected_count", 0))
    v = rng.standard_normal((p.n, ncols)).astype(complex)  # solvers.py:178-180
    if cfg.rr == "auto":
        mode = "hermitian" if p.hermitian else "general"
    else:
        mode = cfg.rr
    moments = ctx.apply(v, moments=cfg.n_moments)
    stacked = np.hstack(moments)
    best_res = np.inf
    lam = x = res = None
    ranks = []
    it = 0
    for it in range(cfg.max_refine):  # solvers.py:186-203
        try:
            q = rank_truncate_svd(stacked, cfg.rank_rel_tol)
        except RankZeroError:
            break
        ranks.append(q.shape[1])
        w, xs = rayleigh_ritz(p, q, mode)
        keep = _inside(contour, w, mode == "hermitian")
        if not np.any(keep):
            lam = None
            break
        lam, x = w[keep], xs[:, keep]
        res = residuals(p, lam, x)
        best_res = min(best_res, float(res.max()))
        if res.max() <= cfg.tol:
            break
        if it + 1 >= cfg.max_refine:
            break
        stacked = ctx.apply(x, moments=1)[0]
    elapsed = time.perf_counter() - t0
    if lam is None or lam.size == 0:  # solvers.py:211-214
        raise NoEigenvaluesFound("no eigenvalues inside contour")
    if res.max() > cfg.tol:  # solvers.py:215-219
        conv = res <= cfg.tol
        if not np.any(conv):
            raise ConvergenceError(best_res)
        lam, x, res = lam[conv], x[:, conv], res[conv]
    order = np.argsort(lam)  # solvers.py:220 (complex: lexicographic re, im)
    return OracleResult(lam[order], x[:, order], res[order], contour, it + 1,
                        ctx.n_linear_solves, ctx.n_factorizations, elapsed, ranks)


def feast_solve(pencil, contour, cfg: OracleConfig | None = None, seed: int = 0):
    """solvers.py:230-285: filtered subspace iteration U <- orth(P U) with a
    Rayleigh-Ritz extraction after each projector application (one moment,
    so the moment centring delta does not apply); the general Rayleigh-Ritz
    (delta 3) when the pencil is not Hermitian."""
    cfg = cfg or OracleConfig()
    t0 = time.perf_counter()
    p = Pencil.of(pencil)
    nodes, weights = quadrature(contour, cfg.n_q)  # 236
    ctx = Projector(p, nodes, weights, cfg, moment_frame(contour))  # 237
    rng = np.random.default_rng(seed)  # 238
    ncols = cfg.cols_for(getattr(contour, "expected_count", 0))  # 239
    u = rng.standard_normal((p.n, ncols)).astype(complex)  # 240
    mode = cfg.rr if cfg.rr != "auto" else ("hermitian" if p.hermitian else "general")
    best_res = np.inf
    lam = x = res = None
    found_any = False
    ranks = []
    for it in range(cfg.max_refine):  # 245
        y = ctx.apply(u, moments=1)[0]  # 246
        try:
            q = orthonormalize(y, cfg.drop_tol)  # 248
        except RankZeroError:  # 249-250
            break
        ranks.append(q.shape[1])
        w, xs = rayleigh_ritz(p, q, mode)  # 251
        keep = _inside(contour, w, mode == "hermitian")  # 252
        u = xs  # 253: the full filtered Ritz block is the next iterate
        if not np.any(keep):  # 254-255
            continue
        found_any = True
        lam, x = w[keep], xs[:, keep]
        res = residuals(p, lam, x)  # 258
        best_res = min(best_res, float(res.max()))
        if res.max() <= cfg.tol:  # 260-261
            break
    elapsed = time.perf_counter() - t0
    if not found_any or lam is None:  # 269-272
        raise NoEigenvaluesFound("no eigenvalues inside contour")
    if res.max() > cfg.tol:  # 273-277
        conv = res <= cfg.tol
        if not np.any(conv):
            raise ConvergenceError(best_res)
        lam, x, res = lam[conv], x[:, conv], res[conv]
    order = np.argsort(lam)  # 278
    return OracleResult(lam[order], x[:, order], res[order], contour, it + 1,
                        ctx.n_linear_solves, ctx.n_factorizations, elapsed, ranks)


@dataclass
class OracleMulti:
    results: list
    errors: list
    elapsed: float

    @property
    def eigenvalues(self):
        vals = [r.eigenvalues for r in self.results if r is not None]
        return np.sort(np.concatenate(vals)) if vals else np.array([])


def solve_multi(pencil, contours, cfg: OracleConfig | None = None, seed: int = 0, solver: str = "cirr"):
    """solvers.py:312-339 (per-contour seed+i, isolated failures, dedupe)."""
    cfg = cfg or OracleConfig()
    fn = {"cirr": cirr_solve, "feast": feast_solve}[solver]  # 316-318
    t0 = time.perf_counter()
    p = Pencil.of(pencil)
    results, errors = [], []
    for i, c in enumerate(contours):
        try:
            results.append(fn(p, c, cfg, seed=seed + i))
            errors.append(None)
        except (NoEigenvaluesFound, ConvergenceError, SingularShiftError, RankZeroError) as exc:
            results.append(None)
            errors.append(exc)
    _dedupe(results)
    return OracleMulti(results, errors, time.perf_counter() - t0)


def _dedupe_complex_drops(vals_list) -> dict:
    """Complex eigenvalues (non-Hermitian pencils): a 1-D sort does not put
    near-equal complex values next to each other (conjugate pairs found by two
    overlapping contours share a real part to rounding), so match by distance.
    Candidates are visited by ascending residual (ties in input order); one is
    dropped when a value already kept from a DIFFERENT contour lies within
    1e-8 of the span, so each duplicate cluster keeps its smallest residual,
    as the reference's rule does for real values (solvers.py:342-377)."""
    vals = np.array([v[0] for v in vals_list])
    span = float(np.abs(vals[:, None] - vals[None, :]).max())
    tol = 1e-8 * max(span, 1e-300)
    order = sorted(range(len(vals_list)), key=lambda t: (vals_list[t][1], t))
    kept: list = []
    drop: dict = {}
    for idx in order:
        v, ri = vals_list[idx][0], vals_list[idx][2]
        if any(vals_list[k][2] != ri and abs(v - vals_list[k][0]) <= tol for k in kept):
            drop.setdefault(ri, set()).add(vals_list[idx][3])
        else:
            kept.append(idx)
    return drop


def _dedupe(results):  # solvers.py:342-377; span uses |.| for complex values
    allv = [(r.eigenvalues[i], r.residuals[i], ri, i)
            for ri, r in enumerate(results) if r is not None
            for i in range(len(r.eigenvalues))]
    if len(allv) < 2:
        return
    vals = np.array([v[0] for v in allv])
    if np.iscomplexobj(vals) and np.any(vals.imag != 0):
        drop = _dedupe_complex_drops(allv)
    else:
        span = abs(vals.max() - vals.min())
        tol = 1e-8 * max(span, 1e-300)
        order = np.argsort(vals)
        drop: dict = {}
        prev = order[0]
        for idx in order[1:]:
            if abs(allv[idx][0] - allv[prev][0]) <= tol and allv[idx][2] != allv[prev][2]:
                loser = idx if allv[idx][1] >= allv[prev][1] else prev
                winner = idx if loser is prev else prev
                drop.setdefault(allv[loser][2], set()).add(allv[loser][3])
                prev = winner
            else:
                prev = idx
    for ri, cols in drop.items():
        r = results[ri]
        keep = np.array([i not in cols for i in range(len(r.eigenvalues))])
        r.eigenvalues = r.eigenvalues[keep]
        r.eigenvectors = r.eigenvectors[:, keep]
        r.residuals = r.residuals[keep]
