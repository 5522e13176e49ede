"""Fixed-budget Krylov scouts on the device LU.

Mirrors the reference's scouting API (`/root/reference/pkg/src/cieig/
scouting.py`): `scout(pencil, method, k_iters, m, seed) -> RitzEstimate`
(scouting.py:153-180) with the same three methods, the same random start
vectors, budgets, stopping tests and output (the m dominant Ritz values of
A^-1 B mapped back to eigenvalues, ascending), plus `scout_contour`
(scouting.py:183-211) and `calibrate_margin` (scouting.py:214-229), which are
host arithmetic on the Ritz values.

What runs on the GPU: the one factorisation of (0*B - A) = -A (K1 + K2:
`cirr_assemble` with the single shift 0 and `cirr_zgetrf_batched`), every
application of A^-1 (K3 `cirr_zgetrs_batched`, one right-hand side), every
product with B (`cirr_gemm`, real B), the B- or Euclidean inner products and
the re-orthogonalisation (`cirr_gemm` GEMVs against the stored basis, split-K
for the long reductions), and the final small symmetric / general eigenvalue
problem (`cirr_small_eig`).  Scalar recurrences (alpha, beta, the break
tests) are read back to the host, as the reference computes them there.

Deviation: the reference re-orthogonalises with modified Gram-Schmidt over
the basis, one projection at a time (scouting.py:54-55, 82-89, 122-124).
Here each pass is classical Gram-Schmidt done as two GEMVs, and every method
takes two passes (CGS2), which is at least as stable as one MGS pass; the
Ritz values agree with the reference's to rounding (tests/test_gpu_scout.py).
"""
from __future__ import annotations

import time
import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib
from .contours import Contour
from .errors import EmptyPredictionError, ParameterError, ParameterWarning, SingularShiftError
from .solvers import PIVOT_REL_TOL, DevicePencil, _h2d, _ptr, _stream, _torch

SCOUT_METHODS = ("lanczos", "arnoldi", "krylov-schur-restarted")


@dataclass(frozen=True)
class RitzEstimate:
    method: str
    k_iters: int
    ritz_values: np.ndarray  # ascending
    elapsed: float


class _Device:
    """A^-1 and B on the device from one LU of (0*B - A) (linalg.py:55-71 at z = 0)."""

    def __init__(self, dp: DevicePencil):
        torch = _torch()
        self.torch, self.dp, self.n = torch, dp, dp.n
        n, st = self.n, _stream()
        self.fac = torch.empty((1, n, n), dtype=torch.complex128, device="cuda")
        maxabs = torch.empty(1, dtype=torch.float64, device="cuda")
        self.perm = torch.empty((1, n), dtype=torch.int32, device="cuda")
        ipiv = torch.empty((1, n), dtype=torch.int32, device="cuda")
        minpiv = torch.empty(1, dtype=torch.float64, device="cuda")
        info = torch.empty(1, dtype=torch.int32, device="cuda")
        z = _h2d(np.zeros(1, dtype=np.complex128))
        dp.assemble(z, 1, self.fac, maxabs, st)
        lws = torch.empty(int(_lib.call("cirr_zgetrf_ws_bytes", n, 1)), dtype=torch.uint8, device="cuda")
        _lib.call("cirr_zgetrf_batched", _ptr(self.fac), n, n, n * n, 1, _ptr(ipiv), _ptr(self.perm),
                  _ptr(minpiv), _ptr(info), _ptr(lws), st)
        self.dinv = torch.empty(int(_lib.call("cirr_diag_inv_bytes", n, 1)), dtype=torch.uint8, device="cuda")
        _lib.call("cirr_diag_inverses", _ptr(self.fac), n, n, n * n, 1, _ptr(self.dinv), st)
        scale = max(float(maxabs.item()), 1e-300)
        if int(info.item()) != 0 or not float(minpiv.item()) >= PIVOT_REL_TOL * scale:
            raise SingularShiftError(0j)
        self.rhs_of = _h2d(np.zeros(1, dtype=np.int32))

    def new(self, k: int = 1):
        return self.torch.zeros((self.n, k), dtype=self.torch.complex128, device="cuda")

    def inv(self, x, real: bool):
        """A^-1 x = -(0*B - A)^-1 x for an (n x 1) device vector (scouting.py:163-166)."""
        n = self.n
        y = self.new()
        _lib.call("cirr_zgetrs_batched", _ptr(self.fac), n, n, n * n, 1, _ptr(self.perm), _ptr(x), 1, n,
                  _ptr(self.rhs_of), 1, _ptr(y), 1, n, _ptr(self.dinv), _stream())
        y.neg_()
        if real:
            y.imag.zero_()
        return y

    def bmul(self, x):
        n = self.n
        out = self.new(x.shape[1])
        _lib.call("cirr_gemm", self.dp.gemm_kind, n, x.shape[1], n, 1, _ptr(self.dp.b), n, 0, _ptr(x), x.shape[1], 0,
                  _ptr(out),
                  x.shape[1], 0, 1.0, 0, _stream())
        return out

    def dots(self, Ut, j: int, w):
        """h[i] = vdot(Ut[i], w) for the first j rows of Ut ((cap x n) rows), w (n x 1)."""
        h = self.torch.empty((j, 1), dtype=self.torch.complex128, device="cuda")
        _lib.call("cirr_gemm", 1, j, 1, self.n, 1, _ptr(Ut), self.n, 0, _ptr(w), 1, 0, _ptr(h), 1, 0, 1.0, 0,
                  _stream())
        return h

    def sub_comb(self, w, Qt, j: int, h):
        """w -= sum_i h[i] Qt[i] (rows 0..j-1) as the GEMV w^T -= h^T Qt."""
        _lib.call("cirr_gemm", 0, 1, self.n, j, 1, _ptr(h), j, 0, _ptr(Qt), self.n, 0, _ptr(w), self.n, 0, -1.0, 1,
                  _stream())

    def vdot(self, u, w) -> complex:
        """vdot(u, w) for (n x 1) device vectors (split-K GEMV, read back)."""
        return complex(self.dots(u, 1, w).item())

    def small_eigvals(self, h: np.ndarray, hermitian: bool) -> np.ndarray:
        """Eigenvalues of a small k x k matrix on the device (cirr_small_eig with B = I)."""
        torch = self.torch
        k = h.shape[0]
        if k == 0:
            return np.zeros(0)
        At = _h2d(np.ascontiguousarray(h, dtype=np.complex128)[None])
        Bt = _h2d(np.eye(k, dtype=np.complex128)[None])
        kd = _h2d(np.array([k], dtype=np.int32))
        wsb = int(_lib.call("cirr_small_eig_ws_bytes", k))
        ws = torch.empty((wsb + 255) // 256 * 256, dtype=torch.uint8, device="cuda")
        lam = torch.zeros((1, k), dtype=torch.complex128, device="cuda")
        S = torch.zeros((1, k, k), dtype=torch.complex128, device="cuda")
        info = torch.zeros(1, dtype=torch.int32, device="cuda")
        _lib.call("cirr_small_eig", 1 if hermitian else 0, _ptr(At), _ptr(Bt), k, k * k, _ptr(kd), k, 1, _ptr(ws),
                  _ptr(lam), _ptr(S), k, k * k, _ptr(info), _stream())
        if int(info.item()) != 0:
            raise RuntimeError(f"small eigensolver failed (info {int(info.item())})")
        out = lam.cpu().numpy()[0]
        return out.real.copy() if hermitian else out


def _cgs2(d: _Device, w, Qt, Ut, j: int, hacc=None):
    """Two classical Gram-Schmidt passes of w against rows 0..j-1 of Qt, with
    coefficients vdot(Ut[i], w) (Ut = B Q for the B-inner product, Ut = Q for the
    Euclidean one).  hacc (j x 1) accumulates the coefficients when given."""
    for _ in range(2):
        h = d.dots(Ut, j, w)
        d.sub_comb(w, Qt, j, h)
        if hacc is not None:
            hacc += h


def _lanczos(d: _Device, k: int, rng) -> np.ndarray:
    """B-inner-product Lanczos with full re-orthogonalisation (scouting.py:37-70)."""
    torch, n = d.torch, d.n
    kk = min(k, n)
    Qt = torch.zeros((kk + 1, n), dtype=torch.complex128, device="cuda")    # basis rows
    BQt = torch.zeros_like(Qt)                                            # B basis rows
    v = torch.from_numpy(rng.standard_normal(n).astype(complex)).to("cuda")[:, None]
    bv = d.bmul(v)
    v /= np.sqrt(d.vdot(v, bv).real)
    Qt[0].copy_(v[:, 0])
    BQt[0].copy_(d.bmul(v)[:, 0])
    alphas, betas = [], []
    j = 1
    for _ in range(kk):
        w = d.inv(BQt[j - 1][:, None].clone(), real=True)
        alpha = float(d.dots(BQt[j - 1:j], 1, w).real.item())
        alphas.append(alpha)
        w -= alpha * Qt[j - 1][:, None]
        if j > 1:
            w -= betas[-1] * Qt[j - 2][:, None]
        _cgs2(d, w, Qt, BQt, j)
        bw = d.bmul(w)
        beta = float(np.sqrt(max(d.vdot(w, bw).real, 0.0)))
        if beta < 1e-14:
            break
        betas.append(beta)
        Qt[j].copy_(w[:, 0] / beta)
        BQt[j].copy_(bw[:, 0] / beta)
        j += 1
    t = np.diag(np.array(alphas))
    if betas:
        off = np.array(betas[: len(alphas) - 1])
        t += np.diag(off, 1) + np.diag(off, -1)
    return d.small_eigvals(t, hermitian=True)


def _arnoldi(d: _Device, k: int, rng) -> np.ndarray:
    """Euclidean Arnoldi on A^-1 B (scouting.py:73-98); complex Ritz values."""
    torch, n = d.torch, d.n
    kk = min(k, n)
    Qt = torch.zeros((kk + 1, n), dtype=torch.complex128, device="cuda")
    v = torch.from_numpy(rng.standard_normal(n).astype(complex)).to("cuda")[:, None]
    v /= np.sqrt(d.vdot(v, v).real)
    Qt[0].copy_(v[:, 0])
    h = np.zeros((kk + 1, kk), dtype=complex)
    steps = 0
    for j in range(kk):
        w = d.inv(d.bmul(Qt[j][:, None].clone()), real=False)
        hj = torch.zeros((j + 1, 1), dtype=torch.complex128, device="cuda")
        _cgs2(d, w, Qt, Qt, j + 1, hacc=hj)
        h[: j + 1, j] = hj.cpu().numpy()[:, 0]
        steps = j + 1
        nrm = float(np.sqrt(d.vdot(w, w).real))
        h[j + 1, j] = nrm
        if nrm < 1e-14:
            break
        Qt[j + 1].copy_(w[:, 0] / nrm)
    return d.small_eigvals(h[:steps, :steps], hermitian=False)


def _thick_restart(d: _Device, k: int, m: int, rng) -> np.ndarray:
    """Thick-restart Lanczos with the basis capped at 2m (scouting.py:101-150):
    k operator applications; images op(B q) are kept and rotated with the
    basis at each restart, so no extra solves are needed."""
    torch, n = d.torch, d.n
    cap = min(max(2 * m, 4), n)
    rows = cap + 1
    Vt = torch.zeros((rows, n), dtype=torch.complex128, device="cuda")    # basis rows
    BVt = torch.zeros_like(Vt)                                          # B basis rows
    Wt = torch.zeros_like(Vt)                                           # images op(B basis)
    v = torch.from_numpy(rng.standard_normal(n).astype(complex)).to("cuda")[:, None]
    v /= np.sqrt(d.vdot(v, d.bmul(v)).real)
    Vt[0].copy_(v[:, 0])
    BVt[0].copy_(d.bmul(v)[:, 0])
    nb, ni = 1, 0          # basis vectors, images

    def projected(cnt):
        # Re(V^T B W), symmetrised; V^T B W = (B V)^T W with B symmetric, as rows: conj(BVt) . Wt^T
        hm = torch.empty((cnt, cnt), dtype=torch.complex128, device="cuda")
        WT = Wt[:cnt].transpose(0, 1).contiguous()
        _lib.call("cirr_gemm", 1, cnt, cnt, n, 1, _ptr(BVt), n, 0, _ptr(WT), cnt, 0, _ptr(hm), cnt, 0, 1.0, 0,
                  _stream())
        h = hm.cpu().numpy().real
        return 0.5 * (h + h.T)

    def small_eigh(h):
        """Ascending eigenvalues and eigenvectors of a small real symmetric matrix (device)."""
        kk = h.shape[0]
        At = _h2d(np.ascontiguousarray(h, dtype=np.complex128)[None])
        Bt = _h2d(np.eye(kk, dtype=np.complex128)[None])
        kd = _h2d(np.array([kk], dtype=np.int32))
        wsb = int(_lib.call("cirr_small_eig_ws_bytes", kk))
        ws = torch.empty((wsb + 255) // 256 * 256, dtype=torch.uint8, device="cuda")
        lam = torch.zeros((1, kk), dtype=torch.complex128, device="cuda")
        S = torch.zeros((1, kk, kk), dtype=torch.complex128, device="cuda")
        info = torch.zeros(1, dtype=torch.int32, device="cuda")
        _lib.call("cirr_small_eig", 1, _ptr(At), _ptr(Bt), kk, kk * kk, _ptr(kd), kk, 1, _ptr(ws), _ptr(lam),
                  _ptr(S), kk, kk * kk, _ptr(info), _stream())
        # the eigenvectors of a real symmetric matrix are real up to a phase per
        # column: remove it (largest-modulus entry real positive), keep real parts
        s = S[0].cpu().numpy()
        piv = np.argmax(np.abs(s), axis=0)
        ph = s[piv, np.arange(kk)]
        s = (s * (np.abs(ph) / ph)[None, :]).real
        return lam.cpu().numpy()[0].real, s

    applied, budget = 0, min(k, n)
    while applied < budget:
        w = d.inv(d.bmul(Vt[nb - 1][:, None].clone()), real=True)
        applied += 1
        Wt[ni].copy_(w[:, 0])
        ni += 1
        w_orth = w.clone()
        # two passes of Re(<B q, w>) projections (the reference's 2 x MGS)
        for _ in range(2):
            hcoef = d.dots(BVt, nb, w_orth)
            hcoef.imag.zero_()
            d.sub_comb(w_orth, Vt, nb, hcoef)
        bwo = d.bmul(w_orth)
        beta = float(np.sqrt(max(d.vdot(w_orth, bwo).real, 0.0)))
        if beta < 1e-12 * float(np.sqrt(d.vdot(w, w).real)):
            break  # invariant subspace reached
        w_orth /= beta
        bwo /= beta
        if nb >= cap:
            h = projected(ni)
            theta, s = small_eigh(h)
            order = np.argsort(-np.abs(theta), kind="stable")[:m]
            # kept rows: (V s)^T = s^T V^T, as rows: sel^T (m x ni) . Vt (ni x n)
            selT = _h2d(np.ascontiguousarray(s[:, order].T, dtype=np.complex128))
            newV = torch.empty((m, n), dtype=torch.complex128, device="cuda")
            newW = torch.empty_like(newV)
            newBV = torch.empty_like(newV)
            for src, dst in ((Vt, newV), (Wt, newW), (BVt, newBV)):
                _lib.call("cirr_gemm", 0, m, n, ni, 1, _ptr(selT), ni, 0, _ptr(src), n, 0, _ptr(dst), n, 0, 1.0, 0,
                          _stream())
            Vt.zero_(); Wt.zero_(); BVt.zero_()
            Vt[:m].copy_(newV); Wt[:m].copy_(newW); BVt[:m].copy_(newBV)
            Vt[m].copy_(w_orth[:, 0]); BVt[m].copy_(bwo[:, 0])
            nb, ni = m + 1, m
        else:
            Vt[nb].copy_(w_orth[:, 0])
            BVt[nb].copy_(bwo[:, 0])
            nb += 1
    h = projected(ni)
    return d.small_eigvals(h, hermitian=True)


def scout(pencil, method: str, k_iters: int, m: int, seed: int) -> RitzEstimate:
    """Fixed-budget Krylov scout for the m smallest-magnitude eigenvalues
    (scouting.py:153-180) on the device LU.  `pencil` is a reference
    MatrixPencil, a DevicePencil or an (A, B) pair."""
    if method not in SCOUT_METHODS:
        raise ParameterError(f"unknown scout method {method!r}")
    if k_iters < m:
        raise ParameterError("k_iters must be >= m")
    t0 = time.perf_counter()
    if isinstance(pencil, DevicePencil):
        dp = pencil
    elif isinstance(pencil, tuple):
        dp = DevicePencil(*pencil)
    else:
        dp = DevicePencil(pencil.a, pencil.b, hermitian=getattr(pencil, "hermitian", None) or None)
    d = _Device(dp)
    rng = np.random.default_rng(seed)
    if method == "lanczos":
        theta = _lanczos(d, k_iters, rng)
    elif method == "arnoldi":
        theta = np.real(_arnoldi(d, k_iters, rng))
    else:
        theta = _thick_restart(d, k_iters, m, rng)
    theta = theta[np.abs(theta) > 1e-300]
    order = np.argsort(-np.abs(theta), kind="stable")[:m]
    lam = np.sort(1.0 / theta[order])
    return RitzEstimate(method=method, k_iters=k_iters, ritz_values=lam, elapsed=time.perf_counter() - t0)


def scout_contour(ritz: RitzEstimate, margin_factor: float = 1.2) -> Contour:
    """Margin-expanded bounding rectangle around the Ritz values
    (scouting.py:183-211): the real span widened by (margin_factor - 1)/2 of
    its width on each side, and a height of a fifth of the widened width
    (aspect 5, the largest a rect contour allows)."""
    if margin_factor < 1.0:
        raise ParameterError("margin_factor must be >= 1")
    vals = np.asarray(ritz.ritz_values, dtype=float)
    if vals.size == 0:
        raise EmptyPredictionError("empty Ritz estimate")
    lo, hi = float(vals.min()), float(vals.max())
    width = hi - lo
    if width <= 0.0:
        width = 1e-6 * max(abs(lo), 1e-300)
        warnings.warn("degenerate Ritz span; using minimum width", ParameterWarning)
        lo, hi = lo - 0.5 * width, hi + 0.5 * width
    grow = 0.5 * (margin_factor - 1.0) * width
    re_min, re_max = lo - grow, hi + grow
    half_h = (re_max - re_min) / 10.0
    return Contour(shape="rect", re_min=re_min, re_max=re_max, im_min=-half_h, im_max=half_h,
                   expected_count=len(vals), source="scout")


def calibrate_margin(ritz: RitzEstimate, truth, step: float = 0.01) -> float:
    """Smallest margin factor 1 + i*step whose scout rectangle contains every
    ground-truth eigenvalue (scouting.py:214-229)."""
    if step <= 0:
        raise ParameterError("step must be positive")
    eigs = np.asarray(truth.eigenvalues, dtype=float)
    i = 0
    while True:
        mf = 1.0 + i * step
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", ParameterWarning)
            c = scout_contour(ritz, mf)
        if eigs.min() >= c.re_min and eigs.max() <= c.re_max:
            return mf
        i += 1
