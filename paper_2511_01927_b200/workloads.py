"""Seeded synthetic inputs for the five BASELINE.json configs.

BASELINE.json names no public dataset; these generators *are* the
measurement set.  Every draw comes from ``numpy.random.default_rng`` with the
seeding scheme recorded in each docstring.  A and B are returned dense and
real (float64).  Contour placement needs eigenvalues of the pencil; helper
``place_contours`` takes them as input (computed by the caller, e.g. the
golden-fixture script, with a dense host eigensolver).

``grf_2d`` restates the reference's log-normal spectral GRF
(cieig/problems.py:98-127) so config 2/3 fields match it bit-for-bit
(pinned in tests/test_workloads.py against a reference-generated fixture);
``grf_3d`` is the same synthesis in 3-D for config 5.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .contours import Contour


@dataclass
class Workload:
    name: str
    a: np.ndarray
    b: np.ndarray
    contours: list = field(default_factory=list)
    n_q: int = 32
    source_cols: int = 16
    n_moments: int = 4
    hermitian: bool = True
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return self.a.shape[0]


# ---------------------------------------------------------------------------
# random fields


def grf_2d(nx: int, ny: int, mean: float, variance: float, length_scale: float, seed: int):
    """Log-normal field on the interior nodes, row-major y-then-x
    (problems.py:98-127: 2x padded periodic spectral synthesis)."""
    if variance == 0.0:
        return np.full(nx * ny, float(mean))
    rng = np.random.default_rng(seed)
    hx, hy = 1.0 / (nx + 1), 1.0 / (ny + 1)
    npx, npy = 2 * (nx + 1), 2 * (ny + 1)
    kx = 2.0 * np.pi * np.fft.fftfreq(npx, d=hx)
    ky = 2.0 * np.pi * np.fft.fftfreq(npy, d=hy)
    k2 = kx[None, :] ** 2 + ky[:, None] ** 2
    amp = np.exp(-0.25 * length_scale**2 * k2)
    noise = rng.standard_normal((npy, npx)) + 1j * rng.standard_normal((npy, npx))
    g = np.real(np.fft.ifft2(noise * amp))
    g *= np.sqrt(variance) * (npx * npy) / np.linalg.norm(amp)
    g = g[1:ny + 1, 1:nx + 1]
    return mean * np.exp(g).ravel()


def grf_3d(nx: int, mean: float, variance: float, length_scale: float, rng):
    """3-D analogue of grf_2d on an nx^3 interior grid (z-then-y-then-x order)."""
    h = 1.0 / (nx + 1)
    npd = 2 * (nx + 1)
    k = 2.0 * np.pi * np.fft.fftfreq(npd, d=h)
    k2 = k[:, None, None] ** 2 + k[None, :, None] ** 2 + k[None, None, :] ** 2
    amp = np.exp(-0.25 * length_scale**2 * k2)
    noise = rng.standard_normal((npd,) * 3) + 1j * rng.standard_normal((npd,) * 3)
    g = np.real(np.fft.ifftn(noise * amp))
    g *= np.sqrt(variance) * (npd**3) / np.linalg.norm(amp)
    g = g[1:nx + 1, 1:nx + 1, 1:nx + 1]
    return mean * np.exp(g).ravel()


# ---------------------------------------------------------------------------
# operators


def fd_operator_2d(a_field: np.ndarray, nx: int, ny: int) -> np.ndarray:
    """5-point -div(a grad u), FV scaling (no 1/h^2), Dirichlet boundary.

    Interior faces use the arithmetic mean (a_i + a_j)/2; a face to the
    boundary uses the interior node's own value a_i.
    """
    n = nx * ny
    a = a_field.reshape(ny, nx)
    m = np.zeros((n, n))
    idx = np.arange(n).reshape(ny, nx)
    diag = np.zeros((ny, nx))
    # x-faces
    fx = 0.5 * (a[:, 1:] + a[:, :-1])
    diag[:, 1:] += fx
    diag[:, :-1] += fx
    m[idx[:, 1:].ravel(), idx[:, :-1].ravel()] = -fx.ravel()
    m[idx[:, :-1].ravel(), idx[:, 1:].ravel()] = -fx.ravel()
    # y-faces
    fy = 0.5 * (a[1:, :] + a[:-1, :])
    diag[1:, :] += fy
    diag[:-1, :] += fy
    m[idx[1:, :].ravel(), idx[:-1, :].ravel()] = -fy.ravel()
    m[idx[:-1, :].ravel(), idx[1:, :].ravel()] = -fy.ravel()
    # boundary faces
    diag[:, 0] += a[:, 0]
    diag[:, -1] += a[:, -1]
    diag[0, :] += a[0, :]
    diag[-1, :] += a[-1, :]
    m[idx.ravel(), idx.ravel()] = diag.ravel()
    return m


def fd_operator_3d(e_field: np.ndarray, nx: int, h: float):
    """7-point -div(E grad u), FV scaling (face area h^2 / distance h = h)."""
    n = nx**3
    e = e_field.reshape(nx, nx, nx)
    idx = np.arange(n).reshape(nx, nx, nx)
    a = np.zeros((n, n))
    diag = np.zeros((nx, nx, nx))
    pairs = []
    for ax in range(3):
        sl_hi = [slice(None)] * 3
        sl_lo = [slice(None)] * 3
        sl_hi[ax] = slice(1, None)
        sl_lo[ax] = slice(None, -1)
        f = 0.5 * (e[tuple(sl_hi)] + e[tuple(sl_lo)])
        diag[tuple(sl_hi)] += f
        diag[tuple(sl_lo)] += f
        i, j = idx[tuple(sl_hi)].ravel(), idx[tuple(sl_lo)].ravel()
        a[i, j] = -h * f.ravel()
        a[j, i] = -h * f.ravel()
        pairs.append((i, j))
        first = [slice(None)] * 3
        last = [slice(None)] * 3
        first[ax] = 0
        last[ax] = -1
        diag[tuple(first)] += e[tuple(first)]
        diag[tuple(last)] += e[tuple(last)]
    a[idx.ravel(), idx.ravel()] = h * diag.ravel()
    return a, pairs


# ---------------------------------------------------------------------------
# contour placement


def cut_point(eigs: np.ndarray, i: int) -> float:
    """Midpoint between the i-th and (i+1)-th smallest eigenvalues (1-based i)."""
    return 0.5 * (eigs[i - 1] + eigs[i])


def largest_gap_cut(eigs: np.ndarray, i: int, window: int = 2) -> int:
    """Move a nominal cut after index i (1-based) to the largest relative gap
    (l_{k+1}-l_k)/|l_{k+1}+l_k| within +-window indices."""
    best, best_k = -1.0, i
    for k in range(max(1, i - window), min(len(eigs) - 1, i + window) + 1):
        g = (eigs[k] - eigs[k - 1]) / abs(eigs[k] + eigs[k - 1])
        if g > best:
            best, best_k = g, k
    return best_k


def circles_between_cuts(eigs: np.ndarray, cuts: list[int], source: str = "manual"):
    """One circle per consecutive pair of cuts; cut k sits between l_k and l_{k+1}."""
    out = []
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        left, right = cut_point(eigs, lo), cut_point(eigs, hi)
        out.append(Contour(shape="circle", center=complex(0.5 * (left + right), 0.0),
                           radius=0.5 * (right - left), expected_count=hi - lo, source=source))
    return out


def sorted_real_eigs(a: np.ndarray, b: np.ndarray, upto: int | None = None) -> np.ndarray:
    import scipy.linalg as sla
    if upto is None:
        return np.sort(sla.eigh(a, b, eigvals_only=True))
    return np.sort(sla.eigh(a, b, eigvals_only=True, subset_by_index=[0, upto - 1]))


# ---------------------------------------------------------------------------
# the five configs


def config1_matrices(seed: int = 0, n: int = 512):
    """1-D P1-FEM Sturm-Liouville: h = 1/(n+1), n+1 elements; p_e ~ U[1,2] then
    q_e ~ U[0,10] from one default_rng(seed).  A = sum_e p_e/h [[1,-1],[-1,1]]
    + q_e h/6 [[2,1],[1,2]] (consistent q-term) on interior nodes; B =
    (h/6) tridiag(1,4,1)."""
    ne = n + 1
    h = 1.0 / ne
    rng = np.random.default_rng(seed)
    p = rng.uniform(1.0, 2.0, ne)
    q = rng.uniform(0.0, 10.0, ne)
    full = np.zeros((n + 2, n + 2))
    for e in range(ne):
        ke = p[e] / h * np.array([[1.0, -1.0], [-1.0, 1.0]]) + q[e] * h / 6.0 * np.array([[2.0, 1.0], [1.0, 2.0]])
        full[e:e + 2, e:e + 2] += ke
    a = full[1:-1, 1:-1].copy()
    b = (h / 6.0) * (4.0 * np.eye(n) + np.eye(n, k=1) + np.eye(n, k=-1))
    return a, b


def config1(seed: int = 0, eigs=None) -> Workload:
    a, b = config1_matrices(seed)
    if eigs is None:
        eigs = sorted_real_eigs(a, b, upto=80)
    left, right = cut_point(eigs, 39), cut_point(eigs, 72)  # encloses l_40..l_72
    c = Contour(shape="circle", center=complex(0.5 * (left + right), 0.0),
                radius=0.5 * (right - left), expected_count=33)
    return Workload("config1-sturm-liouville-n512", a, b, [c], n_q=32, source_cols=16,
                    n_moments=4, hermitian=True, meta={"seed": seed})


def config2_matrices(s: int, nx: int = 16):
    """GEP s of the batch: a = exp(GRF(len 0.2, var 0.5, seed s)); c ~ U[0.5,1.5]
    from default_rng(10000 + s); B = diag(h^2 c)."""
    h = 1.0 / (nx + 1)
    a_field = grf_2d(nx, nx, 1.0, 0.5, 0.2, s)
    a = fd_operator_2d(a_field, nx, nx)
    c = np.random.default_rng(10000 + s).uniform(0.5, 1.5, nx * nx)
    b = np.diag(h * h * c)
    return a, b


def config2_gep(s: int, eigs=None) -> Workload:
    a, b = config2_matrices(s)
    if eigs is None:
        eigs = sorted_real_eigs(a, b, upto=48)
    cuts = [largest_gap_cut(eigs, i) for i in (4, 16, 28)]
    return Workload(f"config2-gep{s}", a, b, circles_between_cuts(eigs, cuts), n_q=16,
                    source_cols=8, n_moments=4, hermitian=True, meta={"seed": s, "cuts": cuts})


def config3_matrices(seed: int = 0, nx: int = 48):
    """a from GRF seed `seed`; k ~ U[0,50] then c ~ U[0.5,1.5] from
    default_rng(20000 + seed); A = FD(a) + diag(h^2 k); B = diag(h^2 c)."""
    h = 1.0 / (nx + 1)
    a_field = grf_2d(nx, nx, 1.0, 0.5, 0.2, seed)
    a = fd_operator_2d(a_field, nx, nx)
    rng = np.random.default_rng(20000 + seed)
    kk = rng.uniform(0.0, 50.0, nx * nx)
    c = rng.uniform(0.5, 1.5, nx * nx)
    a[np.arange(nx * nx), np.arange(nx * nx)] += h * h * kk
    b = np.diag(h * h * c)
    return a, b


def config3(seed: int = 0, eigs=None) -> Workload:
    a, b = config3_matrices(seed)
    if eigs is None:
        eigs = sorted_real_eigs(a, b, upto=200)
    cuts = [99, 131, 163, 195]  # l_100..l_131 | l_132..l_163 | l_164..l_195
    return Workload("config3-helmholtz-48x48", a, b, circles_between_cuts(eigs, cuts), n_q=32,
                    source_cols=32, n_moments=4, hermitian=True, meta={"seed": seed})


def config4_matrices(seed: int = 0, n: int = 4096):
    """default_rng(seed): G ~ N(0,1) (n x n), d ~ U[-2,2], H ~ N(0,1);
    A = G/sqrt(n) + diag(d), B = I + 0.05 H/sqrt(n)."""
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((n, n))
    d = rng.uniform(-2.0, 2.0, n)
    hh = rng.standard_normal((n, n))
    s = 1.0 / np.sqrt(n)
    a = g * s
    a[np.arange(n), np.arange(n)] += d
    b = hh * (0.05 * s)
    b[np.arange(n), np.arange(n)] += 1.0
    return a, b


def config4(seed: int = 0, n: int = 4096, expected=(118, 110)) -> Workload:
    a, b = config4_matrices(seed, n)
    cs = [Contour(shape="ellipse", center=complex(0.5, 0.0), semi_re=0.3, semi_im=0.15,
                  expected_count=expected[0]),
          Contour(shape="ellipse", center=complex(-0.5, 0.0), semi_re=0.3, semi_im=0.15,
                  expected_count=expected[1])]
    return Workload(f"config4-dense-nonhermitian-n{n}", a, b, cs, n_q=64, source_cols=32,
                    n_moments=8, hermitian=False, meta={"seed": seed})


def config5_matrices(seed: int = 0, nx: int = 20):
    """default_rng(seed): 3-D GRF noise (len 0.25, var 0.5) then rho ~ U[0.8,1.2].
    A = 7-point FV -div(E grad u); B: diag 0.5 h^3 rho_i, neighbour entries
    h^3 (rho_i + rho_j)/24 (symmetrised, SURVEY.md section 0 finding 4)."""
    h = 1.0 / (nx + 1)
    rng = np.random.default_rng(seed)
    e = grf_3d(nx, 1.0, 0.5, 0.25, rng)
    rho = rng.uniform(0.8, 1.2, nx**3)
    a, pairs = fd_operator_3d(e, nx, h)
    n = nx**3
    b = np.zeros((n, n))
    b[np.arange(n), np.arange(n)] = 0.5 * h**3 * rho
    for i, j in pairs:
        v = h**3 * (rho[i] + rho[j]) / 24.0
        b[i, j] = v
        b[j, i] = v
    return a, b


def config5(seed: int = 0, eigs=None) -> Workload:
    a, b = config5_matrices(seed)
    if eigs is None:
        eigs = sorted_real_eigs(a, b, upto=460)
    cuts = [199, 263, 327, 391, 455]  # four groups of 64: l_200..l_455
    return Workload("config5-3d-20x20x20", a, b, circles_between_cuts(eigs, cuts), n_q=32,
                    source_cols=64, n_moments=4, hermitian=True, meta={"seed": seed})
