"""Complex-valued pencils (the reference's MatrixPencil holds complex128 CSR
values, sparse.py:14-43) on the device path, against the
CPU oracle run on the same pencil, contour and seed: exact in-contour count,
eigenvalues to 1e-8, residuals <= 1e-10."""
import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle import cirr as O  # noqa: E402  (test-side checker only)


def _match(a, b):
    a, b = np.sort_complex(np.asarray(a, complex)), np.sort_complex(np.asarray(b, complex))
    return np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)) if len(a) else 0.0


def _run(a, b, contour, L, M, herm):
    from paper_2511_01927_b200 import DevicePencil, SolverConfig, solve_multi
    dp = DevicePencil(a, b)
    assert dp.complex and dp.hermitian == herm
    m = solve_multi(dp, [contour], SolverConfig(n_q=32, source_cols=L, n_moments=M, tol=1e-10), seed=0)
    r = m.results[0]
    o = O.cirr_solve(O.Pencil(a, b), contour, O.OracleConfig(n_q=32, source_cols=L, n_moments=M, tol=1e-10), seed=0)
    return r, o


def test_complex_hermitian_pencil():
    from paper_2511_01927_b200 import Contour
    n = 300
    rng = np.random.default_rng(3)
    g = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    a = (g + g.conj().T) / (2 * np.sqrt(n)) + np.diag(np.linspace(0.0, 10.0, n))
    h = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    b = np.eye(n) + 0.1 * (h @ h.conj().T) / n
    w = sla.eigh(a, b, eigvals_only=True)
    lo, hi = 0.5 * (w[39] + w[40]), 0.5 * (w[51] + w[52])
    c = Contour(shape="circle", center=complex(0.5 * (lo + hi), 0.0), radius=0.5 * (hi - lo), expected_count=12)
    r, o = _run(a, b, c, 24, 4, True)
    assert len(r.eigenvalues) == len(o.eigenvalues) == 12
    assert _match(r.eigenvalues, o.eigenvalues) <= 1e-8
    assert _match(r.eigenvalues, w[40:52]) <= 1e-8
    assert r.residuals.max() <= 1e-10
    x = r.eigenvectors
    res = np.linalg.norm(a @ x - (b @ x) * r.eigenvalues[None, :], axis=0) / (
        np.linalg.norm(a @ x, axis=0) + np.abs(r.eigenvalues) * np.linalg.norm(b @ x, axis=0))
    assert np.allclose(res, r.residuals, rtol=1e-6, atol=1e-15)


def test_complex_general_pencil_and_csr_input():
    from paper_2511_01927_b200 import Contour
    n = 300
    rng = np.random.default_rng(4)
    a = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(2 * n) + np.diag(
        rng.uniform(-2.0, 2.0, n) + 0.3j * rng.uniform(-1.0, 1.0, n))
    b = np.eye(n) + 0.05 * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(n)
    w = sla.eig(a, b, right=False)
    c = Contour(shape="ellipse", center=0.5 + 0.05j, semi_re=0.4, semi_im=0.25)
    q = ((w.real - 0.5) / 0.4) ** 2 + ((w.imag - 0.05) / 0.25) ** 2
    truth = w[q < 1]
    assert np.min(np.abs(q - 1)) > 1e-3 and len(truth) >= 4
    c = Contour(shape="ellipse", center=0.5 + 0.05j, semi_re=0.4, semi_im=0.25, expected_count=len(truth))
    r, o = _run(sp.csr_matrix(a), sp.csr_matrix(b), c, 2 * len(truth) + 8, 4, False)
    assert len(r.eigenvalues) == len(o.eigenvalues) == len(truth)
    assert _match(r.eigenvalues, o.eigenvalues) <= 1e-8
    assert _match(r.eigenvalues, truth) <= 1e-8
    assert r.residuals.max() <= 1e-10


def test_complex_kernels():
    """cirr_assemble_c equals numpy's z*B - A to rounding; cirr_hermitian_c."""
    from paper_2511_01927_b200 import _lib
    n = 77
    rng = np.random.default_rng(5)
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    b = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    z = np.array([0.3 + 0.7j, -1.1 + 0.2j, 2.0 - 0.5j])
    A, B, Z = (torch.from_numpy(m).cuda() for m in (a, b, z))
    P = torch.empty((3, n, n), dtype=torch.complex128, device="cuda")
    mx = torch.empty(3, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    assert _lib.call("cirr_assemble_c", A.data_ptr(), B.data_ptr(), n, n, Z.data_ptr(), 3, P.data_ptr(), n, n * n,
                     mx.data_ptr(), st) == 0
    ref = z[:, None, None] * b[None] - a[None]
    got = P.cpu().numpy()
    assert np.abs(got - ref).max() <= 4e-16 * np.abs(ref).max()     # complex product: rounded products and sums
    assert np.allclose(mx.cpu().numpy(), np.abs(ref).reshape(3, -1).max(axis=1), rtol=1e-15)
    hm = (a + a.conj().T) / 2
    hm[3, 5] += 1e-9
    H = torch.from_numpy(hm).cuda()
    out = torch.empty(2, dtype=torch.float64, device="cuda")
    assert _lib.call("cirr_hermitian_c", H.data_ptr(), n, n, out.data_ptr(), st) == 0
    o = out.cpu().numpy()
    assert o[0] == pytest.approx(np.abs(hm - hm.conj().T).max(), rel=1e-12)
    assert o[1] == pytest.approx(np.abs(hm).max(), rel=1e-15)


def test_wide_moment_block_default_source_cols():
    """A contour expecting 100 eigenvalues with the reference's default
    source_cols (max(8, 2 * expected) = 200, solvers.py:41-44) and M = 4: the
    moment block is 800 columns wide (K4 with smaller Jacobi blocks)."""
    from paper_2511_01927_b200 import Contour, DevicePencil, SolverConfig, solve_multi
    n = 1200
    a = 2.0 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    b = np.eye(n)
    w = 2.0 - 2.0 * np.cos(np.arange(1, n + 1) * np.pi / (n + 1))
    lo, hi = 0.5 * (w[199] + w[200]), 0.5 * (w[299] + w[300])
    c = Contour(shape="circle", center=complex(0.5 * (lo + hi), 0.0), radius=0.5 * (hi - lo), expected_count=100)
    cfg = SolverConfig(n_q=32, n_moments=4, tol=1e-10)
    assert cfg.cols_for(100) == 200
    m = solve_multi(DevicePencil(a, b), [c], cfg, seed=0)
    r = m.results[0]
    assert r is not None and len(r.eigenvalues) == 100
    assert _match(r.eigenvalues, w[200:300]) <= 1e-8
    assert r.residuals.max() <= 1e-10


def test_conjugate_pair_variant_off_for_complex_pencils():
    """M(conj z) = conj(M(z)) needs real A and B: with complex values the
    labelled conjugate-pair variant must factor every node (same result)."""
    from paper_2511_01927_b200 import Contour, DevicePencil, SolverConfig, solve_multi
    n = 200
    rng = np.random.default_rng(6)
    g = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    a = (g + g.conj().T) / (2 * np.sqrt(n)) + np.diag(np.linspace(0.0, 5.0, n))
    b = np.eye(n)
    w = np.linalg.eigvalsh(a)
    lo, hi = 0.5 * (w[19] + w[20]), 0.5 * (w[29] + w[30])
    c = Contour(shape="circle", center=complex(0.5 * (lo + hi), 0.0), radius=0.5 * (hi - lo), expected_count=10)
    dp = DevicePencil(a, b)
    base = solve_multi(dp, [c], SolverConfig(n_q=32, source_cols=20, n_moments=4), seed=0)
    var = solve_multi(dp, [c], SolverConfig(n_q=32, source_cols=20, n_moments=4, conjugate_pairs=True), seed=0)
    assert var.results[0].stats.n_factorizations == 32 == base.results[0].stats.n_factorizations
    assert np.array_equal(var.eigenvalues, base.eigenvalues)
    assert _match(base.eigenvalues, w[20:30]) <= 1e-8
