"""The int8 tensor-core (Ozaki splitting) GEMM update against numpy: the error
must stay at the FP64 GEMM level relative to rowmax(A) * colmax(B), also for
badly scaled rows and columns, ragged shapes and sub-blocks of larger arrays."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.fail("gpu test without CUDA")
    from paper_2511_01927_b200 import _lib
    return _lib


def S():
    return torch.cuda.current_stream().cuda_stream


def crandn(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def bound(A, B):
    """|error_ij| <= K * 2^-50 * rowmax_i(A) * colmax_j(B) (3 bits of slack on the 2^-53 per-term bound)."""
    K = A.shape[-1]
    ra = np.maximum(np.abs(A.real), np.abs(A.imag)).max(axis=-1)
    cb = np.maximum(np.abs(B.real), np.abs(B.imag)).max(axis=-2)
    return K * 2.0 ** -50 * ra[..., :, None] * cb[..., None, :]


@pytest.mark.parametrize("shape", [(128, 32, 32), (256, 64, 512), (200, 45, 96), (1000, 333, 512), (130, 1, 64),
                                   (256, 40, 1024), (384, 70, 4096)])
def test_ozaki_matches_numpy(lib, shape):
    M, N, K = shape
    rng = np.random.default_rng(M + N + K)
    batch = 3
    A = crandn(rng, batch, M, K)
    B = crandn(rng, batch, K, N)
    C0 = crandn(rng, batch, M, N)
    C = torch.from_numpy(C0.copy()).cuda()
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    rc = lib.call("cirr_ozaki_zgemm_sub", dA.data_ptr(), K, M * K, dB.data_ptr(), N, K * N, C.data_ptr(), N, M * N,
                  M, N, K, batch, S())
    assert rc == 0
    torch.cuda.synchronize()
    ref = C0 - A @ B
    err = np.abs(C.cpu().numpy() - ref)
    assert (err <= bound(A, B) + 4e-16 * np.abs(ref)).all(), err.max()


def test_ozaki_graded_rows_and_columns(lib):
    """Rows of A and columns of B spanning 60 orders of magnitude keep their own relative accuracy."""
    M, N, K = 256, 96, 128
    rng = np.random.default_rng(7)
    A = crandn(rng, 1, M, K) * (10.0 ** rng.uniform(-30, 30, (1, M, 1)))
    B = crandn(rng, 1, K, N) * (10.0 ** rng.uniform(-30, 30, (1, 1, N)))
    C0 = np.zeros((1, M, N), dtype=np.complex128)
    C = torch.from_numpy(C0.copy()).cuda()
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    assert lib.call("cirr_ozaki_zgemm_sub", dA.data_ptr(), K, M * K, dB.data_ptr(), N, K * N, C.data_ptr(), N, M * N,
                    M, N, K, 1, S()) == 0
    torch.cuda.synchronize()
    err = np.abs(C.cpu().numpy() + A @ B)
    assert (err <= bound(A, B)).all()


def test_ozaki_subblocks_in_place(lib):
    """The LU's use: A, B and C are blocks of one array (leading dimension n, batch stride n*n)."""
    n, k0, W = 768, 64, 128
    rng = np.random.default_rng(3)
    P0 = crandn(rng, 2, n, n)
    P = torch.from_numpy(P0.copy()).cuda()
    base = P.data_ptr()
    r0 = k0 + W
    m = n - r0
    off = lambda r, c: base + 16 * (r * n + c)
    assert lib.call("cirr_ozaki_zgemm_sub", off(r0, k0), n, n * n, off(k0, r0), n, n * n, off(r0, r0), n, n * n,
                    m, m, W, 2, S()) == 0
    torch.cuda.synchronize()
    ref = P0.copy()
    ref[:, r0:, r0:] -= P0[:, r0:, k0:r0] @ P0[:, k0:r0, r0:]
    got = P.cpu().numpy()
    assert np.array_equal(got[:, :r0, :], P0[:, :r0, :]) and np.array_equal(got[:, r0:, :r0], P0[:, r0:, :r0])
    err = np.abs(got[:, r0:, r0:] - ref[:, r0:, r0:])
    assert (err <= bound(P0[:, r0:, k0:r0], P0[:, k0:r0, r0:]) + 4e-16 * np.abs(ref[:, r0:, r0:])).all()


def test_ozaki_extreme_magnitudes(lib):
    """Rows near the top and the bottom of the FP64 range keep their relative accuracy (the power-of-two
    scales stay finite)."""
    M, N, K = 128, 32, 64
    rng = np.random.default_rng(9)
    A = crandn(rng, 1, M, K)
    B = crandn(rng, 1, K, N)
    A[0, 0] *= 1e300
    A[0, 1] *= 1e-290
    B[0, :, 2] *= 1e-290
    C = torch.zeros((1, M, N), dtype=torch.complex128, device="cuda")
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    assert lib.call("cirr_ozaki_zgemm_sub", dA.data_ptr(), K, M * K, dB.data_ptr(), N, K * N, C.data_ptr(), N, M * N,
                    M, N, K, 1, S()) == 0
    torch.cuda.synchronize()
    got = -C.cpu().numpy()[0]
    with np.errstate(over="ignore", under="ignore"):
        ref = (A @ B)[0]
    for (i, j) in [(0, 5), (1, 5), (7, 2), (0, 2)]:
        assert abs(got[i, j] - ref[i, j]) <= 1e-13 * abs(ref[i, j]) + 1e-300, (i, j, got[i, j], ref[i, j])


def test_ozaki_zero_and_nonfinite(lib):
    """Zero rows / columns give exact zeros; a NaN poisons its row (as the FP64 GEMM would)."""
    M, N, K = 128, 32, 64
    rng = np.random.default_rng(5)
    A = crandn(rng, 1, M, K)
    B = crandn(rng, 1, K, N)
    A[0, 3, :] = 0
    B[0, :, 5] = 0
    A[0, 9, 2] = np.nan
    C = torch.zeros((1, M, N), dtype=torch.complex128, device="cuda")
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    assert lib.call("cirr_ozaki_zgemm_sub", dA.data_ptr(), K, M * K, dB.data_ptr(), N, K * N, C.data_ptr(), N, M * N,
                    M, N, K, 1, S()) == 0
    torch.cuda.synchronize()
    got = C.cpu().numpy()[0]
    assert (got[3] == 0).all() and (got[:, 5][np.arange(M) != 9] == 0).all()
    assert np.isnan(got[9]).all()
    ok = np.ones(M, dtype=bool)
    ok[9] = False
    assert np.isfinite(got[ok]).all()


def test_ozaki_deterministic(lib):
    M, N, K = 384, 200, 512
    rng = np.random.default_rng(11)
    A, B = crandn(rng, 2, M, K), crandn(rng, 2, K, N)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    outs = []
    for _ in range(2):
        C = torch.zeros((2, M, N), dtype=torch.complex128, device="cuda")
        assert lib.call("cirr_ozaki_zgemm_sub", dA.data_ptr(), K, M * K, dB.data_ptr(), N, K * N, C.data_ptr(), N,
                        M * N, M, N, K, 2, S()) == 0
        torch.cuda.synchronize()
        outs.append(C.cpu().numpy())
    assert np.array_equal(outs[0].view(np.float64), outs[1].view(np.float64))


@pytest.fixture
def int8_mode(lib):
    prev = lib.call("cirr_set_lu_gemm", 1)
    yield
    lib.call("cirr_set_lu_gemm", prev)


def _factor(lib, A):
    batch, n, _ = A.shape
    F = torch.from_numpy(A.copy()).cuda()
    ipiv = torch.empty((batch, n), dtype=torch.int32, device="cuda")
    perm = torch.empty((batch, n), dtype=torch.int32, device="cuda")
    mp = torch.empty(batch, dtype=torch.float64, device="cuda")
    info = torch.empty(batch, dtype=torch.int32, device="cuda")
    ws = torch.zeros(lib.call("cirr_zgetrf_ws_bytes", n, batch), dtype=torch.uint8, device="cuda")
    lib.call("cirr_zgetrf_batched", F.data_ptr(), n, n, n * n, batch, ipiv.data_ptr(), perm.data_ptr(),
             mp.data_ptr(), info.data_ptr(), ws.data_ptr(), S())
    torch.cuda.synchronize()
    assert (info.cpu().numpy() == 0).all()
    return F, ipiv, perm


def test_int8_lu_and_cached_solves(lib, int8_mode):
    """Dense LU with int8 trailing updates, then blocked solves whose k = 512
    updates read the kept factor slices: backward error at the FP64 level, the
    same pivots as the DMMA LU, gathered sub-ranges of the factors included."""
    import scipy.linalg as sla
    n, batch, K = 2048, 3, 40
    rng = np.random.default_rng(2048)
    A = crandn(rng, batch, n, n)
    F, ipiv, perm = _factor(lib, A)
    lib.call("cirr_set_lu_gemm", 0)
    F0, ipiv0, _ = _factor(lib, A)
    lib.call("cirr_set_lu_gemm", 1)
    assert np.array_equal(ipiv.cpu().numpy(), ipiv0.cpu().numpy())
    dlu = (F - F0).abs().max().item() / F0.abs().max().item()
    assert dlu < 1e-11, dlu

    def backward_error(Ft, piv, j=0):
        """max |P A - L U| / (n max|A|) of pencil j, formed in FP64 on the host."""
        lu = Ft[j].cpu().numpy()
        L = np.tril(lu, -1) + np.eye(n)
        U = np.triu(lu)
        pa = A[j].copy()
        for i, pi in enumerate(piv[j].cpu().numpy()):
            if pi != i:
                pa[[i, pi]] = pa[[pi, i]]
        return np.abs(pa - L @ U).max() / (n * np.abs(A[j]).max())

    be8, be64 = backward_error(F, ipiv), backward_error(F0, ipiv0)
    # the int8 updates are as accurate as the FP64 ones (both far below n u max|A|)
    assert be8 < 2.0 ** -52 and be8 <= 2.0 * be64 + 2.0 ** -60, (be8, be64)
    dinv = torch.zeros(lib.call("cirr_diag_inv_bytes", n, batch), dtype=torch.uint8, device="cuda")
    lib.call("cirr_diag_inverses", F.data_ptr(), n, n, n * n, batch, dinv.data_ptr(), S())
    nbytes = lib.call("cirr_ozaki_factor_bytes", n, batch)
    assert nbytes > batch * n * n * 16
    cache = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    launches0 = lib.call("cirr_launch_count")
    lib.call("cirr_ozaki_split_factors", F.data_ptr(), n, n, n * n, batch, cache.data_ptr(), S())
    assert lib.call("cirr_launch_count") - launches0 == n // 512
    R = crandn(rng, 2, n, K)
    dR = torch.from_numpy(R).cuda()

    def solve(first, cnt):
        rhs_of = torch.from_numpy((np.arange(cnt, dtype=np.int32) % 2)).cuda()
        Y = torch.empty((cnt, n, K), dtype=torch.complex128, device="cuda")
        dpp = lib.call("cirr_diag_inv_bytes", n, 1)
        lib.call("cirr_zgetrs_batched", F[first].data_ptr(), n, n, n * n, cnt, perm[first].data_ptr(), dR.data_ptr(),
                 K, n * K, rhs_of.data_ptr(), K, Y.data_ptr(), K, n * K, dinv.data_ptr() + first * dpp, S())
        torch.cuda.synchronize()
        return Y.cpu().numpy()

    l0 = lib.call("cirr_launch_count")
    y = solve(0, batch)
    with_cache = lib.call("cirr_launch_count") - l0
    for j in range(batch):
        res = np.linalg.norm(A[j] @ y[j] - R[j % 2]) / (np.linalg.norm(A[j]) * np.linalg.norm(y[j]))
        assert res < 1e-14, res
    y1 = solve(1, 2)   # a sub-range of the registered factors
    for j in range(2):
        res = np.linalg.norm(A[1 + j] @ y1[j] - R[j % 2]) / (np.linalg.norm(A[1 + j]) * np.linalg.norm(y1[j]))
        assert res < 1e-14, res
    lib.call("cirr_ozaki_release", F.data_ptr())
    l0 = lib.call("cirr_launch_count")
    y2 = solve(0, batch)   # slices released: DMMA path, same solutions to rounding
    without = lib.call("cirr_launch_count") - l0
    assert with_cache != without          # the cached path really ran (3 launches per update instead of 1)
    assert np.abs(y2 - y).max() / np.abs(y).max() < 1e-10
    # a new factorisation in the same memory drops stale slices by itself
    lib.call("cirr_ozaki_split_factors", F.data_ptr(), n, n, n * n, batch, cache.data_ptr(), S())
    F.copy_(torch.from_numpy(A))
    ws = torch.zeros(lib.call("cirr_zgetrf_ws_bytes", n, batch), dtype=torch.uint8, device="cuda")
    mp = torch.empty(batch, dtype=torch.float64, device="cuda")
    info = torch.empty(batch, dtype=torch.int32, device="cuda")
    lib.call("cirr_zgetrf_batched", F.data_ptr(), n, n, n * n, batch, ipiv.data_ptr(), perm.data_ptr(),
             mp.data_ptr(), info.data_ptr(), ws.data_ptr(), S())
    l0 = lib.call("cirr_launch_count")
    solve(0, batch)
    assert lib.call("cirr_launch_count") - l0 == without


def test_engine_int8_matches_fp64(lib):
    """solve_multi on a dense n = 2048 pencil (config-4 generator): the default int8 updates in the LU
    and in the solves (factor slices cut and released by the engine) against the all-FP64 run --
    same counts, same pass counts, eigenvalues to 1e-10, residuals <= 1e-10; the int8 kernels ran."""
    from paper_2511_01927_b200 import Contour, SolverConfig, solve_multi
    from paper_2511_01927_b200 import workloads as W

    a, b = W.config4_matrices(seed=0, n=2048)

    class Pn:
        pass

    p = Pn()
    p.a, p.b, p.hermitian = a, b, False
    cs = [Contour(shape="ellipse", center=0.5 + 0j, semi_re=0.3, semi_im=0.15, expected_count=60),
          Contour(shape="ellipse", center=-0.5 + 0j, semi_re=0.3, semi_im=0.15, expected_count=60)]
    cfg = SolverConfig(n_q=64, source_cols=32, n_moments=8, tol=1e-10)
    prev = lib.call("cirr_set_lu_gemm", 1)
    try:
        l0 = lib.call("cirr_launch_count")
        r8 = solve_multi(p, cs, cfg, seed=0)
        n8 = lib.call("cirr_launch_count") - l0
        lib.call("cirr_set_lu_gemm", 0)
        l0 = lib.call("cirr_launch_count")
        r64 = solve_multi(p, cs, cfg, seed=0)
        n64 = lib.call("cirr_launch_count") - l0
    finally:
        lib.call("cirr_set_lu_gemm", prev)
    assert n8 != n64   # split kernels + int8 updates replace DMMA launches
    # the same outcome per contour in both arithmetics (a contour with an eigenvalue near its boundary may
    # fail to converge in 8 passes in either)
    compared = 0
    for x, y, ex, ey in zip(r8.results, r64.results, r8.errors, r64.errors):
        assert type(ex) is type(ey), (ex, ey)
        if y is None:
            continue
        compared += 1
        assert len(x.eigenvalues) == len(y.eigenvalues) > 0
        assert x.stats.iterations == y.stats.iterations
        for lam in y.eigenvalues:
            assert np.min(np.abs(x.eigenvalues - lam)) <= 1e-10 * max(1.0, abs(lam))
        assert x.residuals.max() <= 1e-10
    assert compared > 0
    # the per-call switch selects the same two paths and restores the library mode
    import dataclasses
    mode0 = lib.call("cirr_set_lu_gemm", -1)
    rf = solve_multi(p, cs, dataclasses.replace(cfg, arith="f64"), seed=0)
    assert lib.call("cirr_set_lu_gemm", -1) == mode0
    for x, y in zip(rf.results, r64.results):
        if y is not None:
            assert np.array_equal(x.eigenvalues, y.eigenvalues)
    # a second int8 run reuses the engine path from scratch (slices re-cut, earlier registration gone)
    r8b = solve_multi(p, cs, cfg, seed=0)
    for x, y in zip(r8.results, r8b.results):
        if x is not None:
            assert np.array_equal(x.eigenvalues, y.eigenvalues)   # integer accumulation: bitwise repeatable


def test_ozaki_many_streams(lib):
    """More launching streams than workspace slots: the oldest workspace is recycled, results stay right."""
    M, N, K = 128, 16, 32
    rng = np.random.default_rng(21)
    A, B = crandn(rng, 1, M, K), crandn(rng, 1, K, N)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    ref = -(A @ B)
    streams = [torch.cuda.Stream() for _ in range(20)]
    for st in streams:
        with torch.cuda.stream(st):
            C = torch.zeros((1, M, N), dtype=torch.complex128, device="cuda")
            assert lib.call("cirr_ozaki_zgemm_sub", dA.data_ptr(), K, M * K, dB.data_ptr(), N, K * N, C.data_ptr(), N,
                            M * N, M, N, K, 1, st.cuda_stream) == 0
            st.synchronize()
            assert np.abs(C.cpu().numpy() - ref).max() < 1e-13
