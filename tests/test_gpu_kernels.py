"""Per-kernel numerics on the B200 (each kernel vs numpy/scipy on seeded inputs)."""
import numpy as np
import pytest
import scipy.linalg as sla

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.fail("gpu test without CUDA")
    from paper_2511_01927_b200 import _lib
    return _lib


def P(t):
    return t.data_ptr()


def ws_lu(n, batch):
    from paper_2511_01927_b200 import _lib
    return cuda(np.zeros(_lib.call("cirr_zgetrf_ws_bytes", n, batch), dtype=np.uint8))


def S():
    return torch.cuda.current_stream().cuda_stream


_KEEP = []


def cuda(x):
    """Device copy kept alive for the test module (raw pointers outlive temporaries)."""
    t = torch.from_numpy(np.ascontiguousarray(x)).to("cuda")
    _KEEP.append(t)
    if len(_KEEP) > 64:
        del _KEEP[:32]
    return t


@pytest.mark.parametrize("n", [5, 64, 300])
def test_assemble_bitwise(lib, n):
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n))
    b = rng.standard_normal((n, n))
    z = rng.standard_normal(11) + 1j * rng.standard_normal(11)
    out = torch.empty((11, n, n), dtype=torch.complex128, device="cuda")
    mx = torch.empty(11, dtype=torch.float64, device="cuda")
    lib.call("cirr_assemble", P(cuda(a)), P(cuda(b)), n, n, P(cuda(z)), 11, P(out), n, n * n, P(mx), S())
    got = out.cpu().numpy()
    for j in range(11):
        ref = z[j] * b - a
        assert np.array_equal(got[j].view(np.float64), ref.view(np.float64)), j
        assert mx.cpu().numpy()[j] == pytest.approx(np.abs(ref).max(), rel=1e-15)


@pytest.mark.parametrize("kind", [0, 1, 2])
@pytest.mark.parametrize("shape", [(64, 64, 64), (100, 37, 250), (7, 130, 5), (256, 256, 4096)])
def test_gemm(lib, kind, shape):
    M, N, K = shape
    rng = np.random.default_rng(M + N + K + kind)
    batch = 2
    if kind == 2:
        A = rng.standard_normal((batch, M, K))
    else:
        A = rng.standard_normal((batch, M, K)) + 1j * rng.standard_normal((batch, M, K))
    B = rng.standard_normal((batch, K, N)) + 1j * rng.standard_normal((batch, K, N))
    C0 = rng.standard_normal((batch, M, N)) + 1j * rng.standard_normal((batch, M, N))
    opA = np.conj(A) if kind == 1 else A
    for beta in (0, 1):
        C = cuda(C0.copy())
        lib.call("cirr_gemm", kind, M, N, K, batch, P(cuda(A)), K, M * K, P(cuda(B)), N, K * N, P(C), N, M * N,
                 -0.5, beta, S())
        ref = beta * C0 - 0.5 * opA @ B
        err = np.abs(C.cpu().numpy() - ref).max() / max(1.0, np.abs(ref).max())
        assert err < 1e-13 * np.sqrt(K), (beta, err)


@pytest.mark.parametrize("K,use_dinv", [(37, False), (100, False), (100, True), (1, True), (2, True), (1, False)])
@pytest.mark.parametrize("n,batch", [(3, 2), (100, 3), (256, 4), (333, 2), (700, 2), (1024, 2)])
def test_getrf_getrs(lib, n, batch, K, use_dinv):
    rng = np.random.default_rng(n)
    A = rng.standard_normal((batch, n, n)) + 1j * rng.standard_normal((batch, n, n))
    F = cuda(A.copy())
    ipiv = torch.empty((batch, n), dtype=torch.int32, device="cuda")
    perm = torch.empty((batch, n), dtype=torch.int32, device="cuda")
    mp = torch.empty(batch, dtype=torch.float64, device="cuda")
    info = torch.empty(batch, dtype=torch.int32, device="cuda")
    lib.call("cirr_zgetrf_batched", P(F), n, n, n * n, batch, P(ipiv), P(perm), P(mp), P(info), P(ws_lu(n, batch)), S())
    assert (info.cpu().numpy() == 0).all()
    dinv = 0
    if use_dinv:
        dinv_t = cuda(np.zeros(lib.call("cirr_diag_inv_bytes", n, batch), dtype=np.uint8))
        lib.call("cirr_diag_inverses", P(F), n, n, n * n, batch, P(dinv_t), S())
        dinv = P(dinv_t)
    R = rng.standard_normal((2, n, K)) + 1j * rng.standard_normal((2, n, K))
    rhs_of = cuda(np.arange(batch, dtype=np.int32) % 2)
    Y = torch.empty((batch, n, K), dtype=torch.complex128, device="cuda")
    lib.call("cirr_zgetrs_batched", P(F), n, n, n * n, batch, P(perm), P(cuda(R)), K, n * K, P(rhs_of), K, P(Y), K,
             n * K, dinv, S())
    y = Y.cpu().numpy()
    lu = F.cpu().numpy()
    for j in range(batch):
        r = R[j % 2]
        res = np.linalg.norm(A[j] @ y[j] - r) / (np.linalg.norm(A[j]) * np.linalg.norm(y[j]))
        assert res < 1e-14, res
        # LAPACK agreement on the pivots' magnitudes
        lu_ref, piv_ref = sla.lu_factor(A[j])
        assert np.allclose(np.sort(np.abs(np.diag(lu[j]))), np.sort(np.abs(np.diag(lu_ref))), rtol=1e-8)
        assert mp.cpu().numpy()[j] == pytest.approx(np.abs(np.diag(lu[j])).min())


@pytest.mark.parametrize("K,use_dinv", [(8, False), (37, True), (37, False), (2, True)])
@pytest.mark.parametrize("n", [256, 333])
def test_getrs_gather(lib, n, K, use_dinv):
    """cirr_zgetrs_gather over a scattered subset of the factors equals
    cirr_zgetrs_batched on each factor alone, bit for bit."""
    rng = np.random.default_rng(n + K)
    nfac = 7
    A = rng.standard_normal((nfac, n, n)) + 1j * rng.standard_normal((nfac, n, n))
    F = cuda(A.copy())
    ipiv = torch.empty((nfac, n), dtype=torch.int32, device="cuda")
    perm = torch.empty((nfac, n), dtype=torch.int32, device="cuda")
    mp = torch.empty(nfac, dtype=torch.float64, device="cuda")
    info = torch.empty(nfac, dtype=torch.int32, device="cuda")
    lib.call("cirr_zgetrf_batched", P(F), n, n, n * n, nfac, P(ipiv), P(perm), P(mp), P(info), P(ws_lu(n, nfac)), S())
    dpp = lib.call("cirr_diag_inv_bytes", n, 1)
    dinv_t = cuda(np.zeros(dpp * nfac, dtype=np.uint8))
    if use_dinv:
        lib.call("cirr_diag_inverses", P(F), n, n, n * n, nfac, P(dinv_t), S())
    pen = np.array([5, 1, 6, 2], dtype=np.int32)
    R = rng.standard_normal((2, n, K)) + 1j * rng.standard_normal((2, n, K))
    Rd = cuda(R)
    rhs_of = cuda(np.array([0, 1, 1, 0], dtype=np.int32))
    Y = torch.empty((len(pen), n, K), dtype=torch.complex128, device="cuda")
    lib.call("cirr_zgetrs_gather", P(F), n, n, n * n, nfac, P(cuda(pen)), len(pen), P(perm), P(Rd), K, n * K,
             P(rhs_of), K, P(Y), K, n * K, P(dinv_t) if use_dinv else 0, S())
    got = Y.cpu().numpy()
    for j, f in enumerate(pen):
        Y1 = torch.empty((1, n, K), dtype=torch.complex128, device="cuda")
        ro = cuda(np.array([rhs_of.cpu().numpy()[j]], dtype=np.int32))
        lib.call("cirr_zgetrs_batched", P(F[f]), n, n, n * n, 1, P(perm[f]), P(Rd), K, n * K, P(ro), K, P(Y1), K,
                 n * K, (P(dinv_t) + int(f) * dpp) if use_dinv else 0, S())
        assert np.array_equal(got[j], Y1.cpu().numpy()[0]), (j, f)
        r = R[rhs_of.cpu().numpy()[j]]
        res = np.linalg.norm(A[f] @ got[j] - r) / (np.linalg.norm(A[f]) * np.linalg.norm(got[j]))
        assert res < 1e-14, res


@pytest.mark.parametrize("n", [70, 256])
def test_getrf_large_batch_short_panels(lib, n):
    """Large batches of short panels (config 2's regime: the 128-thread panel,
    4 CTAs per SM): solutions, pivots and pivot magnitudes as LAPACK's for a
    sample of the 1024 factors; min |U_ii| as reported."""
    batch = 1024
    rng = np.random.default_rng(n + 7)
    A = rng.standard_normal((batch, n, n)) + 1j * rng.standard_normal((batch, n, n))
    F = cuda(A.copy())
    ipiv = torch.empty((batch, n), dtype=torch.int32, device="cuda")
    perm = torch.empty((batch, n), dtype=torch.int32, device="cuda")
    mp = torch.empty(batch, dtype=torch.float64, device="cuda")
    info = torch.empty(batch, dtype=torch.int32, device="cuda")
    lib.call("cirr_zgetrf_batched", P(F), n, n, n * n, batch, P(ipiv), P(perm), P(mp), P(info), P(ws_lu(n, batch)),
             S())
    assert (info.cpu().numpy() == 0).all()
    K = 5
    R = rng.standard_normal((1, n, K)) + 1j * rng.standard_normal((1, n, K))
    rhs_of = cuda(np.zeros(batch, dtype=np.int32))
    Y = torch.empty((batch, n, K), dtype=torch.complex128, device="cuda")
    lib.call("cirr_zgetrs_batched", P(F), n, n, n * n, batch, P(perm), P(cuda(R)), K, n * K, P(rhs_of), K, P(Y), K,
             n * K, 0, S())
    y, lu, piv_h, mph = Y.cpu().numpy(), F.cpu().numpy(), ipiv.cpu().numpy(), mp.cpu().numpy()
    for j in list(range(0, batch, 97)) + [batch - 1]:
        res = np.linalg.norm(A[j] @ y[j] - R[0]) / (np.linalg.norm(A[j]) * np.linalg.norm(y[j]))
        assert res < 1e-14, (j, res)
        lu_ref, piv_ref = sla.lu_factor(A[j])
        assert np.array_equal(piv_h[j], piv_ref), j          # izamax pivoting, first index on ties
        assert np.allclose(np.abs(np.diag(lu[j])), np.abs(np.diag(lu_ref)), rtol=1e-9)
        assert mph[j] == pytest.approx(np.abs(np.diag(lu[j])).min())


def test_getrf_singular(lib):
    n = 70
    A = np.diag(np.arange(1.0, n + 1)).astype(complex)
    A[5, 5] = 0.0
    F = cuda(A[None].copy())
    ipiv = torch.empty((1, n), dtype=torch.int32, device="cuda")
    mp = torch.empty(1, dtype=torch.float64, device="cuda")
    info = torch.empty(1, dtype=torch.int32, device="cuda")
    lib.call("cirr_zgetrf_batched", P(F), n, n, n * n, 1, P(ipiv), 0, P(mp), P(info), P(ws_lu(n, 1)), S())
    assert info.item() == 6 and mp.item() == 0.0


@pytest.mark.parametrize("n,c", [(500, 12), (4096, 64), (1500, 800), (1200, 1000)])   # wide blocks: smaller Jacobi blocks
def test_orth_graded(lib, n, c):
    rng = np.random.default_rng(c)
    U, _ = np.linalg.qr(rng.standard_normal((n, c)) + 1j * rng.standard_normal((n, c)))
    V, _ = np.linalg.qr(rng.standard_normal((c, c)) + 1j * rng.standard_normal((c, c)))
    s = np.logspace(0, -14, c)
    s[(s > 2e-13) & (s < 5e-12)] = 1e-11  # keep the 1e-12 cut away from any sigma
    Smat = (U * s) @ V.conj().T
    W = cuda(np.ascontiguousarray(Smat.T))
    sig = torch.empty(c, dtype=torch.float64, device="cuda")
    order = torch.empty(c, dtype=torch.int32, device="cuda")
    kept = torch.empty(1, dtype=torch.int32, device="cuda")
    Qt = torch.empty((c, n), dtype=torch.complex128, device="cuda")
    ws = torch.empty(lib.call("cirr_orth_ws_bytes", c, 1), dtype=torch.uint8, device="cuda")
    sw = torch.zeros(1, dtype=torch.int32, device="cuda")
    lib.call("cirr_orth", P(W), n, c * n, n, c, 1, 1e-12, P(sig), P(order), P(kept), P(Qt), n, c * n, P(ws), P(sw),
             S())
    k = kept.item()
    ref = np.linalg.svd(Smat, compute_uv=False)
    got = sig.cpu().numpy()
    assert np.allclose(got, ref, rtol=1e-3, atol=1e-15), (got, ref, sw.item())
    assert np.allclose(got[:k], ref[:k], rtol=1e-6, atol=1e-15)
    assert k == int(np.count_nonzero(ref >= 1e-12 * ref[0]))
    q = Qt.cpu().numpy()[:k].T
    assert np.abs(q.conj().T @ q - np.eye(k)).max() < 1e-11
    # span: the kept basis captures S up to the dropped singular values
    resid = np.linalg.norm(Smat - q @ (q.conj().T @ Smat), 2)
    assert resid <= 1e-12 * ref[0] + (ref[k] if k < c else 0.0)


@pytest.mark.parametrize("n,c,nprob", [(256, 32, 40), (300, 17, 16), (64, 64, 20)])
def test_orth_small_batch(lib, n, c, nprob):
    """Many small blocks take the one-CTA-per-problem kernel (whole block in
    shared memory): singular values, rank cut, orthonormality and span against
    numpy's SVD per problem, graded spectra down to 1e-14 as in test_orth_graded."""
    rng = np.random.default_rng(n + c)
    mats, Ws = [], []
    for p_ in range(nprob):
        U, _ = np.linalg.qr(rng.standard_normal((n, c)) + 1j * rng.standard_normal((n, c)))
        V, _ = np.linalg.qr(rng.standard_normal((c, c)) + 1j * rng.standard_normal((c, c)))
        s = np.logspace(0, -(14 if p_ % 2 else 6), c)
        s[(s > 2e-13) & (s < 5e-12)] = 1e-11
        m = (U * s) @ V.conj().T
        mats.append(m)
        Ws.append(m.T)
    W = cuda(np.ascontiguousarray(np.stack(Ws)))
    sig = torch.empty((nprob, c), dtype=torch.float64, device="cuda")
    order = torch.empty((nprob, c), dtype=torch.int32, device="cuda")
    kept = torch.empty(nprob, dtype=torch.int32, device="cuda")
    Qt = torch.zeros((nprob, c, n), dtype=torch.complex128, device="cuda")
    ws = torch.empty(lib.call("cirr_orth_ws_bytes", c, nprob), dtype=torch.uint8, device="cuda")
    sw = torch.zeros(1, dtype=torch.int32, device="cuda")
    lib.call("cirr_orth", P(W), n, c * n, n, c, nprob, 1e-12, P(sig), P(order), P(kept), P(Qt), n, c * n, P(ws),
             P(sw), S())
    ks, got, qs = kept.cpu().numpy(), sig.cpu().numpy(), Qt.cpu().numpy()
    assert 0 < sw.item() <= 60
    for p_, m in enumerate(mats):
        ref = np.linalg.svd(m, compute_uv=False)
        k = int(ks[p_])
        assert np.allclose(got[p_], ref, rtol=1e-3, atol=1e-15)
        assert np.allclose(got[p_, :k], ref[:k], rtol=1e-6, atol=1e-15)
        assert k == int(np.count_nonzero(ref >= 1e-12 * ref[0]))
        q = qs[p_, :k].T
        assert np.abs(q.conj().T @ q - np.eye(k)).max() < 1e-11
        resid = np.linalg.norm(m - q @ (q.conj().T @ m), 2)
        assert resid <= 1e-12 * ref[0] + (ref[k] if k < c else 0.0)


@pytest.mark.parametrize("kind,M,N,K,batch,beta", [(1, 118, 118, 4096, 2, 0), (1, 70, 33, 2000, 3, 1),
                                                    (2, 4096, 118, 4096, 1, 0), (0, 5, 7, 4096, 1, 1)])
def test_gemm_splitk(lib, kind, M, N, K, batch, beta):
    """Shapes that take the split-K path (small output, long K): same result as
    numpy; repeat calls are bitwise identical (fixed-order slice reduction)."""
    rng = np.random.default_rng(M + K)
    if kind == 2:
        a = rng.standard_normal((batch, M, K))
    else:
        a = rng.standard_normal((batch, M, K)) + 1j * rng.standard_normal((batch, M, K))
    b = rng.standard_normal((batch, K, N)) + 1j * rng.standard_normal((batch, K, N))
    c0 = rng.standard_normal((batch, M, N)) + 1j * rng.standard_normal((batch, M, N))
    ref = 0.5 * np.einsum("bmk,bkn->bmn", np.conj(a) if kind == 1 else a, b) + (c0 if beta else 0)
    A, B = cuda(a), cuda(b)
    outs = []
    for _ in range(2):
        C = cuda(c0.copy())
        assert lib.call("cirr_gemm", kind, M, N, K, batch, P(A), K, M * K, P(B), N, K * N, P(C), N, M * N, 0.5, beta,
                        S()) == 0
        outs.append(C.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])
    assert np.abs(outs[0] - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("M", [1, 3, 8])
def test_moments(lib, M):
    """S_m = sum_j coef[j][m] Y_j per contour, written transposed (K3 epilogue)."""
    n, K = 300, 37
    nodes = [5, 7]
    rng = np.random.default_rng(M)
    npen = sum(nodes)
    Y = rng.standard_normal((npen, n, K)) + 1j * rng.standard_normal((npen, n, K))
    coef = rng.standard_normal((npen, M)) + 1j * rng.standard_normal((npen, M))
    off = np.concatenate([[0], np.cumsum(nodes)]).astype(np.int32)
    St = torch.zeros((len(nodes), M * K, n), dtype=torch.complex128, device="cuda")
    assert lib.call("cirr_moments", P(cuda(Y)), K, n * K, n, K, P(cuda(coef)), M, P(cuda(off)), len(nodes), P(St),
                    n, M * K * n, S()) == 0
    torch.cuda.synchronize()
    got = St.cpu().numpy()
    for c in range(len(nodes)):
        for m in range(M):
            ref = np.einsum("j,jrk->rk", coef[off[c]:off[c + 1], m], Y[off[c]:off[c + 1]])
            assert np.allclose(got[c, m * K:(m + 1) * K].T, ref, rtol=0, atol=1e-13 * np.abs(ref).max())


@pytest.mark.parametrize("K,M,use_dinv,gather", [(32, 8, True, False), (118, 1, True, True), (8, 4, False, False),
                                                  (2, 1, True, False), (37, 16, True, True)])
@pytest.mark.parametrize("n", [333, 600])
def test_zgetrs_moments_fused(lib, n, K, M, use_dinv, gather):
    """cirr_zgetrs_moments (solve with the moment accumulation inside the call,
    block row by block row on the blocked path) equals cirr_zgetrs_batched /
    _gather followed by cirr_moments, bit for bit, for every solve path."""
    rng = np.random.default_rng(n * K + M)
    nodes = [3, 4]
    nfac = 9
    A = rng.standard_normal((nfac, n, n)) + 1j * rng.standard_normal((nfac, n, n))
    F = cuda(A.copy())
    ipiv = torch.empty((nfac, n), dtype=torch.int32, device="cuda")
    perm = torch.empty((nfac, n), dtype=torch.int32, device="cuda")
    mp = torch.empty(nfac, dtype=torch.float64, device="cuda")
    info = torch.empty(nfac, dtype=torch.int32, device="cuda")
    lib.call("cirr_zgetrf_batched", P(F), n, n, n * n, nfac, P(ipiv), P(perm), P(mp), P(info), P(ws_lu(n, nfac)), S())
    dinv = 0
    if use_dinv:
        dinv_t = cuda(np.zeros(lib.call("cirr_diag_inv_bytes", n, nfac), dtype=np.uint8))
        lib.call("cirr_diag_inverses", P(F), n, n, n * n, nfac, P(dinv_t), S())
        dinv = P(dinv_t)
    batch = sum(nodes)
    pen_of = np.array([8, 1, 3, 0, 5, 6, 2], dtype=np.int32) if gather else None
    R = cuda(rng.standard_normal((2, n, K)) + 1j * rng.standard_normal((2, n, K)))
    rhs_of = cuda(np.repeat(np.arange(2, dtype=np.int32), nodes))
    coef = cuda(rng.standard_normal((batch, M)) + 1j * rng.standard_normal((batch, M)))
    off = cuda(np.concatenate([[0], np.cumsum(nodes)]).astype(np.int32))
    Y1 = torch.empty((batch, n, K), dtype=torch.complex128, device="cuda")
    Y2 = torch.empty_like(Y1)
    S1 = torch.zeros((2, M * K, n), dtype=torch.complex128, device="cuda")
    S2 = torch.zeros_like(S1)
    if gather:
        po = cuda(pen_of)
        assert lib.call("cirr_zgetrs_gather", P(F), n, n, n * n, nfac, P(po), batch, P(perm), P(R), K, n * K,
                        P(rhs_of), K, P(Y1), K, n * K, dinv, S()) == 0
        pp = P(po)
    else:
        assert lib.call("cirr_zgetrs_batched", P(F), n, n, n * n, batch, P(perm), P(R), K, n * K, P(rhs_of), K,
                        P(Y1), K, n * K, dinv, S()) == 0
        pp = 0
    assert lib.call("cirr_moments", P(Y1), K, n * K, n, K, P(coef), M, P(off), 2, P(S1), n, M * K * n, S()) == 0
    assert lib.call("cirr_zgetrs_moments", P(F), n, n, n * n, nfac, pp, batch, P(perm), P(R), K, n * K, P(rhs_of),
                    K, P(Y2), K, n * K, dinv, P(coef), M, P(off), 2, P(S2), n, M * K * n, S()) == 0
    torch.cuda.synchronize()
    assert torch.equal(Y1, Y2)
    assert torch.equal(S1, S2)


def _cholqr2(lib, mats, c, kappa_max=1e5):
    """mats: list of n x c_p blocks (c_p <= c); returns (Qt rows, ok) per block."""
    nb, n = len(mats), mats[0].shape[0]
    Wh = np.zeros((nb, c, n), dtype=np.complex128)
    for b, m in enumerate(mats):
        Wh[b, : m.shape[1]] = m.T
    W = cuda(Wh)
    cd = cuda(np.array([m.shape[1] for m in mats], dtype=np.int32))
    Qt = torch.empty((nb, c, n), dtype=torch.complex128, device="cuda")
    ws = torch.empty(lib.call("cirr_orth_cholqr2_ws_bytes", n, c, nb), dtype=torch.uint8, device="cuda")
    ok = torch.full((nb,), -1, dtype=torch.int32, device="cuda")
    assert lib.call("cirr_orth_cholqr2", P(W), n, c * n, n, c, nb, P(cd), kappa_max, P(Qt), n, c * n, P(ws), P(ok),
                    S()) == 0
    assert np.array_equal(Wh, W.cpu().numpy())  # input untouched
    return Qt.cpu().numpy(), ok.cpu().numpy()


@pytest.mark.parametrize("c", [120, 200])   # shared-memory factor (c <= 160) and the global-memory one
def test_orth_cholqr2(lib, c):
    """Certified CholeskyQR2: orthonormal rows spanning range(S) when
    ||R||_F ||R^-1||_F <= kappa_max; rejected (ok = 0) for a graded block
    the SVD path must truncate, and for a zero block."""
    n = 4096
    rng = np.random.default_rng(5)
    good = []
    for cp, cond in ((c, 1e3), (c - 23, 1e2)):
        U, _ = np.linalg.qr(rng.standard_normal((n, cp)) + 1j * rng.standard_normal((n, cp)))
        V, _ = np.linalg.qr(rng.standard_normal((cp, cp)) + 1j * rng.standard_normal((cp, cp)))
        good.append((U * np.logspace(0, -np.log10(cond), cp)) @ V.conj().T * 3.7)
    Qt, ok = _cholqr2(lib, good, c)
    assert ok.tolist() == [1, 1]
    for b, m in enumerate(good):
        cp = m.shape[1]
        q = Qt[b, :cp].T
        assert np.abs(q.conj().T @ q - np.eye(cp)).max() < 1e-13
        assert cp == c or np.abs(Qt[b, cp:]).max() == 0.0
        assert np.linalg.norm(m - q @ (q.conj().T @ m), 2) <= 1e-13 * np.linalg.norm(m, 2)
    U, _ = np.linalg.qr(rng.standard_normal((n, c)) + 1j * rng.standard_normal((n, c)))
    graded = (U * np.logspace(0, -12, c))
    _, ok = _cholqr2(lib, [graded, np.zeros((n, c), dtype=np.complex128)], c)
    assert ok.tolist() == [0, 0]


@pytest.mark.parametrize("k", [1, 6, 64, 80, 81, 200])
def test_small_eig_hermitian(lib, k):
    rng = np.random.default_rng(k)
    x = rng.standard_normal((k, k)) + 1j * rng.standard_normal((k, k))
    a = x + x.conj().T
    y = rng.standard_normal((k, k)) + 1j * rng.standard_normal((k, k))
    b = y @ y.conj().T + k * np.eye(k)
    lam, s, info = _small(lib, a, b, k, 1)
    assert info == 0
    w = sla.eigh(a, b, eigvals_only=True)
    assert np.allclose(lam.real, w, rtol=1e-10, atol=1e-12 * np.abs(w).max())
    r = a @ s - (b @ s) * lam.real[None, :]
    assert np.abs(r).max() <= 1e-10 * (np.linalg.norm(a) + np.abs(lam).max() * np.linalg.norm(b))
    assert np.abs(s.conj().T @ b @ s - np.eye(k)).max() < 1e-10


@pytest.mark.parametrize("k", [2, 7, 64, 180])
def test_small_eig_general(lib, k):
    rng = np.random.default_rng(100 + k)
    a = rng.standard_normal((k, k)) + 1j * rng.standard_normal((k, k))
    b = np.eye(k) + 0.05 * (rng.standard_normal((k, k)) + 1j * rng.standard_normal((k, k)))
    lam, s, info = _small(lib, a, b, k, 0)
    assert info == 0
    w = sla.eig(a, b, right=False)
    w = w[np.lexsort((w.imag, w.real))]
    assert np.abs(lam - w).max() < 1e-10 * np.abs(w).max()
    r = a @ s - (b @ s) * lam[None, :]
    rel = np.linalg.norm(r, axis=0) / (np.linalg.norm(a @ s, axis=0) + np.abs(lam) * np.linalg.norm(b @ s, axis=0))
    assert rel.max() < 1e-11


@pytest.mark.parametrize("ks", [[100], [256, 200, 130], [90, 90]])
def test_small_eig_hermitian_definite_batch(lib, ks):
    """k > 78 with A~ positive definite (the projected stiffness of configs 3/5):
    the one-sided Jacobi across the GPU (cirr_orth on A' = L^-1 A~ L^-H) gives
    eigh's eigenvalues and B~-orthonormal eigenvectors; padded problems of
    different sizes in one batch.  (The indefinite cases of
    test_small_eig_hermitian take the per-CTA fallback.)"""
    kmax, nb = max(ks), len(ks)
    rng = np.random.default_rng(sum(ks))
    A = np.zeros((nb, kmax, kmax), complex)
    B = np.zeros((nb, kmax, kmax), complex)
    for p_, k in enumerate(ks):
        x = rng.standard_normal((k, k)) + 1j * rng.standard_normal((k, k))
        A[p_, :k, :k] = x @ x.conj().T / k + np.diag(rng.uniform(0.5, 2.0, k))
        y = rng.standard_normal((k, k)) + 1j * rng.standard_normal((k, k))
        B[p_, :k, :k] = y @ y.conj().T / k + np.eye(k)
    kd = torch.tensor(ks, dtype=torch.int32, device="cuda")
    wsb = lib.call("cirr_small_eig_ws_bytes", kmax)
    ws = torch.empty(nb * ((wsb + 255) // 256 * 256), dtype=torch.uint8, device="cuda")
    lam = torch.zeros((nb, kmax), dtype=torch.complex128, device="cuda")
    s = torch.zeros((nb, kmax, kmax), dtype=torch.complex128, device="cuda")
    info = torch.zeros(nb, dtype=torch.int32, device="cuda")
    lib.call("cirr_small_eig", 1, P(cuda(A)), P(cuda(B)), kmax, kmax * kmax, P(kd), kmax, nb, P(ws), P(lam), P(s),
             kmax, kmax * kmax, P(info), S())
    assert (info.cpu().numpy() == 0).all()
    lh, sh = lam.cpu().numpy(), s.cpu().numpy()
    for p_, k in enumerate(ks):
        a, b = A[p_, :k, :k], B[p_, :k, :k]
        w = sla.eigh(a, b, eigvals_only=True)
        got, x = lh[p_, :k].real, sh[p_, :k, :k]
        assert np.allclose(got, w, rtol=1e-10, atol=1e-12 * np.abs(w).max()), (p_, np.abs(got - w).max())
        r = a @ x - (b @ x) * got[None, :]
        assert np.abs(r).max() <= 1e-10 * (np.linalg.norm(a) + np.abs(got).max() * np.linalg.norm(b))
        assert np.abs(x.conj().T @ b @ x - np.eye(k)).max() < 1e-10


def test_small_eig_indefinite(lib):
    a = np.eye(2, dtype=complex)
    b = np.diag([1.0, -1.0]).astype(complex)
    _, _, info = _small(lib, a, b, 2, 1)
    assert info == 2


def _small(lib, a, b, k, herm):
    kd = torch.tensor([k], dtype=torch.int32, device="cuda")
    wsb = lib.call("cirr_small_eig_ws_bytes", k)
    ws = torch.empty(wsb + 256, dtype=torch.uint8, device="cuda")
    lam = torch.empty(k, dtype=torch.complex128, device="cuda")
    s = torch.empty((k, k), dtype=torch.complex128, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    lib.call("cirr_small_eig", herm, P(cuda(a)), P(cuda(b)), k, k * k, P(kd), k, 1, P(ws), P(lam), P(s), k, k * k,
             P(info), S())
    return lam.cpu().numpy(), s.cpu().numpy(), info.item()


def _banded(rng, batch, n, kl, ku):
    A = rng.standard_normal((batch, n, n)) + 1j * rng.standard_normal((batch, n, n))
    i, j = np.indices((n, n))
    A[:, (i - j > kl) | (j - i > ku)] = 0.0
    return A


@pytest.mark.parametrize("n,batch,kl,ku", [(100, 3, 3, 5), (256, 2, 16, 16), (700, 2, 40, 10), (2304, 2, 48, 48),
                                           (256, 1100, 16, 16), (300, 2, 0, 7)])
def test_band_lu_and_solves_bitwise(lib, n, batch, kl, ku):
    """The band-limited LU and solves (cirr_zgetrf_band, cirr_zgetrs_band) on
    banded pencils give the pivots of the dense LU and, with the same blocking
    (n < 256: single 64-column steps in both), bitwise its factors -- the
    skipped blocks are exact zeros; banded pencils of n >= 256 take single
    steps where the dense LU uses multi-level ones, so equal to rounding there.
    The band-limited solves are bitwise the dense solves on the same factors,
    and L's reported lower bandwidth bounds its nonzeros."""
    rng = np.random.default_rng(n + kl)
    A = _banded(rng, batch, n, kl, ku)
    outs = {}
    for mode in ("dense", "band"):
        F = cuda(A.copy())
        ipiv = torch.empty((batch, n), dtype=torch.int32, device="cuda")
        perm = torch.empty((batch, n), dtype=torch.int32, device="cuda")
        mp = torch.empty(batch, dtype=torch.float64, device="cuda")
        info = torch.empty(batch, dtype=torch.int32, device="cuda")
        lbw = torch.zeros(batch, dtype=torch.int32, device="cuda")
        if mode == "dense":
            lib.call("cirr_zgetrf_batched", P(F), n, n, n * n, batch, P(ipiv), P(perm), P(mp), P(info),
                     P(ws_lu(n, batch)), S())
        else:
            lib.call("cirr_zgetrf_band", P(F), n, n, n * n, batch, kl, ku, P(ipiv), P(perm), P(mp), P(info), P(lbw),
                     P(ws_lu(n, batch)), S())
        outs[mode] = (F, ipiv, perm, mp, lbw)
    Fd, Fb = outs["dense"][0], outs["band"][0]
    if n < 256:   # both single 64-column steps: the same products in the same order
        assert torch.equal(Fd, Fb)
        assert torch.equal(outs["dense"][3], outs["band"][3])
    else:         # banded pencils take PB = 1 steps, the dense LU multi-level ones: equal to rounding
        assert (Fd - Fb).abs().max().item() <= 1e-12 * Fd.abs().max().item()
    assert torch.equal(outs["dense"][1], outs["band"][1])
    klL = max(kl, int(outs["band"][4].max().item()))
    kuU = min(n - 1, kl + ku)
    lu = Fb.cpu().numpy()
    i, j = np.indices((n, n))
    low = np.abs(lu[:, (i - j > klL)]).max(initial=0.0)
    upp = np.abs(lu[:, (j - i > kuU)]).max(initial=0.0)
    assert low == 0.0 and upp == 0.0, (klL, kuU, low, upp)
    perm = outs["band"][2]
    for K, use_dinv in ((8, False), (37, True), (37, False)):
        dinv = 0
        if use_dinv:
            dinv_t = cuda(np.zeros(lib.call("cirr_diag_inv_bytes", n, batch), dtype=np.uint8))
            lib.call("cirr_diag_inverses", P(Fb), n, n, n * n, batch, P(dinv_t), S())
            dinv = P(dinv_t)
        R = rng.standard_normal((1, n, K)) + 1j * rng.standard_normal((1, n, K))
        Rt = cuda(R)
        rhs_of = cuda(np.zeros(batch, dtype=np.int32))
        Yd = torch.empty((batch, n, K), dtype=torch.complex128, device="cuda")
        Yb = torch.empty_like(Yd)
        lib.call("cirr_zgetrs_batched", P(Fb), n, n, n * n, batch, P(perm), P(Rt), K, n * K, P(rhs_of), K, P(Yd), K,
                 n * K, dinv, S())
        lib.call("cirr_zgetrs_band", P(Fb), n, n, n * n, batch, 0, batch, P(perm), P(Rt), K, n * K, P(rhs_of), K,
                 P(Yb), K, n * K, dinv, 0, 0, 0, 0, 0, 0, 0, klL, kuU, S())
        assert torch.equal(Yd, Yb), (K, use_dinv)
        y = Yb.cpu().numpy()
        for b in (0, batch - 1):
            res = np.linalg.norm(A[b] @ y[b] - R[0]) / (np.linalg.norm(A[b]) * np.linalg.norm(y[b]))
            assert res < 1e-13, (K, b, res)
