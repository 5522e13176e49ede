"""Device counterparts of the reference's linalg known-answer tests
(tests/test_linalg.py:57-170 of the reference): the K3 solve, the FEAST
orthonormalisation (CGS2), the rank-truncating orth (K4) and the Hermitian
small eigensolver (K6), called through the C ABI on the same inputs."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_2511_01927_b200 import _lib  # noqa: E402

_KEEP = []


def dev(x):
    t = torch.from_numpy(np.ascontiguousarray(x)).to("cuda")
    _KEEP.append(t)
    return t


def S():
    return torch.cuda.current_stream().cuda_stream


def solve_diag(shift, rhs):
    """Factor shift*I - diag(1, 3) and solve for the columns of rhs."""
    n, K = rhs.shape
    a, b = np.diag([1.0, 3.0]), np.eye(2)
    pen = torch.empty((1, n, n), dtype=torch.complex128, device="cuda")
    mx = torch.empty(1, dtype=torch.float64, device="cuda")
    ipiv = torch.empty((1, n), dtype=torch.int32, device="cuda")
    perm = torch.empty((1, n), dtype=torch.int32, device="cuda")
    mp = torch.empty(1, dtype=torch.float64, device="cuda")
    info = torch.empty(1, dtype=torch.int32, device="cuda")
    _lib.call("cirr_assemble", dev(a).data_ptr(), dev(b).data_ptr(), n, n, dev(np.array([shift + 0j])).data_ptr(),
              1, pen.data_ptr(), n, n * n, mx.data_ptr(), S())
    _lib.call("cirr_zgetrf_batched", pen.data_ptr(), n, n, n * n, 1, ipiv.data_ptr(), perm.data_ptr(), mp.data_ptr(),
              info.data_ptr(), 0, S())
    Y = torch.zeros((1, n, max(K, 1)), dtype=torch.complex128, device="cuda")
    R = dev(rhs.astype(complex).reshape(1, n, K)) if K else Y
    rhs_of = dev(np.zeros(1, np.int32))
    rc = _lib.call("cirr_zgetrs_batched", pen.data_ptr(), n, n, n * n, 1, perm.data_ptr(), R.data_ptr(), max(K, 1),
                   n * max(K, 1), rhs_of.data_ptr(), K, Y.data_ptr(), max(K, 1), n * max(K, 1), 0, S())
    return rc, Y.cpu().numpy()[0, :, :K]


def test_solve_block_diagonal_inverse():
    rc, y = solve_diag(2.0, np.eye(2))
    assert rc == 0
    assert np.allclose(y, np.diag([1.0, -1.0]), atol=1e-14)


def test_solve_block_empty_rhs():
    rc, y = solve_diag(2.0, np.zeros((2, 0)))
    assert rc == 0 and y.shape == (2, 0)


def cgs2(block, drop_tol=1e-10):
    n, c = block.shape
    Yt = dev(np.ascontiguousarray(block.T.astype(complex)))
    Qt = torch.zeros((c, n), dtype=torch.complex128, device="cuda")
    kept = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.call("cirr_orthonormalize", Yt.data_ptr(), n, c * n, n, c, 1, drop_tol, Qt.data_ptr(), n, c * n,
              kept.data_ptr(), S())
    k = kept.item()
    return Qt.cpu().numpy()[:k].T


def test_orthonormalize_idempotent_on_orthonormal():
    q0 = np.linalg.qr(np.random.default_rng(2).standard_normal((10, 4)))[0]
    q = cgs2(q0)
    assert np.abs(q.conj().T @ q - np.eye(4)).max() <= 1e-12
    assert np.abs(q0 @ q0.conj().T - q @ q.conj().T).max() <= 1e-8


def test_orthonormalize_drops_duplicates():
    v = np.random.default_rng(3).standard_normal(20)
    assert cgs2(np.column_stack([v, v])).shape[1] == 1


def test_orthonormalize_gram_accuracy():
    q = cgs2(np.random.default_rng(4).standard_normal((50, 8)))
    assert np.abs(q.conj().T @ q - np.eye(q.shape[1])).max() <= 1e-12


def test_orthonormalize_rank_zero():
    assert cgs2(np.zeros((5, 3))).shape[1] == 0  # the engine raises RankZeroError on kept == 0


def orth(block, rel_tol=1e-12):
    n, c = block.shape
    W = dev(np.ascontiguousarray(block.T.astype(complex)))
    sig = torch.empty(c, dtype=torch.float64, device="cuda")
    order = torch.empty(c, dtype=torch.int32, device="cuda")
    kept = torch.empty(1, dtype=torch.int32, device="cuda")
    Qt = torch.zeros((c, n), dtype=torch.complex128, device="cuda")
    ws = torch.empty(_lib.call("cirr_orth_ws_bytes", c, 1), dtype=torch.uint8, device="cuda")
    sw = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.call("cirr_orth", W.data_ptr(), n, c * n, n, c, 1, rel_tol, sig.data_ptr(), order.data_ptr(),
              kept.data_ptr(), Qt.data_ptr(), n, c * n, ws.data_ptr(), sw.data_ptr(), S())
    k = kept.item()
    return Qt.cpu().numpy()[:k].T


def test_rank_truncate_rank_one():
    u = np.random.default_rng(5).standard_normal(12)
    v = np.random.default_rng(6).standard_normal(4)
    assert orth(np.outer(u, v), rel_tol=1e-8).shape[1] == 1


def test_rank_truncate_orthonormal_keeps_all():
    q0 = np.linalg.qr(np.random.default_rng(7).standard_normal((10, 5)))[0]
    q = orth(q0)
    assert q.shape[1] == 5
    assert np.abs(q0 @ q0.conj().T - q @ q.conj().T).max() <= 1e-8


def test_rank_truncate_near_duplicate():
    rng = np.random.default_rng(8)
    v = rng.standard_normal(30)
    w = rng.standard_normal(30)
    assert orth(np.column_stack([v, v + 1e-12 * w]), rel_tol=1e-8).shape[1] == 1


def test_rank_truncate_zero_block():
    assert orth(np.zeros((4, 2))).shape[1] == 0  # RankZeroError in the engine


def herm_gep(a, b):
    k = a.shape[0]
    kd = torch.tensor([k], dtype=torch.int32, device="cuda")
    ws = torch.empty(_lib.call("cirr_small_eig_ws_bytes", k) + 256, dtype=torch.uint8, device="cuda")
    lam = torch.empty(k, dtype=torch.complex128, device="cuda")
    Sv = torch.zeros((k, k), dtype=torch.complex128, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.call("cirr_small_eig", 1, dev(a.astype(complex)).data_ptr(), dev(b.astype(complex)).data_ptr(), k, k * k,
              kd.data_ptr(), k, 1, ws.data_ptr(), lam.data_ptr(), Sv.data_ptr(), k, k * k, info.data_ptr(), S())
    return lam.cpu().numpy().real, Sv.cpu().numpy(), info.item()


def test_gep_diagonal():
    w, _, info = herm_gep(np.diag([3.0, 1.0]), np.eye(2))
    assert info == 0 and np.allclose(w, [1.0, 3.0], atol=1e-14)


def test_gep_reciprocal_scaling():
    w, _, info = herm_gep(np.eye(2), np.diag([2.0, 4.0]))
    assert info == 0 and np.allclose(np.sort(w), [0.25, 0.5], atol=1e-14)


def _random_pair(seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((6, 6)) + 1j * rng.standard_normal((6, 6))
    y = rng.standard_normal((6, 6)) + 1j * rng.standard_normal((6, 6))
    return x + x.conj().T, y @ y.conj().T + 6 * np.eye(6), rng


def test_gep_random_residuals():
    a, b, _ = _random_pair(9)
    w, v, info = herm_gep(a, b)
    assert info == 0
    for i in range(6):
        r = np.linalg.norm(a @ v[:, i] - w[i] * (b @ v[:, i]))
        assert r <= 1e-10 * (np.linalg.norm(a) + abs(w[i]) * np.linalg.norm(b))
    assert np.abs(v.conj().T @ b @ v - np.eye(6)).max() <= 1e-10


def test_gep_congruence_invariance():
    a, b, rng = _random_pair(10)
    t = rng.standard_normal((6, 6)) + 0.1 * np.eye(6)
    w1, _, _ = herm_gep(a, b)
    w2, _, _ = herm_gep(t.conj().T @ a @ t, t.conj().T @ b @ t)
    assert np.abs(w1 - w2).max() <= 1e-10 * max(1.0, np.abs(w1).max())


def test_gep_indefinite_b():
    _, _, info = herm_gep(np.eye(2), np.diag([1.0, -1.0]))
    assert info > 0  # IndefiniteBError in the engine
