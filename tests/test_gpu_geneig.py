"""Split non-Hermitian eigensolver (eigenvalues, then selected eigenvectors)."""
import numpy as np
import pytest
import scipy.linalg as sla

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from paper_2511_01927_b200 import _lib  # noqa: E402


@pytest.mark.parametrize("ks", [[3], [7, 5], [64, 60], [120, 112], [256, 255]])
def test_gen_eig_split(ks):
    kmax, nb = max(ks), len(ks)
    rng = np.random.default_rng(sum(ks))
    A = np.zeros((nb, kmax, kmax), complex)
    B = np.zeros((nb, kmax, kmax), complex)
    for b, k in enumerate(ks):
        A[b, :k, :k] = rng.standard_normal((k, k)) + 1j * rng.standard_normal((k, k))
        B[b, :k, :k] = np.eye(k) + 0.05 * (rng.standard_normal((k, k)) + 1j * rng.standard_normal((k, k)))
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    kdim = torch.tensor(ks, dtype=torch.int32, device="cuda")
    ws = torch.empty(_lib.call("cirr_gen_eig_ws_bytes", kmax, nb), dtype=torch.uint8, device="cuda")
    lam = torch.zeros((nb, kmax), dtype=torch.complex128, device="cuda")
    info = torch.zeros(nb, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    _lib.call("cirr_gen_eig_values", At.data_ptr(), Bt.data_ptr(), kdim.data_ptr(), kmax, nb, ws.data_ptr(),
              lam.data_ptr(), info.data_ptr(), st)
    assert (info.cpu().numpy() == 0).all()
    lh = lam.cpu().numpy()
    sel = np.zeros((nb, kmax), np.int32)
    cnt = np.array(ks, np.int32)
    for b, k in enumerate(ks):
        w = sla.eig(A[b, :k, :k], B[b, :k, :k], right=False)
        w = w[np.lexsort((w.imag, w.real))]
        got = lh[b, :k]
        # nearest matching (conjugate-free random matrices: sorted order is stable)
        assert np.abs(got - w).max() <= 1e-10 * np.abs(w).max(), (b, np.abs(got - w).max())
        sel[b, :k] = np.arange(k)
    smax = kmax
    scr = torch.empty(_lib.call("cirr_gen_eig_vec_scratch_bytes", kmax, nb, smax), dtype=torch.uint8, device="cuda")
    S = torch.zeros((nb, kmax, smax), dtype=torch.complex128, device="cuda")
    sel_t, cnt_t = torch.from_numpy(sel).cuda(), torch.from_numpy(cnt).cuda()
    _lib.call("cirr_gen_eig_vectors", ws.data_ptr(), kdim.data_ptr(), kmax, nb, lam.data_ptr(), sel_t.data_ptr(),
              cnt_t.data_ptr(), smax, scr.data_ptr(), S.data_ptr(), smax, kmax * smax, st)
    s = S.cpu().numpy()
    for b, k in enumerate(ks):
        x = s[b, :k, :k]
        l = lh[b, :k]
        a, bb = A[b, :k, :k], B[b, :k, :k]
        r = np.linalg.norm(a @ x - (bb @ x) * l[None, :], axis=0) / (
            np.linalg.norm(a @ x, axis=0) + np.abs(l) * np.linalg.norm(bb @ x, axis=0))
        assert r.max() < 1e-12, (b, r.max())
        assert np.allclose(np.linalg.norm(x, axis=0), 1.0)
