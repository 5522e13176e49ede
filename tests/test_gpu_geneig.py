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


def _refine(A, B, ks, W0, iters=8):
    nb, kmax = A.shape[0], A.shape[1]
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    kdim = torch.tensor(ks, dtype=torch.int32, device="cuda")
    W0h = torch.from_numpy(np.ascontiguousarray(np.conj(np.transpose(W0, (0, 2, 1))))).cuda()
    ws = torch.empty(_lib.call("cirr_gen_eig_refine_ws_bytes", kmax, nb), dtype=torch.uint8, device="cuda")
    lam = torch.zeros((nb, kmax), dtype=torch.complex128, device="cuda")
    S = torch.zeros((nb, kmax, kmax), dtype=torch.complex128, device="cuda")
    info = torch.zeros(nb, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    _lib.call("cirr_gen_eig_refine", At.data_ptr(), Bt.data_ptr(), kdim.data_ptr(), kmax, nb, W0h.data_ptr(), kmax,
              kmax * kmax, iters, ws.data_ptr(), lam.data_ptr(), S.data_ptr(), kmax, kmax * kmax, info.data_ptr(), st)
    return lam.cpu().numpy(), S.cpu().numpy(), info.cpu().numpy()


@pytest.mark.parametrize("ks,noise,nbad", [([3], 1e-3, 0), ([64, 60], 1e-4, 0), ([120, 112], 1e-3, 0),
                                            ([120, 118], 1e-7, 0), ([256, 200], 1e-4, 0), ([120, 112], 1e-6, 4),
                                            ([64, 64], 1e-5, 1), ([200, 150], 1e-6, 30)])
def test_gen_eig_refine(ks, noise, nbad):
    """Newton refinement of a perturbed eigenbasis (the refinement-round K6):
    eigenvalues equal to LAPACK's to 1e-12, unit eigenvectors with projected
    residuals at the rounding level, same (re, im) order as the QR path.
    nbad columns are mixtures of several eigenvectors (the unconverged Ritz
    pairs of a refinement round), which the block step has to sort out."""
    kmax, nb = max(ks), len(ks)
    rng = np.random.default_rng(7 * sum(ks))
    A = np.zeros((nb, kmax, kmax), complex)
    B = np.zeros((nb, kmax, kmax), complex)
    W0 = np.zeros((nb, kmax, kmax), complex)
    truth = []
    for b, k in enumerate(ks):
        A[b, :k, :k] = rng.standard_normal((k, k)) / np.sqrt(k) + np.diag(rng.uniform(-2, 2, k))
        B[b, :k, :k] = np.eye(k) + 0.05 * rng.standard_normal((k, k)) / np.sqrt(k)
        w, v = sla.eig(A[b, :k, :k], B[b, :k, :k])
        truth.append(w[np.lexsort((w.imag, w.real))])
        # an eigenbasis in scrambled order, columns scaled and perturbed
        perm = rng.permutation(k)
        pert = noise * (rng.standard_normal((k, k)) + 1j * rng.standard_normal((k, k)))
        W = v[:, perm] + pert
        if nbad:
            cols = rng.choice(k, size=min(nbad, k), replace=False)
            mix = rng.standard_normal((len(cols), len(cols))) + 1j * rng.standard_normal((len(cols), len(cols)))
            W[:, cols] = W[:, cols] @ mix + 0.3 * v @ (rng.standard_normal((k, len(cols))) / np.sqrt(k))
        W0[b, :k, :k] = W * rng.uniform(0.5, 2.0, k)[None, :]
    lh, s, info = _refine(A, B, ks, W0)
    assert (info == 0).all(), info
    for b, k in enumerate(ks):
        got = lh[b, :k]
        # real matrices: conjugate pairs share a real part, so the sorted order
        # within a pair is decided by rounding -- match nearest
        assert np.all(np.diff(got.real) >= 0)
        d = np.abs(got[:, None] - truth[b][None, :]).min(axis=1)
        assert d.max() <= 1e-12 * np.abs(truth[b]).max(), (b, d.max())
        x, a, bb = s[b, :k, :k], A[b, :k, :k], B[b, :k, :k]
        r = np.linalg.norm(a @ x - (bb @ x) * got[None, :], axis=0) / (
            np.linalg.norm(a @ x, axis=0) + np.abs(got) * np.linalg.norm(bb @ x, axis=0))
        assert r.max() < 1e-12, (b, r.max())
        assert np.allclose(np.linalg.norm(x, axis=0), 1.0)


def test_gen_eig_refine_reports_nonconvergence():
    """A basis that is not near an eigenbasis (random) or a singular one comes
    back as info = -1, so the caller falls back to the QR path."""
    k, nb = 48, 2
    rng = np.random.default_rng(5)
    A = rng.standard_normal((nb, k, k)) + 0j
    B = np.stack([np.eye(k, dtype=complex)] * nb)
    W0 = rng.standard_normal((nb, k, k)) + 1j * rng.standard_normal((nb, k, k))
    W0[1, :, 3] = W0[1, :, 2]       # singular basis
    _, _, info = _refine(A, B, [k, k], W0, iters=3)
    assert (info == -1).all(), info
