"""Regression: a K3 solve must give bit-identical results while kernels of
another (higher-priority) stream share its SMs.  Before the proxy fence in
zgemm_sub_tma's stage release, co-resident CTAs slowed the shared-memory pipe
enough for the TMA refill to overtake a pending LDS (profiles/r01_pipeline_r01.txt)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_solve_bitwise_under_concurrent_kernels():
    import torch
    from paper_2511_01927_b200 import _lib

    n, P, K, k = 4096, 32, 121, 121
    rng = np.random.default_rng(0)
    a = torch.from_numpy(rng.standard_normal((n, n)) / np.sqrt(n) + np.diag(rng.uniform(-2, 2, n))).cuda()
    b = torch.from_numpy(np.eye(n) + 0.05 * rng.standard_normal((n, n)) / np.sqrt(n)).cuda()
    z = torch.from_numpy(0.5 + 0.3 * np.exp(2j * np.pi * (np.arange(P) + 0.5) / P)).cuda()
    pen = torch.empty((P, n, n), dtype=torch.complex128, device="cuda")
    mx = torch.empty(P, dtype=torch.float64, device="cuda")
    ipiv = torch.empty((P, n), dtype=torch.int32, device="cuda")
    perm = torch.empty((P, n), dtype=torch.int32, device="cuda")
    mp = torch.empty(P, dtype=torch.float64, device="cuda")
    info = torch.empty(P, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    lws = torch.empty(_lib.call("cirr_zgetrf_ws_bytes", n, P), dtype=torch.uint8, device="cuda")
    dinv = torch.empty(_lib.call("cirr_diag_inv_bytes", n, P), dtype=torch.uint8, device="cuda")
    _lib.call("cirr_assemble", a.data_ptr(), b.data_ptr(), n, n, z.data_ptr(), P, pen.data_ptr(), n, n * n,
              mx.data_ptr(), st)
    _lib.call("cirr_zgetrf_batched", pen.data_ptr(), n, n, n * n, P, ipiv.data_ptr(), perm.data_ptr(),
              mp.data_ptr(), info.data_ptr(), lws.data_ptr(), st)
    _lib.call("cirr_diag_inverses", pen.data_ptr(), n, n, n * n, P, dinv.data_ptr(), st)
    R = torch.from_numpy(rng.standard_normal((1, n, K)) + 1j * rng.standard_normal((1, n, K))).cuda()
    rhs_of = torch.zeros(P, dtype=torch.int32, device="cuda")
    Y = torch.empty((P, n, K), dtype=torch.complex128, device="cuda")
    AX = torch.from_numpy(rng.standard_normal((n, k)) + 0j).cuda()
    BX = torch.from_numpy(rng.standard_normal((n, k)) + 0j).cuda()
    lam = torch.ones((1, k), dtype=torch.complex128, device="cuda")
    cnt = torch.full((1,), k, dtype=torch.int32, device="cuda")
    res = torch.zeros((1, k), dtype=torch.float64, device="cuda")

    def solve(s):
        _lib.call("cirr_zgetrs_batched", pen.data_ptr(), n, n, n * n, P, perm.data_ptr(), R.data_ptr(), K, n * K,
                  rhs_of.data_ptr(), K, Y.data_ptr(), K, n * K, dinv.data_ptr(), s.cuda_stream)

    lo = torch.cuda.Stream(priority=0)
    hi = torch.cuda.Stream(priority=-1)
    torch.cuda.synchronize()
    solve(lo)
    torch.cuda.synchronize()
    ref = Y.clone()
    for _ in range(3):
        with torch.cuda.stream(lo):
            Y.zero_()
        solve(lo)
        for _ in range(40):  # strided-load kernel whose CTAs co-reside with the GEMM's
            _lib.call("cirr_residuals", AX.data_ptr(), BX.data_ptr(), k, n * k, n, lam.data_ptr(), k,
                      cnt.data_ptr(), k, 1, res.data_ptr(), k, hi.cuda_stream)
        torch.cuda.synchronize()
        assert torch.equal(Y, ref)
