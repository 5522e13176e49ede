"""Can the latency-bound Rayleigh-Ritz kernels (K4 orth + K6 eigenvalues) hide
under the bulk solve GEMMs of another contour?  Times a K=118 solve pass over
64 pencils (low-priority stream), one orth(n x 118) + gen_eig_values(k=118)
(high-priority stream), alone and concurrently, for several cooperative caps.
python tools/overlap_bench.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_01927_b200 import _lib  # noqa: E402


def main(n=4096, P=64, K=118, c=118, nprob=1):
    rng = np.random.default_rng(0)
    g = rng.standard_normal((n, n)) / np.sqrt(n) + np.diag(rng.uniform(-2, 2, n))
    a = torch.from_numpy(g).cuda()
    b = torch.from_numpy(np.eye(n) + 0.05 * rng.standard_normal((n, n)) / np.sqrt(n)).cuda()
    z = torch.from_numpy(0.5 + 0.3 * np.exp(2j * np.pi * (np.arange(P) + 0.5) / P)).cuda()
    pen = torch.empty((P, n, n), dtype=torch.complex128, device="cuda")
    mx = torch.empty(P, dtype=torch.float64, device="cuda")
    ipiv = torch.empty((P, n), dtype=torch.int32, device="cuda")
    perm = torch.empty((P, n), dtype=torch.int32, device="cuda")
    mp = torch.empty(P, dtype=torch.float64, device="cuda")
    info = torch.empty(P, dtype=torch.int32, device="cuda")
    st0 = torch.cuda.current_stream().cuda_stream
    lws = torch.empty(_lib.call("cirr_zgetrf_ws_bytes", n, P), dtype=torch.uint8, device="cuda")
    dinv = torch.empty(_lib.call("cirr_diag_inv_bytes", n, P), dtype=torch.uint8, device="cuda")
    _lib.call("cirr_assemble", a.data_ptr(), b.data_ptr(), n, n, z.data_ptr(), P, pen.data_ptr(), n, n * n,
              mx.data_ptr(), st0)
    _lib.call("cirr_zgetrf_batched", pen.data_ptr(), n, n, n * n, P, ipiv.data_ptr(), perm.data_ptr(),
              mp.data_ptr(), info.data_ptr(), lws.data_ptr(), st0)
    _lib.call("cirr_diag_inverses", pen.data_ptr(), n, n, n * n, P, dinv.data_ptr(), st0)
    R = torch.from_numpy(rng.standard_normal((1, n, K)) + 1j * rng.standard_normal((1, n, K))).cuda()
    rhs_of = torch.zeros(P, dtype=torch.int32, device="cuda")
    Y = torch.empty((P, n, K), dtype=torch.complex128, device="cuda")
    # latency set inputs
    u = np.linalg.qr(rng.standard_normal((n, c)) + 1j * rng.standard_normal((n, c)))[0]
    m = (u * np.logspace(0, -11.5, c)) @ np.linalg.qr(rng.standard_normal((c, c)) + 0j)[0]
    W0 = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(m.T, (nprob, c, n)))).cuda()
    W = W0.clone()
    sig = torch.empty((nprob, c), dtype=torch.float64, device="cuda")
    order = torch.empty((nprob, c), dtype=torch.int32, device="cuda")
    kept = torch.empty(nprob, dtype=torch.int32, device="cuda")
    Qt = torch.empty((nprob, c, n), dtype=torch.complex128, device="cuda")
    ows = torch.empty(_lib.call("cirr_orth_ws_bytes", c, nprob), dtype=torch.uint8, device="cuda")
    sw = torch.zeros(1, dtype=torch.int32, device="cuda")
    A = rng.standard_normal((nprob, c, c)) + 1j * rng.standard_normal((nprob, c, c))
    B = np.eye(c) + 0.05 * (rng.standard_normal((nprob, c, c)) + 1j * rng.standard_normal((nprob, c, c)))
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(np.ascontiguousarray(B)).cuda()
    kd = torch.full((nprob,), c, dtype=torch.int32, device="cuda")
    gws = torch.empty(_lib.call("cirr_gen_eig_ws_bytes", c, nprob), dtype=torch.uint8, device="cuda")
    lam = torch.empty((nprob, c), dtype=torch.complex128, device="cuda")
    ginfo = torch.zeros(nprob, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()

    lo = torch.cuda.Stream(priority=0)
    hi = torch.cuda.Stream(priority=-1)

    def solve(s):
        _lib.call("cirr_zgetrs_batched", pen.data_ptr(), n, n, n * n, P, perm.data_ptr(), R.data_ptr(), K, n * K,
                  rhs_of.data_ptr(), K, Y.data_ptr(), K, n * K, dinv.data_ptr(), s.cuda_stream)

    def latency(s, reps=1, do_orth=True, do_eig=True):
        with torch.cuda.stream(s):
            for _ in range(reps):
                if do_orth:
                    W.copy_(W0)
                    _lib.call("cirr_orth", W.data_ptr(), n, c * n, n, c, nprob, 1e-12, sig.data_ptr(),
                              order.data_ptr(), kept.data_ptr(), Qt.data_ptr(), n, c * n, ows.data_ptr(),
                              sw.data_ptr(), s.cuda_stream)
                if do_eig:
                    _lib.call("cirr_gen_eig_values", At.data_ptr(), Bt.data_ptr(), kd.data_ptr(), c, nprob,
                              gws.data_ptr(), lam.data_ptr(), ginfo.data_ptr(), s.cuda_stream)

    def timed(fn_lo, fn_hi):
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record(lo)
        e[2].record(hi)
        if fn_lo:
            fn_lo(lo)
        if fn_hi:
            fn_hi(hi)
        e[1].record(lo)
        e[3].record(hi)
        torch.cuda.synchronize()
        t0 = min(e[0].elapsed_time(e[2]), 0.0)
        return e[0].elapsed_time(e[1]), e[2].elapsed_time(e[3]), max(e[0].elapsed_time(e[1]), e[0].elapsed_time(e[3])) - t0

    # correctness under concurrency: outputs of each side must not change
    _lib.call("cirr_set_coop_ctas", 0)
    timed(solve, None)
    Y_ref = Y.clone()
    timed(None, latency)
    lam_ref, Qt_ref, kept_ref = lam.clone(), Qt.clone(), kept.clone()
    for trial in range(3):
        Y.zero_(); lam.zero_(); Qt.zero_()
        timed(solve, latency)
        print(f"concurrent trial {trial}: Y equal {bool(torch.equal(Y, Y_ref))}, lam equal "
              f"{bool(torch.equal(lam, lam_ref))}, Qt equal {bool(torch.equal(Qt, Qt_ref))}, "
              f"kept {kept.item()} vs {kept_ref.item()}", flush=True)
    # LU of another batch concurrently with the latency set
    pen2 = pen.clone()
    _lib.call("cirr_assemble", a.data_ptr(), b.data_ptr(), n, n, z.data_ptr(), P, pen2.data_ptr(), n, n * n,
              mx.data_ptr(), st0)
    torch.cuda.synchronize()
    pen2_0 = pen2.clone()

    def lu2(s):
        with torch.cuda.stream(s):
            pen2.copy_(pen2_0)
        _lib.call("cirr_zgetrf_batched", pen2.data_ptr(), n, n, n * n, P, ipiv.data_ptr(), perm.data_ptr(),
                  mp.data_ptr(), info.data_ptr(), lws.data_ptr(), s.cuda_stream)
    timed(lu2, None)
    LU_ref = pen2.clone()
    for trial in range(2):
        for do_orth, do_eig in ((True, False), (False, True), (True, True)):
            lam.zero_(); Qt.zero_()
            timed(lu2, lambda s: latency(s, reps=3, do_orth=do_orth, do_eig=do_eig))
            print(f"LU-concurrent trial {trial} orth={do_orth} eig={do_eig}: LU equal "
                  f"{bool(torch.equal(pen2, LU_ref))}, lam equal {bool(torch.equal(lam, lam_ref))}, "
                  f"Qt equal {bool(torch.equal(Qt, Qt_ref))}", flush=True)
    for cap in (0,):
        _lib.call("cirr_set_coop_ctas", cap)
        for _ in range(2):
            s_alone = timed(solve, None)[0]
            l_alone = timed(None, latency)[1]
            s_both, l_both, wall = timed(solve, latency)
        print(f"cap={cap:3d}: solve alone {s_alone:6.2f} ms | latency set alone {l_alone:6.2f} ms | "
              f"together: solve {s_both:6.2f}, latency {l_both:6.2f}, span {wall:6.2f} ms "
              f"(serial {s_alone + l_alone:6.2f})", flush=True)
    # two solves back to back vs solve + 2 latency sets
    _lib.call("cirr_set_coop_ctas", 16)
    print("lam sample", lam[0, :3].cpu().numpy(), "kept", kept.cpu().numpy(), "ginfo", ginfo.cpu().numpy())


if __name__ == "__main__":
    main()
