"""Which kernel corrupts a concurrent K=121 TMA solve?  Runs the solve on a
low-priority stream next to one kernel family at a time on a high-priority
stream and compares the solve output with an idle-device run (bitwise)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_01927_b200 import _lib  # noqa: E402


def main(n=4096, P=64, K=int(os.environ.get("KCOLS", "121"))):
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
    k = 121
    Q = torch.from_numpy(np.linalg.qr(rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k)))[0]).cuda()
    Qt = Q.T.contiguous()
    AQ = torch.empty((n, k), dtype=torch.complex128, device="cuda")
    At = torch.empty((k, k), dtype=torch.complex128, device="cuda")
    Q2 = torch.empty((n, k), dtype=torch.complex128, device="cuda")
    # small eigenproblem inputs (one contour)
    A = rng.standard_normal((1, k, k)) + 1j * rng.standard_normal((1, k, k))
    B = np.eye(k) + 0.05 * (rng.standard_normal((1, k, k)) + 1j * rng.standard_normal((1, k, k)))
    Atl, Btl = torch.from_numpy(A).cuda(), torch.from_numpy(np.ascontiguousarray(B)).cuda()
    kd = torch.full((1,), k, dtype=torch.int32, device="cuda")
    gws = torch.empty(_lib.call("cirr_gen_eig_ws_bytes", k, 1), dtype=torch.uint8, device="cuda")
    lam = torch.empty((1, k), dtype=torch.complex128, device="cuda")
    ginfo = torch.zeros(1, dtype=torch.int32, device="cuda")
    sel = torch.arange(k, dtype=torch.int32, device="cuda").reshape(1, k)
    cnt = torch.full((1,), k, dtype=torch.int32, device="cuda")
    scr = torch.empty(_lib.call("cirr_gen_eig_vec_scratch_bytes", k, 1, k), dtype=torch.uint8, device="cuda")
    Sin = torch.zeros((1, k, k), dtype=torch.complex128, device="cuda")
    c = 123
    W0 = torch.from_numpy(rng.standard_normal((1, c, n)) + 1j * rng.standard_normal((1, c, n))).cuda()
    W = W0.clone()
    sig = torch.empty((1, c), dtype=torch.float64, device="cuda")
    order = torch.empty((1, c), dtype=torch.int32, device="cuda")
    kept = torch.empty(1, dtype=torch.int32, device="cuda")
    Qo = torch.zeros((1, c, n), dtype=torch.complex128, device="cuda")
    ows = torch.empty(_lib.call("cirr_orth_ws_bytes", c, 1), dtype=torch.uint8, device="cuda")
    sw = torch.zeros(1, dtype=torch.int32, device="cuda")
    res = torch.zeros((1, k), dtype=torch.float64, device="cuda")
    lamr = torch.ones((1, k), dtype=torch.complex128, device="cuda")

    def gen_vals(s):
        _lib.call("cirr_gen_eig_values", Atl.data_ptr(), Btl.data_ptr(), kd.data_ptr(), k, 1, gws.data_ptr(),
                  lam.data_ptr(), ginfo.data_ptr(), s.cuda_stream)

    def gen_vecs(s):
        gen_vals(s)
        _lib.call("cirr_gen_eig_vectors", gws.data_ptr(), kd.data_ptr(), k, 1, lam.data_ptr(), sel.data_ptr(),
                  cnt.data_ptr(), k, scr.data_ptr(), Sin.data_ptr(), k, k * k, s.cuda_stream)

    def orth(s):
        W.copy_(W0)
        _lib.call("cirr_orth", W.data_ptr(), n, c * n, n, c, 1, 1e-12, sig.data_ptr(), order.data_ptr(),
                  kept.data_ptr(), Qo.data_ptr(), n, c * n, ows.data_ptr(), sw.data_ptr(), s.cuda_stream)

    def resid(s):
        _lib.call("cirr_residuals", AQ.data_ptr(), Q2.data_ptr(), k, n * k, n, lamr.data_ptr(), k, cnt.data_ptr(),
                  k, 1, res.data_ptr(), k, s.cuda_stream)

    torch.cuda.synchronize()
    lo = torch.cuda.Stream(priority=0)
    hi = torch.cuda.Stream(priority=int(os.environ.get("HI_PRIO", "-1")))

    def solve(s):
        _lib.call("cirr_zgetrs_batched", pen.data_ptr(), n, n, n * n, P, perm.data_ptr(), R.data_ptr(), K, n * K,
                  rhs_of.data_ptr(), K, Y.data_ptr(), K, n * K,
                  0 if os.environ.get("NO_DINV") else dinv.data_ptr(), s.cuda_stream)

    fams = {
        "gemm_real_A": lambda s: _lib.call("cirr_gemm", 2, n, k, n, 1, a.data_ptr(), n, 0, Q.data_ptr(), k, 0,
                                           AQ.data_ptr(), k, 0, 1.0, 0, s.cuda_stream),
        "gemm_conj": lambda s: _lib.call("cirr_gemm", 1, k, k, n, 1, Qt.data_ptr(), n, 0, AQ.data_ptr(), k, 0,
                                         At.data_ptr(), k, 0, 1.0, 0, s.cuda_stream),
        "gemm_cplx": lambda s: _lib.call("cirr_gemm", 0, n, k, k, 1, Q.data_ptr(), k, 0, At.data_ptr(), k, 0,
                                         Q2.data_ptr(), k, 0, 1.0, 0, s.cuda_stream),
        "transpose": lambda s: _lib.call("cirr_transpose", 0, Qt.data_ptr(), n, k * n, k, n, 1, Q2.data_ptr(), k,
                                         n * k, s.cuda_stream),
        "torch_ops": lambda s: [Q2.copy_(Q), Q2.zero_(), torch.zeros_like(Q2).copy_(Q)],
        "gen_vals": gen_vals,
        "gen_vecs": gen_vecs,
        "orth": orth,
        "resid": resid,
    }
    solve(lo)
    torch.cuda.synchronize()
    Y_ref = Y.clone()
    # same stream, no concurrency: does resid touch Y?
    Y_keep = Y.clone()
    with torch.cuda.stream(lo):
        for _ in range(30):
            resid(lo)
    torch.cuda.synchronize()
    print("resid after solve on the same stream: Y unchanged", bool(torch.equal(Y, Y_keep)), flush=True)
    # concurrency with a torch elementwise kernel that only spins on its own buffer
    junk = torch.zeros(1 << 20, dtype=torch.float64, device="cuda")
    bad = 0
    for trial in range(4):
        Y.zero_()
        torch.cuda.synchronize()
        solve(lo)
        with torch.cuda.stream(hi):
            for _ in range(300):
                junk.add_(1.0)
        torch.cuda.synchronize()
        bad += int(not torch.equal(Y, Y_ref))
    print(f"junk adds   : solve differs in {bad}/4 trials", flush=True)
    if os.environ.get("LU_TEST"):
        pen0 = pen.clone()
        small = 12  # pencils
        def lu(s):
            with torch.cuda.stream(s):
                pen[:small].copy_(pen0[:small])
            _lib.call("cirr_zgetrf_batched", pen.data_ptr(), n, n, n * n, small, ipiv.data_ptr(), perm.data_ptr(),
                      mp.data_ptr(), info.data_ptr(), lws.data_ptr(), s.cuda_stream)
        lu(lo)
        torch.cuda.synchronize()
        ref = pen[:small].clone()
        for trial in range(3):
            lu(lo)
            with torch.cuda.stream(hi):
                for _ in range(200):
                    resid(hi)
            torch.cuda.synchronize()
            d = (pen[:small] != ref).any(dim=2).any(dim=1).cpu().numpy()
            print(f"LU with resid: differs {not torch.equal(pen[:small], ref)}; pencils {np.nonzero(d)[0]}", flush=True)
        return
    if os.environ.get("SLEEP_TEST"):
        sl = [torch.cuda.Stream(priority=0) for _ in range(16)]
        for trial in range(3):
            Y.zero_()
            torch.cuda.synchronize()
            solve(lo)
            for _ in range(20):
                for s_ in sl:
                    with torch.cuda.stream(s_):
                        torch.cuda._sleep(100000)
            torch.cuda.synchronize()
            print(f"sleep kernels: solve differs {not torch.equal(Y, Y_ref)}", flush=True)
        return
    only = os.environ.get("ONLY")
    for name, fn in fams.items():
        if only and name != only:
            continue
        bad = 0
        for trial in range(4):
            Y.zero_()
            torch.cuda.synchronize()
            solve(lo)
            with torch.cuda.stream(hi):
                for _ in range(30 if name not in ("gen_vals", "gen_vecs", "orth") else 3):
                    fn(hi)
            torch.cuda.synchronize()
            bad += int(not torch.equal(Y, Y_ref))
            if not torch.equal(Y, Y_ref) and name == "resid" and trial == 0:
                d = (Y - Y_ref).abs().cpu().numpy() > 0
                pb, rr_, cc_ = np.nonzero(d)
                rows_bad = np.nonzero(d.any(axis=(0, 2)))[0]
                print(f"  first bad row {rows_bad.min()}, rows with diffs {len(rows_bad)}", flush=True)
                print(f"  diff entries {d.sum()}; pencils {np.unique(pb)[:20]} ({len(np.unique(pb))}); rows "
                      f"{rr_.min()}..{rr_.max()}; cols {cc_.min()}..{cc_.max()}", flush=True)
                D = (Y - Y_ref).abs().cpu().numpy()
                Yr = Y_ref.abs().cpu().numpy()
                for p_ in np.unique(pb)[:4]:
                    rws = np.nonzero(d[p_].any(axis=1))[0]
                    for r_ in rws[:4]:
                        cols = np.nonzero(d[p_, r_])[0]
                        print(f"    pencil {p_} row {r_}: cols {cols.min()}..{cols.max()} ({len(cols)}), "
                              f"max|d| {D[p_, r_].max():.3e} vs |y| {Yr[p_, r_].max():.3e}", flush=True)
                for p_ in np.unique(pb)[:0]:
                    m = d[p_]
                    rows = np.nonzero(m.any(axis=1))[0]
                    print(f"  pencil {p_}: rows {rows.min()}..{rows.max()} ({len(rows)} rows), first rows {rows[:10]}",
                          flush=True)
        print(f"{name:12s}: solve differs in {bad}/4 trials", flush=True)


if __name__ == "__main__":
    main()
