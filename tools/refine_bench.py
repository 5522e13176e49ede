"""Dev tool: time the pieces of cirr_gen_eig_refine at refinement-round size
(k = 120, 2 problems) against the QR path."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_01927_b200 import _lib  # noqa: E402


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


def main(k=120, nb=2):
    st = torch.cuda.current_stream().cuda_stream
    rng = np.random.default_rng(0)
    kk = k * k
    A = torch.from_numpy(rng.standard_normal((nb, k, k)) + 1j * rng.standard_normal((nb, k, k))).cuda()
    B = torch.from_numpy(np.stack([np.eye(k)] * nb) + 0j).cuda()
    W = A.clone()
    C = torch.empty_like(A)
    ipiv = torch.empty((nb, k), dtype=torch.int32, device="cuda")
    perm = torch.empty_like(ipiv)
    minpiv = torch.empty(nb, dtype=torch.float64, device="cuda")
    info = torch.empty(nb, dtype=torch.int32, device="cuda")
    rhs = torch.arange(nb, dtype=torch.int32, device="cuda")
    p = lambda t: t.data_ptr()  # noqa: E731
    out = {}
    out["gemm"] = timeit(lambda: _lib.call("cirr_gemm", 0, k, k, k, nb, p(A), k, kk, p(W), k, kk, p(C), k, kk, 1.0, 0,
                                           st))

    def lu():
        W.copy_(A)
        _lib.call("cirr_zgetrf_batched", p(W), k, k, kk, nb, p(ipiv), p(perm), p(minpiv), p(info), None, st)
    out["copy+getrf"] = timeit(lu)
    out["getrs"] = timeit(lambda: _lib.call("cirr_zgetrs_batched", p(W), k, k, kk, nb, p(perm), p(A), k, kk, p(rhs), k,
                                            p(C), k, kk, None, st))
    # refine end to end with an exact eigenbasis (converges at the first step)
    Ah = A.cpu().numpy()
    W0 = np.stack([np.linalg.eig(Ah[b])[1] for b in range(nb)])
    W0h = torch.from_numpy(np.ascontiguousarray(np.conj(np.transpose(W0, (0, 2, 1))))).cuda()
    kdim = torch.full((nb,), k, dtype=torch.int32, device="cuda")
    ws = torch.empty(_lib.call("cirr_gen_eig_refine_ws_bytes", k, nb), dtype=torch.uint8, device="cuda")
    lam = torch.empty((nb, k), dtype=torch.complex128, device="cuda")
    S = torch.empty_like(A)
    for it in (1, 3, 6):
        out[f"refine it={it}"] = timeit(lambda: _lib.call(
            "cirr_gen_eig_refine", p(A), p(B), p(kdim), k, nb, p(W0h), k, kk, it, p(ws), p(lam), p(S), k, kk, p(info),
            st), reps=5)
    gws = torch.empty(_lib.call("cirr_gen_eig_ws_bytes", k, nb), dtype=torch.uint8, device="cuda")
    out["qr values"] = timeit(lambda: _lib.call("cirr_gen_eig_values", p(A), p(B), p(kdim), k, nb, p(gws), p(lam),
                                                p(info), st), reps=3)
    n0 = _lib.call("cirr_launch_count")
    _lib.call("cirr_gen_eig_refine", p(A), p(B), p(kdim), k, nb, p(W0h), k, kk, 6, p(ws), p(lam), p(S), k, kk, p(info),
              st)
    out["refine launches (it=6)"] = _lib.call("cirr_launch_count") - n0
    for kname, v in out.items():
        print(f"{kname:28s} {v:10.1f}", flush=True)


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
