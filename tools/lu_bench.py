"""Time the batched LU (K1+K2) and one solve pass (K3) on config-4-sized pencils."""
import sys
import os
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_01927_b200 import _lib  # noqa: E402


def main(n=4096, P=128, reps=3, K=32):
    rng = np.random.default_rng(0)
    a = torch.from_numpy(rng.standard_normal((n, n))).cuda()
    b = torch.from_numpy(np.eye(n) + 0.05 * rng.standard_normal((n, n)) / np.sqrt(n)).cuda()
    z = torch.from_numpy(0.5 + 0.3 * np.exp(2j * np.pi * (np.arange(P) + 0.5) / P)).cuda()
    pen = torch.empty((P, n, n), dtype=torch.complex128, device="cuda")
    mx = torch.empty(P, dtype=torch.float64, device="cuda")
    ipiv = torch.empty((P, n), dtype=torch.int32, device="cuda")
    perm = torch.empty((P, n), dtype=torch.int32, device="cuda")
    mp = torch.empty(P, dtype=torch.float64, device="cuda")
    info = torch.empty(P, dtype=torch.int32, device="cuda")
    R = torch.from_numpy(rng.standard_normal((1, n, K)) + 0j).cuda()
    rhs_of = torch.zeros(P, dtype=torch.int32, device="cuda")
    Y = torch.empty((P, n, K), dtype=torch.complex128, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    lws = torch.empty(_lib.call("cirr_zgetrf_ws_bytes", n, P), dtype=torch.uint8, device="cuda")
    dinv = torch.empty(_lib.call("cirr_diag_inv_bytes", n, P), dtype=torch.uint8, device="cuda")
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for r in range(reps):
        e[0].record()
        _lib.call("cirr_assemble", a.data_ptr(), b.data_ptr(), n, n, z.data_ptr(), P, pen.data_ptr(), n, n * n,
                  mx.data_ptr(), st)
        e[1].record()
        _lib.call("cirr_zgetrf_batched", pen.data_ptr(), n, n, n * n, P, ipiv.data_ptr(), perm.data_ptr(),
                  mp.data_ptr(), info.data_ptr(), lws.data_ptr(), st)
        _lib.call("cirr_diag_inverses", pen.data_ptr(), n, n, n * n, P, dinv.data_ptr(), st)
        e[2].record()
        _lib.call("cirr_zgetrs_batched", pen.data_ptr(), n, n, n * n, P, perm.data_ptr(), R.data_ptr(), K, n * K,
                  rhs_of.data_ptr(), K, Y.data_ptr(), K, n * K, dinv.data_ptr(), st)
        e[3].record()
        torch.cuda.synchronize()
        t_as, t_lu, t_s = e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), e[2].elapsed_time(e[3])
        lu_tf = P * 8 * n**3 / 3 / (t_lu / 1e3) / 1e12
        s_tf = P * 8 * n * n * K / (t_s / 1e3) / 1e12
        print(f"rep{r}: assemble {t_as:.2f} ms ({P * n * n * 16 / t_as / 1e6:.0f} GB/s)  LU {t_lu:.1f} ms "
              f"({lu_tf:.2f} TF/s)  solve K={K} {t_s:.1f} ms ({s_tf:.2f} TF/s)", flush=True)
    print("info", int(info.abs().max().item()))


if __name__ == "__main__":
    args = [int(x) for x in sys.argv[1:]]
    main(*args)
