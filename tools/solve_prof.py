"""Time one K3 solve pass (config-4 shaped: n=4096, 64 pencils, K RHS) and
optionally profile it: python tools/solve_prof.py [n] [P] [K] [reps]."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_01927_b200 import _lib  # noqa: E402


def main(n=4096, P=64, K=118, reps=3):
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
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for r in range(reps):
        torch.cuda.synchronize()
        e0.record()
        _lib.call("cirr_zgetrs_batched", pen.data_ptr(), n, n, n * n, P, perm.data_ptr(), R.data_ptr(), K, n * K,
                  rhs_of.data_ptr(), K, Y.data_ptr(), K, n * K, dinv.data_ptr(), st)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        print(f"solve n={n} P={P} K={K}: {t:.2f} ms  {P * 8.0 * n * n * K / (t / 1e3) / 1e12:.2f} TF/s", flush=True)
    # accuracy: || P M y - r || / (||M|| ||y||) on pencil 0 (CPU, complex128)
    j = 0
    m = z[j].item() * np.asarray(b.cpu()) - np.asarray(a.cpu())
    y = Y[j].cpu().numpy()
    r = R[0].cpu().numpy()
    res = np.linalg.norm(m @ y - r) / (np.linalg.norm(m) * np.linalg.norm(y))
    print(f"relative residual pencil0: {res:.3e}")


if __name__ == "__main__":
    main(*[int(x) for x in sys.argv[1:]])
