"""Shift hints for the eigenvalue QR: unhinted vs hinted (hints = the true
eigenvalues perturbed by 1e-10 relative, plus 10 % spurious random values);
eigenvalue agreement, sweeps and time."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_01927_b200 import _lib  # noqa: E402


def run(A, B, hint=None, reps=3):
    nprob, k, _ = A.shape
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(np.ascontiguousarray(B)).cuda()
    kd = torch.full((nprob,), k, dtype=torch.int32, device="cuda")
    ws = torch.empty(_lib.call("cirr_gen_eig_ws_bytes", k, nprob), dtype=torch.uint8, device="cuda")
    lam = torch.empty((nprob, k), dtype=torch.complex128, device="cuda")
    info = torch.zeros(nprob, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    if hint is not None:
        ht = torch.from_numpy(np.ascontiguousarray(hint)).cuda()
        hc = torch.full((nprob,), hint.shape[1], dtype=torch.int32, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        if hint is None:
            _lib.call("cirr_gen_eig_values", At.data_ptr(), Bt.data_ptr(), kd.data_ptr(), k, nprob, ws.data_ptr(),
                      lam.data_ptr(), info.data_ptr(), st)
        else:
            _lib.call("cirr_gen_eig_values_hinted", At.data_ptr(), Bt.data_ptr(), kd.data_ptr(), k, nprob,
                      ws.data_ptr(), lam.data_ptr(), info.data_ptr(), ht.data_ptr(), hc.data_ptr(), hint.shape[1], st)
        e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    q = (ctypes.c_longlong * 8)()
    _lib.call("cirr_gen_eig_qr_stats", ctypes.addressof(q))
    return lam.cpu().numpy(), info.cpu().numpy(), min(ts), q[0]


if __name__ == "__main__":
    for k in (120, 256):
        rng = np.random.default_rng(k)
        A = rng.standard_normal((2, k, k)) + 1j * rng.standard_normal((2, k, k))
        B = np.eye(k) + 0.05 * (rng.standard_normal((2, k, k)) + 1j * rng.standard_normal((2, k, k)))
        lam0, i0, t0, sw0 = run(A, B)
        ref = np.array([np.linalg.eigvals(np.linalg.solve(B[p], A[p])) for p in range(2)])
        hint = ref * (1 + 1e-10 * rng.standard_normal(ref.shape))
        nsp = k // 10
        hint[:, :nsp] = (rng.standard_normal((2, nsp)) + 1j * rng.standard_normal((2, nsp))) * np.abs(ref).mean()
        rng.shuffle(hint, axis=1)
        lam1, i1, t1, sw1 = run(A, B, hint)
        d = np.max(np.abs(lam1 - lam0) / np.abs(lam0))
        e = max(np.max(np.abs(np.sort_complex(lam1[p]) - np.sort_complex(ref[p])) / np.abs(np.sort_complex(ref[p])))
                for p in range(2))
        print(f"k={k}: unhinted {t0:.2f} ms ({sw0} sweeps)  hinted {t1:.2f} ms ({sw1} sweeps)  "
              f"max rel diff {d:.1e}  vs numpy {e:.1e}  info {i0} {i1}", flush=True)
