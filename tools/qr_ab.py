"""A/B of the eigenvalue QR sweeps: wavefront (default) vs windowed
(CIRR_QR_WINDOW=1) on random non-Hermitian pencils; eigenvalue agreement and time."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_01927_b200 import _lib  # noqa: E402


def run(k, nprob, window, seed, reps=3):
    os.environ["CIRR_QR_WINDOW"] = "1" if window else "0"
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((nprob, k, k)) + 1j * rng.standard_normal((nprob, k, k))
    B = np.eye(k) + 0.05 * (rng.standard_normal((nprob, k, k)) + 1j * rng.standard_normal((nprob, k, k)))
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(np.ascontiguousarray(B)).cuda()
    kd = torch.full((nprob,), k, dtype=torch.int32, device="cuda")
    ws = torch.empty(_lib.call("cirr_gen_eig_ws_bytes", k, nprob), dtype=torch.uint8, device="cuda")
    lam = torch.empty((nprob, k), dtype=torch.complex128, device="cuda")
    info = torch.zeros(nprob, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        _lib.call("cirr_gen_eig_values", At.data_ptr(), Bt.data_ptr(), kd.data_ptr(), k, nprob, ws.data_ptr(),
                  lam.data_ptr(), info.data_ptr(), st)
        e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    q = (ctypes.c_longlong * 8)()
    _lib.call("cirr_gen_eig_qr_stats", ctypes.addressof(q))
    return lam.cpu().numpy(), info.cpu().numpy(), min(ts), list(q[:8]), A, B


if __name__ == "__main__":
    for k in (8, 33, 120, 200, 256):
        for seed in (0, 1):
            lw, iw, tw, qw, A, B = run(k, 2, True, seed)
            lf, iff, tf, qf, _, _ = run(k, 2, False, seed)
            ref = np.sort_complex(np.linalg.eigvals(np.linalg.solve(B[0], A[0])))
            same = np.array_equal(lw, lf)
            d = np.max(np.abs(lw - lf) / np.maximum(np.abs(lw), 1e-300))
            e = np.max(np.abs(np.sort_complex(lf[0]) - ref) / np.abs(ref))
            print(f"k={k} seed={seed}: window {tw:.2f} ms (sw {qw[0]} rot {qw[1]} chain {qw[3]/1e6:.1f}M far {qw[4]/1e6:.1f}M) "
                  f"wavefront {tf:.2f} ms (sw {qf[0]} rot {qf[1]} chain {qf[3]/1e6:.1f}M tail {qf[4]/1e6:.1f}M) "
                  f"bitwise={same} maxrel={d:.1e} vs numpy {e:.1e} info {iw} {iff}", flush=True)
