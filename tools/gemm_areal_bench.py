"""Time the real-A products of Rayleigh-Ritz (A Q with A n x n real, Q n x k
complex, batch 2) on cirr_gemm (cp.async DMMA kernel, split-K)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_01927_b200 import _lib  # noqa: E402

n, k, nb = 4096, 121, 2
rng = np.random.default_rng(0)
A = torch.from_numpy(rng.standard_normal((n, n))).cuda()
Q = torch.from_numpy(rng.standard_normal((nb, n, k)) + 1j * rng.standard_normal((nb, n, k))).cuda()
C = torch.empty((nb, n, k), dtype=torch.complex128, device="cuda")
Qt = torch.from_numpy(rng.standard_normal((nb, k, n)) + 1j * rng.standard_normal((nb, k, n))).cuda()
G = torch.empty((nb, k, k), dtype=torch.complex128, device="cuda")
st = torch.cuda.current_stream().cuda_stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, f, fl in (("A Q (real A)", lambda: _lib.call("cirr_gemm", 2, n, k, n, nb, A.data_ptr(), n, 0, Q.data_ptr(), k,
                                                    n * k, C.data_ptr(), k, n * k, 1.0, 0, st), 4.0 * n * n * k * nb),
                    ("Q^H (AQ)", lambda: _lib.call("cirr_gemm", 1, k, k, n, nb, Qt.data_ptr(), n, k * n, C.data_ptr(), k,
                                                   n * k, G.data_ptr(), k, k * k, 1.0, 0, st), 8.0 * k * k * n * nb)):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10
    print(f"{name}: {t:.3f} ms  {fl / t / 1e9:.1f} TF/s", flush=True)
