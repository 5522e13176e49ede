"""Ozaki int8 GEMM update vs the DMMA trailing update at the LU's shapes (one B200).
Usage: python tools/ozaki_bench.py [m] [batch]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2511_01927_b200 import _lib

m = int(sys.argv[1]) if len(sys.argv) > 1 else 3584
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 16
W = 512
n = m + W
g = torch.Generator(device="cuda").manual_seed(0)
P = torch.randn((batch, n, n), dtype=torch.complex128, device="cuda", generator=g)
st = torch.cuda.current_stream().cuda_stream
base = P.data_ptr()
off = lambda r, c: base + 16 * (r * n + c)
ref = P.clone()
ref[:, W:, W:] -= P[:, W:, :W] @ P[:, :W, W:]


def run():
    rc = _lib.call("cirr_ozaki_zgemm_sub", off(W, 0), n, n * n, off(0, W), n, n * n, off(W, W), n, n * n, m, m, W,
                   batch, st)
    assert rc == 0


P0 = P.clone()
run()
torch.cuda.synchronize()
err = (P[:, W:, W:] - ref[:, W:, W:]).abs().max().item() / ref[:, W:, W:].abs().max().item()
print(f"m={m} batch={batch}: max rel err vs torch (cuBLAS) {err:.2e}")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(2):
    run()
e0.record()
reps = 5
for _ in range(reps):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
fl = 8.0 * m * m * W * batch
print(f"ozaki: {ms:.2f} ms per update of {batch} pencils, {fl / ms * 1e-9:.1f} TF/s FP64-equivalent")
C = P[:, W:, W:]
A = P[:, W:, :W].contiguous()
B = P[:, :W, W:].contiguous()
for _ in range(2):
    torch.baddbmm(C, A, B, alpha=-1.0)
e0.record()
for _ in range(reps):
    torch.baddbmm(C, A, B, alpha=-1.0)
e1.record()
torch.cuda.synchronize()
ms2 = e0.elapsed_time(e1) / reps
print(f"cuBLAS zgemm (baddbmm): {ms2:.2f} ms, {fl / ms2 * 1e-9:.1f} TF/s")
