"""Break down one scout: LU of -A, A^-1 (look-back TRSV), B products, GEMVs."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_01927_b200 import DevicePencil, scouting  # noqa: E402
from paper_2511_01927_b200 import workloads as W  # noqa: E402


def t(f, reps=20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


dp = DevicePencil(*W.config4_matrices())
scouting._Device(dp)
torch.cuda.synchronize()
t0 = time.perf_counter()
d = scouting._Device(dp)
torch.cuda.synchronize()
print(f"LU of -A (n={dp.n}): {(time.perf_counter() - t0) * 1e3:.1f} ms")
x = d.new()
x.real.normal_()
print(f"A^-1 x: {t(lambda: d.inv(x, True)):.3f} ms")
print(f"B x: {t(lambda: d.bmul(x)):.3f} ms")
Qt = torch.randn((101, dp.n), dtype=torch.complex128, device="cuda")
print(f"dots 100 x n: {t(lambda: d.dots(Qt, 100, x)):.3f} ms")
h = torch.randn((100, 1), dtype=torch.complex128, device="cuda")
print(f"sub_comb 100: {t(lambda: d.sub_comb(x, Qt, 100, h)):.3f} ms")
print(f"vdot (sync): {t(lambda: d.vdot(x, x)):.3f} ms")
