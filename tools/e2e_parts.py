"""Dev tool: where config 4's e2e time beyond the device step goes (host
numpy A, B -> DevicePencil, results back)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_01927_b200 import DevicePencil  # noqa: E402
from paper_2511_01927_b200 import workloads as W  # noqa: E402


def t(fn, reps=3):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        out.append(time.perf_counter() - t0)
    return sorted(out)[len(out) // 2] * 1e3


a, b = W.config4_matrices()
print("pencil (pageable, hermitian=False -> device check)", t(lambda: DevicePencil(a, b, hermitian=False)))
print("pencil (pageable, hermitian=True)", t(lambda: DevicePencil(a, b, hermitian=True)))
print("to(cuda) A only", t(lambda: torch.from_numpy(a).to("cuda")))
pa = torch.from_numpy(a).pin_memory()
print("pinned A to(cuda)", t(lambda: pa.to("cuda", non_blocking=True)))
print("pin_memory() A", t(lambda: torch.from_numpy(a).pin_memory()))
