"""Time the cooperative latency-bound kernels (Hessenberg reduction inside
cirr_gen_eig_values, K4 cirr_orth) under CTA caps (cirr_set_coop_ctas)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from paper_2511_01927_b200 import _lib  # noqa: E402
import eig_bench  # noqa: E402
import qr_hint_ab  # noqa: E402

for cap in (0, 148, 96, 64, 32):
    old = _lib.call("cirr_set_coop_ctas", cap)
    out = []
    for k in (120, 256):
        rng = np.random.default_rng(k)
        A = rng.standard_normal((2, k, k)) + 1j * rng.standard_normal((2, k, k))
        B = np.eye(k) + 0.05 * (rng.standard_normal((2, k, k)) + 1j * rng.standard_normal((2, k, k)))
        lam, info, t, sw = qr_hint_ab.run(A, B)
        out.append(f"gen_eig k={k} {t:.2f} ms")
    print(f"cap={cap}: " + ", ".join(out), flush=True)
    eig_bench.t_orth(4096, 256)
    _lib.call("cirr_set_coop_ctas", old)
