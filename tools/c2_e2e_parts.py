"""Dev tool: where config 2's e2e time beyond the device pass goes (256 host
numpy pencils -> DevicePencils, results back)."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_01927_b200 import Contour, DevicePencil, SolverConfig, solve_multi_batch  # noqa: E402
from paper_2511_01927_b200 import workloads as W  # noqa: E402


def t(fn, reps=3):
    out = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        out.append(time.perf_counter() - t0)
    return round(sorted(out)[len(out) // 2] * 1e3, 2)


class HostPencil:
    def __init__(self, a, b, hermitian):
        self.a, self.b, self.hermitian = a, b, hermitian


fix = np.load(os.path.join(ROOT, "tests", "golden", "oracle_config2.npz"))
ng = int(fix["n_gep"])
mats = [W.config2_matrices(s) for s in range(ng)]
cons = [[Contour.from_json_dict(d) for d in json.loads(str(fix[f"s{s}_contours"]))] for s in range(ng)]
cfg = SolverConfig(n_q=16, source_cols=8, n_moments=4)
dps = [DevicePencil(a, b, hermitian=True) for a, b in mats]
hps = [HostPencil(a, b, True) for a, b in mats]
solve_multi_batch(dps, cons, cfg)
print("device batch", t(lambda: solve_multi_batch(dps, cons, cfg)))
print("host batch", t(lambda: solve_multi_batch(hps, cons, cfg)))
print("256 DevicePencils", t(lambda: [DevicePencil(a, b, hermitian=True) for a, b in mats]))
print("np.stack", t(lambda: np.stack([m for ab in mats for m in ab])))
st = np.stack([m for ab in mats for m in ab])
print("stacked pageable to(cuda)", t(lambda: torch.from_numpy(st).to("cuda")))
pin = torch.empty(st.shape, dtype=torch.float64, pin_memory=True)
pv = pin.numpy()


def fill():
    for i, (a, b) in enumerate(mats):
        pv[2 * i] = a
        pv[2 * i + 1] = b


print("fill pinned", t(fill))
print("pinned to(cuda)", t(lambda: pin.to("cuda", non_blocking=True)))
print("pin_memory() of stack", t(lambda: torch.from_numpy(st).pin_memory()))
r = solve_multi_batch(dps, cons, cfg)


def touch():
    s = 0.0
    for m in r:
        for x in m.results:
            if x is not None:
                s += float(np.sum(np.abs(x.eigenvalues))) + float(x.eigenvectors.shape[1])
    return s


print("touch results", t(touch))
