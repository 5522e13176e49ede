"""Dev tool: where the host time of one config-2 solve_multi_batch goes.
Wraps the engine's phases with wall-clock timers and torch.Tensor.cpu (the
device->host syncs) with a wait timer; wall - waits = host-bound time, during
which the GPU idles unless work is queued."""
import collections
import functools
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_01927_b200 import Contour, DevicePencil, SolverConfig, solve_multi_batch  # noqa: E402
from paper_2511_01927_b200 import solvers as S  # noqa: E402
from paper_2511_01927_b200 import workloads as W  # noqa: E402

T = collections.defaultdict(float)
N = collections.defaultdict(int)
WAIT = [0.0]
STACK = []


def wrap(owner, name, label=None):
    fn = getattr(owner, name)
    label = label or name

    @functools.wraps(fn)
    def inner(*a, **k):
        t = time.perf_counter()
        w0 = WAIT[0]
        STACK.append(label)
        try:
            return fn(*a, **k)
        finally:
            STACK.pop()
            dt = time.perf_counter() - t
            if not STACK or label.startswith("~"):  # top-level phases; "~" = nested, inclusive
                T[label] += dt
                T[label + " (waits)"] += WAIT[0] - w0
            N[label] += 1
    setattr(owner, name, inner)


def main():
    fix = np.load(os.path.join(ROOT, "tests", "golden", "oracle_config2.npz"))
    ng = int(fix["n_gep"])
    mats = [W.config2_matrices(s) for s in range(ng)]
    cons = [[Contour.from_json_dict(d) for d in json.loads(str(fix[f"s{s}_contours"]))] for s in range(ng)]
    cfg = SolverConfig(n_q=16, source_cols=8, n_moments=4)
    dps = [DevicePencil(a, b, hermitian=True) for a, b in mats]
    for _ in range(2):
        solve_multi_batch(dps, cons, cfg)
    torch.cuda.synchronize()
    orig_cpu = torch.Tensor.cpu

    def cpu(self, *a, **k):
        t = time.perf_counter()
        r = orig_cpu(self, *a, **k)
        WAIT[0] += time.perf_counter() - t
        return r
    torch.Tensor.cpu = cpu
    E = S._Engine
    for nm in ("factor", "apply", "rayleigh_ritz", "fetch_vectors", "finish", "source_blocks"):
        wrap(E, nm)
    wrap(S, "_multi_result")
    wrap(S, "_Contour", "_Contour.__init__")
    wrap(S, "_waves")
    wrap(S, "_hbm_budget")
    for nm in ("_alloc_factors", "_factor_range", "_live", "_bx"):
        wrap(E, nm, "~" + nm)
    for nm in ("contains_rows", "_pad_stack", "_gather", "_h2d", "_coef_batch", "_source_block"):
        wrap(S, nm, "~" + nm)
    wrap(S.DevicePencil, "assemble", "~assemble")
    wrap(S._lib, "call", "~_lib.call")
    t = time.perf_counter()
    w0 = WAIT[0]
    solve_multi_batch(dps, cons, cfg)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t
    print(f"wall {wall * 1e3:.1f} ms, waits in .cpu() {(WAIT[0] - w0) * 1e3:.1f} ms")
    acc = 0.0
    for k, v in sorted(T.items(), key=lambda x: -x[1]):
        print(f"  {k:32s} {v * 1e3:8.2f} ms  (calls {N.get(k, '')})")
        if "(waits)" not in k and not k.startswith("~"):
            acc += v
    print(f"  {'(other, in solve_multi_batch)':32s} {(wall - acc) * 1e3:8.2f} ms")


if __name__ == "__main__":
    main()
