"""Config 2 timing before/after a config-4 solve in the same process (the
bench runs config 2 after the config-4 steps).  Development driver."""
import gc
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2511_01927_b200 import Contour, DevicePencil, SolverConfig, solve_multi, solve_multi_batch  # noqa: E402
from paper_2511_01927_b200 import workloads as W  # noqa: E402


def c2(dps, cons, cfg, tag):
    import torch
    for r in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        solve_multi_batch(dps, cons, cfg)
        torch.cuda.synchronize()
        print(tag, r, round((time.perf_counter() - t) * 1e3, 2), "ms", flush=True)


def main():
    import torch
    fix = np.load(os.path.join(ROOT, "tests", "golden", "oracle_config2.npz"))
    ng = int(fix["n_gep"])
    mats = [W.config2_matrices(s) for s in range(ng)]
    cons = [[Contour.from_json_dict(d) for d in json.loads(str(fix[f"s{s}_contours"]))] for s in range(ng)]
    cfg = SolverConfig(n_q=16, source_cols=8, n_moments=4)
    dps = [DevicePencil(a, b, hermitian=True) for a, b in mats]
    c2(dps, cons, cfg, "fresh")
    a, b = W.config4_matrices()
    dp4 = DevicePencil(a, b, hermitian=False)
    solve_multi(dp4, W.config4().contours, SolverConfig(n_q=64, source_cols=32, n_moments=8), seed=0)
    del dp4
    c2(dps, cons, cfg, "after_c4")
    print("reserved GB", torch.cuda.memory_reserved() / 1e9, "gc counts", gc.get_count(), flush=True)
    gc.collect()
    c2(dps, cons, cfg, "after_gc")
    torch.cuda.empty_cache()
    c2(dps, cons, cfg, "after_empty_cache")


if __name__ == "__main__":
    main()
