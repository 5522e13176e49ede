"""Time the device Krylov scouts: one LU of -A plus
k_iters single-RHS solves and the CGS2 re-orthogonalisation, on config 3
(n = 2304) and config 4 (n = 4096, dense).  The reference scout's CPU time on
config 3 comes from tests/golden/ref_scout.npz (SuperLU, measured in the build
container when the fixture was made); config 4 is dense (16.7M nonzeros), where
the reference's SuperLU path is impractical.  Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2511_01927_b200 import DevicePencil, scouting
    from paper_2511_01927_b200 import workloads as W
    g = np.load(os.path.join(ROOT, "tests", "golden", "ref_scout.npz"))
    out = {"metric": "scout wall time (LU of -A + k_iters solves)", "unit": "s", "rows": []}
    for name, mats, k, m in (("config3", W.config3_matrices(), 100, 32), ("config4", W.config4_matrices(), 100, 32)):
        dp = DevicePencil(*mats)
        for method in scouting.SCOUT_METHODS:
            scouting.scout(dp, method, k, m, seed=3)      # warm-up
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            est = scouting.scout(dp, method, k, m, seed=3)
            torch.cuda.synchronize()
            t = time.perf_counter() - t0
            row = {"problem": name, "n": dp.n, "method": method, "k_iters": k, "m": m, "gpu_s": round(t, 4)}
            if name == "config3":
                row["reference_cpu_s_build_container"] = round(float(g[f"cfg3_{method}_elapsed"]), 4)
                row["max_rel_diff_vs_reference"] = float(np.max(np.abs(est.ritz_values - g[f"cfg3_{method}"])
                                                               / np.abs(g[f"cfg3_{method}"])))
            out["rows"].append(row)
        del dp
    print(json.dumps(out))


if __name__ == "__main__":
    main()
