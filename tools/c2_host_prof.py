"""Host-side profile of one config-2 solve_multi_batch (256 GEPs): cProfile
of the Python orchestration, plus the device time of the same call."""
import cProfile
import json
import os
import pstats
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_01927_b200 import Contour, DevicePencil, SolverConfig, solve_multi_batch  # noqa: E402
from paper_2511_01927_b200 import solvers as S  # noqa: E402
from paper_2511_01927_b200 import workloads as W  # noqa: E402


def main():
    import torch
    fix = np.load(os.path.join(ROOT, "tests", "golden", "oracle_config2.npz"))
    ng = int(fix["n_gep"])
    mats = [W.config2_matrices(s) for s in range(ng)]
    cons = [[Contour.from_json_dict(d) for d in json.loads(str(fix[f"s{s}_contours"]))] for s in range(ng)]
    cfg = SolverConfig(n_q=16, source_cols=8, n_moments=4)
    dps = [DevicePencil(a, b, hermitian=True) for a, b in mats]
    for _ in range(2):
        solve_multi_batch(dps, cons, cfg)
    torch.cuda.synchronize()
    timer = S.StageTimer()
    S.set_stage_timer(timer)
    t = time.perf_counter()
    solve_multi_batch(dps, cons, cfg)
    torch.cuda.synchronize()
    print("wall with stage timer", time.perf_counter() - t, {k: round(v, 2) for k, v in timer.totals().items()})
    S.set_stage_timer(None)
    torch.cuda.synchronize()
    t = time.perf_counter()
    solve_multi_batch(dps, cons, cfg)
    torch.cuda.synchronize()
    print("wall", time.perf_counter() - t)
    pr = cProfile.Profile()
    pr.enable()
    solve_multi_batch(dps, cons, cfg)
    torch.cuda.synchronize()
    pr.disable()
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(35)


if __name__ == "__main__":
    main()
