"""BASELINE config 2 (256 independent n=256 GEPs, 2 circles each, N=16, L=8,
M=4): one solve_multi_batch pass vs 256 solve_multi calls, CUDA-event timed,
with the counts checked against the oracle fixture.  Development driver."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2511_01927_b200 import Contour, DevicePencil, SolverConfig, solve_multi, solve_multi_batch  # noqa: E402
from paper_2511_01927_b200 import solvers as S  # noqa: E402
from paper_2511_01927_b200 import workloads as W  # noqa: E402


def main(reps: int = 3, seq: bool = True):
    import torch
    fix = np.load(os.path.join(ROOT, "tests", "golden", "oracle_config2.npz"))
    ng = int(fix["n_gep"])
    mats = [W.config2_matrices(s) for s in range(ng)]
    cons = [[Contour.from_json_dict(d) for d in json.loads(str(fix[f"s{s}_contours"]))] for s in range(ng)]
    cfg = SolverConfig(n_q=16, source_cols=8, n_moments=4)
    dps = [DevicePencil(a, b, hermitian=True) for a, b in mats]
    want = [[len(fix[f"s{s}_c{i}_eigs"]) for i in range(len(cons[s]))] for s in range(ng)]
    out = {}
    for r in range(reps):
        timer = S.StageTimer()
        S.set_stage_timer(timer)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = time.perf_counter()
        e0.record()
        ms = solve_multi_batch(dps, cons, cfg)
        e1.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t
        S.set_stage_timer(None)
        got = [[0 if x is None else len(x.eigenvalues) for x in m.results] for m in ms]
        pairs = sum(map(sum, got))
        passes = sum(x.stats.iterations for m in ms for x in m.results if x is not None)
        out[f"batch_rep{r}"] = {"wall_s": wall, "gpu_s": e0.elapsed_time(e1) / 1e3, "pairs": pairs,
                                "counts_equal_oracle": got == want, "contour_passes": passes,
                                "stages_ms": {k: round(v, 2) for k, v in timer.totals().items()}}
        print(json.dumps(out[f"batch_rep{r}"]), flush=True)
    if seq:
        for r in range(2):
            torch.cuda.synchronize()
            t = time.perf_counter()
            ms = [solve_multi(dps[s], cons[s], cfg, seed=0) for s in range(ng)]
            torch.cuda.synchronize()
            wall = time.perf_counter() - t
            got = [[0 if x is None else len(x.eigenvalues) for x in m.results] for m in ms]
            out[f"seq_rep{r}"] = {"wall_s": wall, "counts_equal_oracle": got == want}
            print(json.dumps(out[f"seq_rep{r}"]), flush=True)
    best = min(v["wall_s"] for k, v in out.items() if k.startswith("batch"))
    pairs = out["batch_rep0"]["pairs"]
    summary = {"config": 2, "n_gep": ng, "batch_wall_s": best, "time_per_gep_ms": best / ng * 1e3,
               "eigenpairs_per_s": pairs / best,
               "shifted_solves_per_s": 16 * out["batch_rep0"]["contour_passes"] / best}
    if seq:
        summary["seq_wall_s"] = min(out["seq_rep0"]["wall_s"], out["seq_rep1"]["wall_s"])
    print(json.dumps(summary), flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 3, "--no-seq" not in sys.argv)
