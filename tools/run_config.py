"""Run one BASELINE config through the GPU solve_multi and compare with the
oracle fixture (tests/golden/oracle_configN.npz) -- a development driver."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2511_01927_b200 import Contour, DevicePencil, SolverConfig, solve_multi  # noqa: E402
from paper_2511_01927_b200 import solvers as S  # noqa: E402
from paper_2511_01927_b200 import workloads as W  # noqa: E402


def load(cfgno):
    path = os.path.join(ROOT, "tests", "golden", f"oracle_config{cfgno}.npz")
    return np.load(path) if os.path.exists(path) else None


def main(cfgno: int, reps: int = 2):
    import torch
    g = load(cfgno)
    if cfgno == 1:
        a, b = W.config1_matrices()
    elif cfgno == 3:
        a, b = W.config3_matrices()
    elif cfgno == 4:
        a, b = W.config4_matrices()
    elif cfgno == 5:
        a, b = W.config5_matrices()
    herm = cfgno != 4
    if g is not None:
        contours = [Contour.from_json_dict(d) for d in json.loads(str(g["contours"]))]
    else:
        contours = W.config4().contours
    nq, L, M = {1: (32, 16, 4), 3: (32, 32, 4), 4: (64, 32, 8), 5: (32, 64, 4)}[cfgno]
    cfg = SolverConfig(n_q=nq, source_cols=L, n_moments=M)
    dp = DevicePencil(a, b, hermitian=herm)
    for r in range(reps):
        timer = S.StageTimer()
        S.set_stage_timer(timer)
        torch.cuda.synchronize()
        t = time.perf_counter()
        m = solve_multi(dp, contours, cfg, seed=0)
        torch.cuda.synchronize()
        el = time.perf_counter() - t
        S.set_stage_timer(None)
        st = {k: round(v, 2) for k, v in timer.totals().items()}
        print(f"config{cfgno} rep{r}: {el:.3f}s stages(ms)={st}", flush=True)
    for i, (res, err) in enumerate(zip(m.results, m.errors)):
        line = f"  c{i}: "
        if res is None:
            line += f"error {err!r}"
        else:
            line += (f"{len(res.eigenvalues)} pairs, iters {res.stats.iterations}, "
                     f"max res {res.residuals.max():.2e}")
            if g is not None and f"c{i}_eigs" in g:
                ref = g[f"c{i}_eigs"]
                truth = g[f"c{i}_truth"]
                line += f" | oracle {len(ref)} truth {len(truth)} iters {int(g[f'c{i}_iters'])}"
                if len(ref) == len(res.eigenvalues):
                    # nearest matching (complex eigenvalues need not share the sort order)
                    got = np.asarray(res.eigenvalues, complex)
                    rel = np.array([np.min(np.abs(got - r)) / abs(r) for r in np.asarray(ref, complex)])
                    line += f" max rel diff {rel.max():.2e}"
        print(line, flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]) if len(sys.argv) > 2 else 2)
