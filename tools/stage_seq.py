"""Per-bracket stage times (in launch order) of one solve_multi on a BASELINE
config: which Rayleigh-Ritz round / solve pass costs what.  Development driver."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_01927_b200 import Contour, DevicePencil, SolverConfig, solve_multi  # noqa: E402
from paper_2511_01927_b200 import solvers as S  # noqa: E402
from paper_2511_01927_b200 import workloads as W  # noqa: E402


def main(cfgno=4):
    mk = {1: W.config1_matrices, 3: W.config3_matrices, 4: W.config4_matrices, 5: W.config5_matrices}[cfgno]
    a, b = mk()
    g = np.load(os.path.join(ROOT, "tests", "golden", f"oracle_config{cfgno}.npz"))
    cons = [Contour.from_json_dict(d) for d in json.loads(str(g["contours"]))] if "contours" in g else W.config4().contours
    nq, L, M = {1: (32, 16, 4), 3: (32, 32, 4), 4: (64, 32, 8), 5: (32, 64, 4)}[cfgno]
    cfg = SolverConfig(n_q=nq, source_cols=L, n_moments=M)
    dp = DevicePencil(a, b, hermitian=cfgno != 4)
    solve_multi(dp, cons, cfg, seed=0)
    t = S.StageTimer()
    S.set_stage_timer(t)
    solve_multi(dp, cons, cfg, seed=0)
    torch.cuda.synchronize()
    S.set_stage_timer(None)
    line = []
    for name, e0, e1 in t.events:
        line.append(f"{name}={e0.elapsed_time(e1):.2f}")
    print(" ".join(line))
    print({k: round(v, 2) for k, v in t.totals().items()})


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
