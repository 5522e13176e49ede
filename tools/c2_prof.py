"""Host-side profile of one steady-state solve_multi_batch pass on config 2
(after one warm-up pass): top functions by own time and the callers of the
heaviest ones.  Development tool."""
import cProfile
import json
import os
import pstats
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2511_01927_b200 import Contour, DevicePencil, SolverConfig, solve_multi_batch  # noqa: E402
from paper_2511_01927_b200 import workloads as W  # noqa: E402

import torch  # noqa: E402

fix = np.load(os.path.join(ROOT, "tests", "golden", "oracle_config2.npz"))
ng = int(fix["n_gep"])
cons = [[Contour.from_json_dict(d) for d in json.loads(str(fix[f"s{s}_contours"]))] for s in range(ng)]
cfg = SolverConfig(n_q=16, source_cols=8, n_moments=4)
dps = [DevicePencil(*W.config2_matrices(s), hermitian=True) for s in range(ng)]
solve_multi_batch(dps, cons, cfg)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
solve_multi_batch(dps, cons, cfg)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
st.print_callers("getDeviceCount|builtins.compile|method 'cpu'")
