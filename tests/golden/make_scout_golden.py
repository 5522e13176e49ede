"""Golden vectors for the device Krylov scouts from the
UNMODIFIED reference `cieig.scouting.scout` (scouting.py:153-180).

Run in the build container only (imports /root/reference/pkg/src):

    CIEIG_DISABLE_NUMBA=1 OPENBLAS_NUM_THREADS=1 python tests/golden/make_scout_golden.py

Output: ref_scout.npz --
  thermal20 pencil (CSR, the reference conftest's grf seed 11 problem) and its
  dense ground truth count m;
  for each method in SCOUT_METHODS:
    diag100_full_<method>   scout(diag(1..100), method, 100, 5, seed=0)
    diag100_part_<method>   scout(diag(1..100), method, 30, 3, seed=1)
    t20_<method>            scout(thermal20, method, 60, m, seed=2)
    cfg3_<method>           scout(config 3 pencil, method, 100, 32, seed=3)
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from cieig import problems as rp  # noqa: E402
from cieig.scouting import SCOUT_METHODS, scout  # noqa: E402
from cieig.sparse import MatrixPencil, SparseMatrix  # noqa: E402

from paper_2511_01927_b200 import workloads as W  # noqa: E402


def dense_pencil(a, b):
    return MatrixPencil(a=SparseMatrix.from_dense(a), b=SparseMatrix.from_dense(b), hermitian=True)


def main():
    out = {}
    grid = rp.Grid2D(20, 20)
    t20 = rp.assemble_thermal(rp.grf_sample(grid, 1.0, 0.1, 0.2, seed=11), 1.0)
    m20 = rp.target_count(t20.n)
    for nm, mat in (("a", t20.a), ("b", t20.b)):
        sp = mat.to_scipy().tocsr()
        out[f"t20_{nm}_indptr"], out[f"t20_{nm}_indices"], out[f"t20_{nm}_data"] = sp.indptr, sp.indices, sp.data
    out["t20_n"], out["t20_m"] = t20.n, m20
    diag = dense_pencil(np.diag(np.arange(1.0, 101.0)), np.eye(100))
    a3, b3 = W.config3_matrices()
    cfg3 = dense_pencil(a3, b3)
    for method in SCOUT_METHODS:
        out[f"diag100_full_{method}"] = scout(diag, method, 100, 5, seed=0).ritz_values
        out[f"diag100_part_{method}"] = scout(diag, method, 30, 3, seed=1).ritz_values
        out[f"t20_{method}"] = scout(t20, method, 60, m20, seed=2).ritz_values
        est = scout(cfg3, method, 100, 32, seed=3)
        out[f"cfg3_{method}"] = est.ritz_values
        out[f"cfg3_{method}_elapsed"] = est.elapsed
        print(method, "t20", out[f"t20_{method}"][:3], "cfg3 %.2fs" % est.elapsed, flush=True)
    np.savez_compressed(os.path.join(HERE, "ref_scout.npz"), **out)


if __name__ == "__main__":
    main()
