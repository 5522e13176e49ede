"""Generate golden vectors from the UNMODIFIED reference package.

Run in the build container only (it imports /root/reference/pkg/src/cieig,
which does not exist on the GPU box):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py

Outputs (small, committed):
  ref_kats.npz      -- reference outputs on its own KAT problems
                       (pkg/tests/test_solvers.py:30-142, test_linalg.py)
  ref_thermal.npz   -- thermal10/thermal20 pencils (CSR) + reference CIRR,
                       projector and KDE-contour solve_multi outputs
  ref_grf.npz       -- reference grf_sample fields (pins workloads.grf_2d)
  ref_config2.npz   -- 8 config-2 GEPs solved by the reference solve_multi
                       with largest-gap contours
  ref_config3.npz   -- config 3 solved by the reference solve_multi
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import cieig  # noqa: E402
from cieig import contours as rc  # noqa: E402
from cieig import problems as rp  # noqa: E402
from cieig import solvers as rs  # noqa: E402
from cieig.sparse import MatrixPencil, SparseMatrix  # noqa: E402

from paper_2511_01927_b200 import workloads as W  # noqa: E402


def diag_pencil(da, db=None):
    a = np.diag(np.asarray(da, dtype=float))
    b = np.eye(len(da)) if db is None else np.diag(np.asarray(db, dtype=float))
    return MatrixPencil(a=SparseMatrix.from_dense(a), b=SparseMatrix.from_dense(b),
                        hermitian=True, b_positive_definite=True, problem_id="diag")


def circle(center, radius, count=1):
    return rc.Contour(shape="circle", center=complex(center), radius=radius, expected_count=count)


def csr(m):
    return dict(indptr=m.row_offsets, indices=m.col_indices, data=m.values)


def result_arrays(prefix, r, out):
    out[prefix + "_eigs"] = r.eigenvalues
    out[prefix + "_res"] = r.residuals
    out[prefix + "_vecs"] = r.eigenvectors
    out[prefix + "_stats"] = np.array([r.stats.n_linear_solves, r.stats.n_factorizations,
                                       r.stats.iterations])


def kats():
    out = {}
    p = diag_pencil([1.0, 3.0])
    out["proj_residue"] = rs.apply_projector(p, rc.quadrature_for(circle(1.0, 0.8), 32), np.eye(2))
    out["proj_empty"] = rs.apply_projector(p, rc.quadrature_for(circle(10.0, 1.0), 32), np.eye(2))
    v = np.random.default_rng(0).standard_normal((2, 2))
    out["proj_full_v"] = v
    out["proj_full"] = rs.apply_projector(p, rc.quadrature_for(circle(2.0, 5.0), 32), v)
    for nq in (8, 16, 32):
        out[f"proj_decay_{nq}"] = rs.apply_projector(p, rc.quadrature_for(circle(1.0, 0.8), nq), np.eye(2))
    p4 = diag_pencil([1.0, 2.0, 3.0, 10.0])
    result_arrays("cirr_diag", rs.cirr_solve(p4, circle(2.0, 1.5, 3), rs.SolverConfig(tol=1e-10), seed=0), out)
    result_arrays("cirr_diag_s1", rs.cirr_solve(p4, circle(2.0, 1.5, 3), rs.SolverConfig(), seed=1), out)
    m = rs.solve_multi(diag_pencil([1.0, 2.0, 8.0, 9.0]), [circle(1.5, 1.0, 2), circle(8.5, 1.0, 2)],
                       rs.SolverConfig(tol=1e-10), seed=0)
    out["multi_union"] = m.eigenvalues
    m = rs.solve_multi(diag_pencil([1.0, 2.0, 3.0]), [circle(1.5, 1.0, 2), circle(2.5, 1.0, 2)],
                       rs.SolverConfig(tol=1e-10), seed=0)
    out["multi_dedupe"] = m.eigenvalues
    # quadrature rules
    for nq in (4, 8, 32):
        r = rc.quadrature_for(circle(0.3, 1.7), nq)
        out[f"quad_circle_{nq}_nodes"], out[f"quad_circle_{nq}_weights"] = r.nodes, r.weights
    rect = rc.Contour(shape="rect", re_min=-1.0, re_max=2.0, im_min=-0.5, im_max=0.75)
    r = rc.quadrature_for(rect, 16)
    out["quad_rect_16_nodes"], out["quad_rect_16_weights"] = r.nodes, r.weights
    np.savez_compressed(os.path.join(HERE, "ref_kats.npz"), **out)


def thermal():
    out = {}
    t10 = rp.assemble_thermal(rp.grf_sample(rp.Grid2D(10, 10), 1.0, 0.1, 0.2, seed=7), 1.0)
    t20 = rp.assemble_thermal(rp.grf_sample(rp.Grid2D(20, 20), 1.0, 0.1, 0.2, seed=11), 1.0)
    for name, t in (("t10", t10), ("t20", t20)):
        for mat in ("a", "b"):
            for k, v in csr(getattr(t, mat)).items():
                out[f"{name}_{mat}_{k}"] = v
        out[f"{name}_n"] = np.array(t.n)
    # projector idempotence case (test_solvers.py:54-63)
    truth = rp.dense_ground_truth(t10, 2)
    rad = 0.5 * (truth.eigenvalues[1] - truth.eigenvalues[0])
    rule = rc.quadrature_for(circle(truth.eigenvalues[0], rad, 1), 32)
    v = np.random.default_rng(1).standard_normal((t10.n, 4))
    out["t10_proj_center"] = np.array([truth.eigenvalues[0], rad])
    out["t10_proj_v"] = v
    out["t10_proj_pv"] = rs.apply_projector(t10, rule, v)
    # residual re-verification case (test_solvers.py:106-118)
    truth4 = rp.dense_ground_truth(t20, 4)
    span = truth4.eigenvalues[-1] - truth4.eigenvalues[0]
    mid = 0.5 * (truth4.eigenvalues[0] + truth4.eigenvalues[-1])
    out["t20_rr_circle"] = np.array([mid, 0.75 * span])
    result_arrays("t20_rr", rs.cirr_solve(t20, circle(mid, 0.75 * span, 4), rs.SolverConfig(tol=1e-10), seed=0), out)
    # KDE-contour solve_multi (test_solvers.py:95-103)
    tt = rp.dense_ground_truth(t20, rp.target_count(t20.n))
    _, contours = rc.construct_contours(rc.SpectrumPrediction(values=tt.eigenvalues), n_min=1, n_max=50)
    out["t20_kde_contours"] = np.array(json.dumps([c.to_json_dict() for c in contours]))
    out["t20_kde_truth"] = tt.eigenvalues
    m = rs.solve_multi(t20, contours, rs.SolverConfig(tol=1e-10), seed=0)
    out["t20_kde_eigs"] = m.eigenvalues
    # n_q monotonicity case (test_solvers.py:129-142) -- 10 seeds x 2 n_q
    truth10 = rp.dense_ground_truth(t10, 4)
    mid = 0.5 * (truth10.eigenvalues[0] + truth10.eigenvalues[-1])
    span = truth10.eigenvalues[-1] - truth10.eigenvalues[0]
    out["t10_nq_circle"] = np.array([mid, 0.75 * span])
    for nq in (16, 32):
        worst = 0.0
        for seed in range(10):
            r = rs.cirr_solve(t10, circle(mid, 0.75 * span, 4),
                              rs.SolverConfig(n_q=nq, tol=1e-1, max_refine=1), seed=seed)
            worst = max(worst, r.residuals.max())
        out[f"t10_nq_worst_{nq}"] = np.array(worst)
    np.savez_compressed(os.path.join(HERE, "ref_thermal.npz"), **out)


def grf():
    out = {}
    for s in range(3):
        out[f"c2_s{s}"] = rp.grf_sample(rp.Grid2D(16, 16), 1.0, 0.5, 0.2, s).values
    out["c3_s0"] = rp.grf_sample(rp.Grid2D(48, 48), 1.0, 0.5, 0.2, 0).values
    out["t10_s7"] = rp.grf_sample(rp.Grid2D(10, 10), 1.0, 0.1, 0.2, 7).values
    np.savez_compressed(os.path.join(HERE, "ref_grf.npz"), **out)


def _ref_pencil(a, b):
    return MatrixPencil(a=SparseMatrix.from_dense(a), b=SparseMatrix.from_dense(b), hermitian=True)


def _ref_contours(wl):
    return [circle(c.center.real, float(c.radius), c.expected_count) for c in wl.contours]


def config2(n_gep=8):
    out = {}
    for s in range(n_gep):
        wl = W.config2_gep(s)
        cfg = rs.SolverConfig(n_q=wl.n_q, source_cols=wl.source_cols, n_moments=wl.n_moments)
        m = rs.solve_multi(_ref_pencil(wl.a, wl.b), _ref_contours(wl), cfg, seed=0)
        out[f"s{s}_contours"] = np.array(json.dumps([c.to_json_dict() for c in wl.contours]))
        for i, r in enumerate(m.results):
            out[f"s{s}_c{i}_eigs"] = r.eigenvalues if r is not None else np.array([])
            out[f"s{s}_c{i}_err"] = np.array("" if m.errors[i] is None else type(m.errors[i]).__name__)
    np.savez_compressed(os.path.join(HERE, "ref_config2.npz"), **out)


def config3():
    out = {}
    wl = W.config3()
    cfg = rs.SolverConfig(n_q=wl.n_q, source_cols=wl.source_cols, n_moments=wl.n_moments)
    m = rs.solve_multi(_ref_pencil(wl.a, wl.b), _ref_contours(wl), cfg, seed=0)
    out["contours"] = np.array(json.dumps([c.to_json_dict() for c in wl.contours]))
    for i, r in enumerate(m.results):
        out[f"c{i}_eigs"] = r.eigenvalues
        out[f"c{i}_res"] = r.residuals
        out[f"c{i}_stats"] = np.array([r.stats.n_linear_solves, r.stats.n_factorizations, r.stats.iterations])
    np.savez_compressed(os.path.join(HERE, "ref_config3.npz"), **out)


def feast():
    """The reference's own feast_solve / solve_multi(solver="feast")
    (solvers.py:230-285, 312-339) on thermal20 (one low-end circle at tol 1e-8
    and the KDE contours at tol 1e-10) and on config 3 (N=32, L=40, M=1):
    eigenvalues, residuals, iterations and n_linear_solves per contour. Pins
    the oracle's feast_solve (tests/test_oracle_pin.py) and the GPU FEAST
    (tests/test_gpu_feast.py)."""
    out = {}
    t20 = rp.assemble_thermal(rp.grf_sample(rp.Grid2D(20, 20), 1.0, 0.1, 0.2, seed=11), 1.0)
    full = rp.dense_ground_truth(t20, 5).eigenvalues
    mid = 0.5 * (full[0] + full[3])
    rad = 0.5 * (full[3] + full[4]) - mid
    out["t20_low_circle"] = np.array([mid, rad])
    r = rs.feast_solve(t20, circle(mid, rad, 4), rs.SolverConfig(tol=1e-8), seed=0)
    result_arrays("t20_low", r, out)
    tt = rp.dense_ground_truth(t20, rp.target_count(t20.n))
    _, contours = rc.construct_contours(rc.SpectrumPrediction(values=tt.eigenvalues), n_min=1, n_max=50)
    out["t20_kde_contours"] = np.array(json.dumps([c.to_json_dict() for c in contours]))
    m = rs.solve_multi(t20, contours, rs.SolverConfig(tol=1e-10), solver="feast", seed=0)
    for i, rr in enumerate(m.results):
        result_arrays(f"t20_kde{i}", rr, out)
    wl = W.config3()
    cfg = rs.SolverConfig(n_q=wl.n_q, source_cols=40, n_moments=1)
    out["c3_contours"] = np.array(json.dumps([c.to_json_dict() for c in wl.contours]))
    m = rs.solve_multi(_ref_pencil(wl.a, wl.b), _ref_contours(wl), cfg, solver="feast", seed=0)
    for i, rr in enumerate(m.results):
        result_arrays(f"c3_{i}", rr, out)
    for k in [k for k in out if k.endswith("_vecs")]:
        del out[k]                     # keep the fixture small: eigenvectors are checked by residuals
    np.savez_compressed(os.path.join(HERE, "ref_feast.npz"), **out)


def dataset():
    """A dataset directory written by the reference (problems.write_dataset) and
    its dense matrices and truth (tests/test_gpu_dropin.py reads it back with
    the reference's own read_dataset and solves it on the GPU)."""
    import shutil

    field = rp.grf_sample(rp.Grid2D(8, 8), 1.0, 0.3, 0.25, 11)
    pencil = rp.assemble_thermal(field, 1.0)
    truth = rp.dense_ground_truth(pencil, 6)
    d = os.path.join(HERE, "dataset_thermal8")
    shutil.rmtree(d, ignore_errors=True)
    rp.write_dataset(d, pencil, field, truth)
    out = {"a": pencil.a.to_dense(), "b": pencil.b.to_dense(), "truth": truth.eigenvalues,
           "field": field.values, "problem_id": np.array(pencil.problem_id)}
    np.savez_compressed(os.path.join(HERE, "ref_dataset.npz"), **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["kats", "thermal", "grf", "config2", "config3", "dataset"]
    for w in which:
        globals()[w]()
        print("wrote", w, flush=True)
