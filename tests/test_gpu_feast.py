"""FEAST on the device factors: the reference's own FEAST
KATs (pkg/tests/test_solvers.py:149-169) and CIRR/FEAST agreement (acceptance
A3, tests/test_acceptance.py:130-150)."""
import json

import numpy as np
import pytest
import scipy.linalg as sla

from conftest import diag_pencil, golden

pytestmark = pytest.mark.gpu

from paper_2511_01927_b200 import Contour, SolverConfig, cirr_solve, feast_solve, solve_multi  # noqa: E402
from paper_2511_01927_b200 import workloads as W  # noqa: E402


def circle(center, radius, count=1):
    return Contour(shape="circle", center=complex(center), radius=radius, expected_count=count)


def test_feast_matches_cirr_diagonal():
    p = diag_pencil([1.0, 2.0, 3.0, 10.0])
    c = circle(2.0, 1.5, 3)
    r1 = cirr_solve(p, c, SolverConfig(tol=1e-10), seed=0)
    r2 = feast_solve(p, c, SolverConfig(tol=1e-10), seed=0)
    assert np.allclose(r1.eigenvalues, r2.eigenvalues, atol=1e-10)


def test_feast_thermal_iterations(thermal):
    t20 = thermal["t20"]
    full = np.sort(sla.eigh(t20.a, t20.b, eigvals_only=True))
    m = 4
    mid = 0.5 * (full[0] + full[m - 1])
    rad = 0.5 * (full[m - 1] + full[m]) - mid
    res = feast_solve(t20, circle(mid, rad, m), SolverConfig(tol=1e-8), seed=0)
    assert res.stats.iterations <= 4
    rel = np.abs(res.eigenvalues - full[:m]) / np.abs(full[:m])
    assert rel.max() <= 1e-8


def test_feast_cirr_agree_kde(thermal):
    g = thermal["g"]
    contours = [Contour.from_json_dict(d) for d in json.loads(str(g["t20_kde_contours"]))]
    a = solve_multi(thermal["t20"], contours, SolverConfig(tol=1e-10), solver="cirr", seed=0).eigenvalues
    b = solve_multi(thermal["t20"], contours, SolverConfig(tol=1e-10), solver="feast", seed=0).eigenvalues
    assert len(a) == len(b)
    assert np.abs(a - b).max() <= 1e-8 * np.abs(a).max()


def test_feast_config3_matches_oracle_counts():
    a, b = W.config3_matrices()
    fix = golden("oracle_config3.npz")
    contours = [Contour.from_json_dict(d) for d in json.loads(str(fix["contours"]))]
    m = solve_multi(type("P", (), {"a": a, "b": b, "hermitian": True})(), contours,
                    SolverConfig(n_q=32, source_cols=40, n_moments=1), solver="feast", seed=0)
    for i, r in enumerate(m.results):
        assert r is not None, m.errors[i]
        ref = fix[f"c{i}_eigs"]
        assert len(r.eigenvalues) == len(ref)
        assert np.abs(r.eigenvalues - ref).max() <= 1e-8 * np.abs(ref).max()
        assert r.residuals.max() <= 1e-10


def _stats(r):
    return [r.stats.n_linear_solves, r.stats.n_factorizations, r.stats.iterations]


def test_feast_matches_reference_thermal(thermal):
    """GPU FEAST against the reference's own feast_solve / solve_multi(feast)
    outputs (ref_feast.npz, which also pins oracle.feast_solve): eigenvalues to
    1e-8, the same iteration and solve counts."""
    g = golden("ref_feast.npz")
    mid, rad = g["t20_low_circle"]
    r = feast_solve(thermal["t20"], circle(mid, rad, 4), SolverConfig(tol=1e-8), seed=0)
    assert np.allclose(r.eigenvalues, g["t20_low_eigs"], rtol=1e-8)
    assert _stats(r) == list(g["t20_low_stats"])
    assert r.residuals.max() <= 1e-8
    cs = [Contour.from_json_dict(d) for d in json.loads(str(g["t20_kde_contours"]))]
    m = solve_multi(thermal["t20"], cs, SolverConfig(tol=1e-10), solver="feast", seed=0)
    for i, rr in enumerate(m.results):
        assert np.allclose(rr.eigenvalues, g[f"t20_kde{i}_eigs"], rtol=1e-8)
        assert _stats(rr) == list(g[f"t20_kde{i}_stats"])


def test_feast_matches_reference_config3():
    """Config 3 (n=2304, 3 contours, N=32, L=40): exact counts, eigenvalues to
    1e-8 and the reference's iteration counts per contour (4, 8, 4)."""
    g = golden("ref_feast.npz")
    a, b = W.config3_matrices()
    cs = [Contour.from_json_dict(d) for d in json.loads(str(g["c3_contours"]))]
    m = solve_multi(type("P", (), {"a": a, "b": b, "hermitian": True})(), cs,
                    SolverConfig(n_q=32, source_cols=40, n_moments=1), solver="feast", seed=0)
    for i, rr in enumerate(m.results):
        assert rr is not None, m.errors[i]
        ref = g[f"c3_{i}_eigs"]
        assert len(rr.eigenvalues) == len(ref)
        assert np.allclose(rr.eigenvalues, ref, rtol=1e-8)
        assert _stats(rr) == list(g[f"c3_{i}_stats"])
        assert rr.residuals.max() <= 1e-10
