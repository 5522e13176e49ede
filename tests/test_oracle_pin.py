"""Pin the CPU oracle (oracle/cirr.py) against the unmodified reference.

Golden vectors were produced by tests/golden/make_golden.py importing the
reference package (cieig) in the build container.  The oracle in *reference
mode* (raw moments, SuperLU, Hermitian RR) must reproduce them to rounding;
in its default centred mode it must pass the reference's own KATs.
"""
import json

import numpy as np
import pytest

import oracle
from oracle.cirr import OracleConfig, Pencil, quadrature
from conftest import diag_pencil, golden
from paper_2511_01927_b200.contours import Contour

REF = OracleConfig(moments="raw", lu="superlu", rr="hermitian")


def circle(c, r, k=1):
    return Contour(shape="circle", center=complex(c), radius=r, expected_count=k)


def P(pencil):
    return Pencil(pencil.a, pencil.b, True)


def test_projector_kats_match_reference():
    g = golden("ref_kats.npz")
    p = P(diag_pencil([1.0, 3.0]))
    assert np.abs(oracle.apply_projector(p, circle(1.0, 0.8), np.eye(2), REF) - g["proj_residue"]).max() <= 1e-15
    assert np.abs(oracle.apply_projector(p, circle(10.0, 1.0), np.eye(2), REF) - g["proj_empty"]).max() <= 1e-15
    assert np.abs(oracle.apply_projector(p, circle(2.0, 5.0), g["proj_full_v"], REF) - g["proj_full"]).max() <= 1e-15
    for nq in (8, 16, 32):
        cfg = OracleConfig(n_q=nq, moments="raw", lu="superlu")
        got = oracle.apply_projector(p, circle(1.0, 0.8), np.eye(2), cfg)
        assert np.abs(got - g[f"proj_decay_{nq}"]).max() <= 1e-15


@pytest.mark.parametrize("mode", ["raw", "centred"])
def test_cirr_diag_kat(mode):
    g = golden("ref_kats.npz")
    cfg = OracleConfig(tol=1e-10, moments=mode, lu="superlu" if mode == "raw" else "dense")
    r = oracle.cirr_solve(P(diag_pencil([1.0, 2.0, 3.0, 10.0])), circle(2.0, 1.5, 3), cfg, seed=0)
    assert np.allclose(r.eigenvalues, [1.0, 2.0, 3.0], atol=1e-10)
    assert np.allclose(r.eigenvalues, g["cirr_diag_eigs"], atol=1e-12)
    assert r.residuals.max() <= 1e-10
    assert r.n_factorizations == int(g["cirr_diag_stats"][1]) == 32
    if mode == "raw":
        assert r.iterations == int(g["cirr_diag_stats"][2])
        assert r.n_linear_solves == int(g["cirr_diag_stats"][0])


def test_thermal_reference_mode_matches(thermal):
    g = thermal["g"]
    mid, rad = g["t20_rr_circle"]
    r = oracle.cirr_solve(P(thermal["t20"]), circle(mid, rad, 4), OracleConfig(moments="raw", lu="superlu"), seed=0)
    assert np.allclose(r.eigenvalues, g["t20_rr_eigs"], rtol=1e-12)
    assert r.iterations == int(g["t20_rr_stats"][2])
    assert r.n_linear_solves == int(g["t20_rr_stats"][0])
    c0, rad = g["t10_proj_center"]
    pv = oracle.apply_projector(P(thermal["t10"]), circle(c0, rad, 1), g["t10_proj_v"], REF)
    assert np.abs(pv - g["t10_proj_pv"]).max() <= 1e-12 * np.abs(g["t10_proj_v"]).max()


def test_thermal_kde_both_modes(thermal):
    g = thermal["g"]
    contours = [Contour.from_json_dict(d) for d in json.loads(str(g["t20_kde_contours"]))]
    for cfg in (OracleConfig(moments="raw", lu="superlu"), OracleConfig()):
        m = oracle.solve_multi(P(thermal["t20"]), contours, cfg, seed=0)
        assert np.allclose(m.eigenvalues, g["t20_kde_eigs"], rtol=1e-10)
        assert (np.abs(m.eigenvalues - g["t20_kde_truth"]) / np.abs(g["t20_kde_truth"])).max() <= 1e-8


def test_multi_kats():
    g = golden("ref_kats.npz")
    m = oracle.solve_multi(P(diag_pencil([1.0, 2.0, 8.0, 9.0])), [circle(1.5, 1.0, 2), circle(8.5, 1.0, 2)],
                           OracleConfig(tol=1e-10), seed=0)
    assert np.allclose(m.eigenvalues, g["multi_union"], atol=1e-9)
    m = oracle.solve_multi(P(diag_pencil([1.0, 2.0, 3.0])), [circle(1.5, 1.0, 2), circle(2.5, 1.0, 2)],
                           OracleConfig(tol=1e-10), seed=0)
    assert np.allclose(m.eigenvalues, g["multi_dedupe"], atol=1e-9)


def test_quadrature_matches_reference():
    g = golden("ref_kats.npz")
    for nq in (4, 8, 32):
        nodes, w = quadrature(circle(0.3, 1.7), nq)
        assert np.array_equal(nodes, g[f"quad_circle_{nq}_nodes"])
        assert np.array_equal(w, g[f"quad_circle_{nq}_weights"])
    rect = Contour(shape="rect", re_min=-1.0, re_max=2.0, im_min=-0.5, im_max=0.75)
    nodes, w = quadrature(rect, 16)
    assert np.array_equal(nodes, g["quad_rect_16_nodes"])
    assert np.array_equal(w, g["quad_rect_16_weights"])


def test_config2_reference_goldens():
    """Reference solve_multi on 8 config-2 GEPs: the oracle in reference mode
    reproduces it; the centred oracle finds the exact truth count (the raw
    reference misses pairs on some GEPs -- SURVEY 8(c))."""
    from paper_2511_01927_b200 import workloads as W
    g = golden("ref_config2.npz")
    o = golden("oracle_config2.npz")
    for s in range(8):
        a, b = W.config2_matrices(s)
        contours = [Contour.from_json_dict(d) for d in json.loads(str(g[f"s{s}_contours"]))]
        p = Pencil(a, b, True)
        raw = oracle.solve_multi(p, contours, OracleConfig(n_q=16, source_cols=8, n_moments=4, moments="raw",
                                                           lu="superlu"), seed=0)
        cen = oracle.solve_multi(p, contours, OracleConfig(n_q=16, source_cols=8, n_moments=4), seed=0)
        for i in range(len(contours)):
            ref = g[f"s{s}_c{i}_eigs"]
            r = raw.results[i]
            assert r is not None and np.allclose(r.eigenvalues, ref, rtol=1e-9), (s, i)
            truth = o[f"s{s}_c{i}_truth"]
            c = cen.results[i]
            assert c is not None and len(c.eigenvalues) == len(truth), (s, i)
            assert np.allclose(c.eigenvalues, truth, rtol=1e-8)


def test_config3_reference_golden():
    from paper_2511_01927_b200 import workloads as W
    g = golden("ref_config3.npz")
    o = golden("oracle_config3.npz")
    contours = [Contour.from_json_dict(d) for d in json.loads(str(g["contours"]))]
    for cg, co in zip(json.loads(str(g["contours"])), json.loads(str(o["contours"]))):
        assert abs(cg["center"][0] - co["center"][0]) <= 1e-12 * abs(cg["center"][0])
        assert abs(cg["radius"] - co["radius"]) <= 1e-10 * cg["radius"]
    for i in range(len(contours)):
        ref = g[f"c{i}_eigs"]
        assert np.allclose(o[f"c{i}_eigs"], ref, rtol=1e-10)
        assert len(o[f"c{i}_truth"]) == len(ref)
    del W


def test_config1_reference_fails_oracle_succeeds():
    """SURVEY 0 finding 1: raw moments -> ConvergenceError; centred -> 33/33."""
    o = golden("oracle_config1.npz")
    assert len(o["c0_eigs"]) == len(o["c0_truth"]) == 33
    assert float(o["c0_res"].max()) <= 1e-10


def test_feast_oracle_matches_reference(thermal):
    """oracle.feast_solve (reference mode: SuperLU, Hermitian RR; one moment so
    the centring delta is moot) against the unmodified reference's feast_solve
    (tests/golden/ref_feast.npz, make_golden.py feast): eigenvalues to 1e-10,
    identical iteration and solve counts."""
    g = golden("ref_feast.npz")
    p = P(thermal["t20"])
    mid, rad = g["t20_low_circle"]
    r = oracle.feast_solve(p, circle(mid, rad, 4), OracleConfig(tol=1e-8, lu="superlu", rr="hermitian"), seed=0)
    assert np.allclose(r.eigenvalues, g["t20_low_eigs"], rtol=1e-10)
    assert [r.n_linear_solves, r.n_factorizations, r.iterations] == list(g["t20_low_stats"])
    cs = [Contour.from_json_dict(d) for d in json.loads(str(g["t20_kde_contours"]))]
    m = oracle.solve_multi(p, cs, OracleConfig(tol=1e-10, lu="superlu", rr="hermitian"), seed=0, solver="feast")
    for i, rr in enumerate(m.results):
        assert np.allclose(rr.eigenvalues, g[f"t20_kde{i}_eigs"], rtol=1e-10)
        assert [rr.n_linear_solves, rr.n_factorizations, rr.iterations] == list(g[f"t20_kde{i}_stats"])


@pytest.mark.slow
def test_feast_oracle_matches_reference_config3():
    from paper_2511_01927_b200 import workloads as W
    g = golden("ref_feast.npz")
    a, b = W.config3_matrices()
    cs = [Contour.from_json_dict(d) for d in json.loads(str(g["c3_contours"]))]
    cfg = OracleConfig(n_q=32, source_cols=40, n_moments=1, lu="superlu", rr="hermitian")
    m = oracle.solve_multi(Pencil(a, b, True), cs, cfg, seed=0, solver="feast")
    for i, rr in enumerate(m.results):
        assert np.allclose(rr.eigenvalues, g[f"c3_{i}_eigs"], rtol=1e-10)
        assert [rr.n_linear_solves, rr.n_factorizations, rr.iterations] == list(g[f"c3_{i}_stats"])
