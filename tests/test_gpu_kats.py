"""The reference's own known-answer tests, run through the GPU path.

Mirrors /root/reference/pkg/tests/test_solvers.py:30-229 (projector KATs,
CIRR on analytic pencils, multi-contour orchestration) with the same
tolerances, plus comparison against golden outputs of the unmodified
reference (tests/golden/ref_kats.npz, ref_thermal.npz).
"""
import json

import numpy as np
import pytest

from conftest import diag_pencil, golden

pytestmark = pytest.mark.gpu

from paper_2511_01927_b200 import (  # noqa: E402
    Contour,
    NoEigenvaluesFound,
    SingularShiftError,
    SolverConfig,
    apply_projector,
    cirr_solve,
    quadrature_for,
    solve_multi,
)


def circle(center, radius, count=1):
    return Contour(shape="circle", center=complex(center), radius=radius, expected_count=count)


def test_projector_diagonal_residue():
    p = apply_projector(diag_pencil([1.0, 3.0]), quadrature_for(circle(1.0, 0.8), 32), np.eye(2))
    assert np.abs(p - np.diag([1.0, 0.0])).max() <= 1e-10
    assert np.abs(p - golden("ref_kats.npz")["proj_residue"]).max() <= 1e-14


def test_projector_empty_region():
    p = apply_projector(diag_pencil([1.0, 3.0]), quadrature_for(circle(10.0, 1.0), 32), np.eye(2))
    assert np.abs(p).max() <= 1e-8


def test_projector_full_spectrum_is_identity():
    v = np.random.default_rng(0).standard_normal((2, 2))
    p = apply_projector(diag_pencil([1.0, 3.0]), quadrature_for(circle(2.0, 5.0), 32), v)
    assert np.abs(p - v).max() <= 1e-8


def test_projector_quadrature_error_decay():
    errs = []
    g = golden("ref_kats.npz")
    for nq in (8, 16, 32):
        p = apply_projector(diag_pencil([1.0, 3.0]), quadrature_for(circle(1.0, 0.8), nq), np.eye(2))
        errs.append(np.abs(p - np.diag([1.0, 0.0])).max())
        assert np.abs(p - g[f"proj_decay_{nq}"]).max() <= 1e-13
    assert errs[0] > errs[1] > errs[2]
    assert errs[2] <= 1e-10


def test_projector_idempotence_thermal(thermal):
    g = thermal["g"]
    c0, rad = g["t10_proj_center"]
    rule = quadrature_for(circle(c0, rad, 1), 32)
    v = g["t10_proj_v"]
    pv = apply_projector(thermal["t10"], rule, v)
    assert np.abs(pv - g["t10_proj_pv"]).max() <= 1e-10 * np.abs(v).max()
    ppv = apply_projector(thermal["t10"], rule, pv)
    assert np.abs(ppv - pv).max() <= 1e-8 * np.abs(v).max()


def test_cirr_diagonal():
    res = cirr_solve(diag_pencil([1.0, 2.0, 3.0, 10.0]), circle(2.0, 1.5, 3), SolverConfig(tol=1e-10), seed=0)
    assert np.allclose(res.eigenvalues, [1.0, 2.0, 3.0], atol=1e-10)
    assert res.residuals.max() <= 1e-10
    assert res.stats.n_factorizations == 32
    assert res.to_json_dict()["stats"]["n_factorizations"] == 32


def test_cirr_empty_contour():
    with pytest.raises(NoEigenvaluesFound):
        cirr_solve(diag_pencil([1.0, 2.0, 3.0, 10.0]), circle(100.0, 1.0, 1), SolverConfig(), seed=0)


def test_cirr_singular_shift():
    # a rect with its bottom edge on the real axis puts the n_q=4 Gauss node of
    # that edge (node 0) exactly on the eigenvalue 2.0 (test_linalg.py:36-40)
    rect = Contour(shape="rect", re_min=0.0, re_max=4.0, im_min=0.0, im_max=1.0, expected_count=1)
    with pytest.raises(SingularShiftError) as exc:
        cirr_solve(diag_pencil([1.0, 2.0]), rect, SolverConfig(n_q=4), seed=0)
    assert exc.value.node_index == 0
    assert exc.value.shift == 2.0
    m = solve_multi(diag_pencil([1.0, 2.0]), [rect], SolverConfig(n_q=4))
    assert isinstance(m.errors[0], SingularShiftError)


def test_cirr_thermal_residual_reverification(thermal):
    g = thermal["g"]
    mid, rad = g["t20_rr_circle"]
    res = cirr_solve(thermal["t20"], circle(mid, rad, 4), SolverConfig(tol=1e-10), seed=0)
    assert np.allclose(res.eigenvalues, g["t20_rr_eigs"], rtol=1e-10)
    a, b = thermal["t20"].a, thermal["t20"].b
    for lam, x, r in zip(res.eigenvalues, res.eigenvectors.T, res.residuals):
        ax, bx = a @ x, b @ x
        check = np.linalg.norm(ax - lam * bx) / (np.linalg.norm(ax) + abs(lam) * np.linalg.norm(bx))
        assert check <= 1e-10
        assert check == pytest.approx(r, rel=1e-6, abs=1e-14)


def test_cirr_thermal_kde_contours(thermal):
    g = thermal["g"]
    contours = [Contour.from_json_dict(d) for d in json.loads(str(g["t20_kde_contours"]))]
    multi = solve_multi(thermal["t20"], contours, SolverConfig(tol=1e-10), seed=0)
    got = multi.eigenvalues
    truth = g["t20_kde_truth"]
    assert len(got) == len(truth)
    assert (np.abs(got - truth) / np.abs(truth)).max() <= 1e-8


def test_inside_contour_filter():
    res = cirr_solve(diag_pencil([1.0, 2.0, 3.0, 10.0]), circle(2.0, 1.5, 3), SolverConfig(), seed=1)
    for lam in res.eigenvalues:
        assert abs(lam - 2.0) < 1.5 + 1e-12 * 9.0


def test_nq_monotonicity(thermal):
    g = thermal["g"]
    mid, rad = g["t10_nq_circle"]
    worst = {}
    for nq in (16, 32):
        m = 0.0
        for seed in range(10):
            r = cirr_solve(thermal["t10"], circle(mid, rad, 4), SolverConfig(n_q=nq, tol=1e-1, max_refine=1),
                           seed=seed)
            m = max(m, r.residuals.max())
        worst[nq] = m
    assert worst[16] >= worst[32]


def test_solve_multi_union():
    m = solve_multi(diag_pencil([1.0, 2.0, 8.0, 9.0]), [circle(1.5, 1.0, 2), circle(8.5, 1.0, 2)],
                    SolverConfig(tol=1e-10), seed=0)
    assert np.allclose(m.eigenvalues, [1.0, 2.0, 8.0, 9.0], atol=1e-9)


def test_solve_multi_isolates_failures():
    m = solve_multi(diag_pencil([1.0, 2.0, 8.0, 9.0]), [circle(100.0, 1.0, 1), circle(8.5, 1.0, 2)],
                    SolverConfig(tol=1e-10), seed=0)
    assert m.results[0] is None
    assert isinstance(m.errors[0], NoEigenvaluesFound)
    assert np.allclose(m.eigenvalues, [8.0, 9.0], atol=1e-9)


def test_solve_multi_deterministic(thermal):
    g = thermal["g"]
    contours = [Contour.from_json_dict(d) for d in json.loads(str(g["t20_kde_contours"]))]
    a = solve_multi(thermal["t10"], [circle(*g["t10_nq_circle"], 4)], SolverConfig(tol=1e-10), seed=5)
    b = solve_multi(thermal["t10"], [circle(*g["t10_nq_circle"], 4)], SolverConfig(tol=1e-10), seed=5)
    assert np.array_equal(a.eigenvalues, b.eigenvalues)
    del contours


def test_solve_multi_dedupes_overlap():
    m = solve_multi(diag_pencil([1.0, 2.0, 3.0]), [circle(1.5, 1.0, 2), circle(2.5, 1.0, 2)],
                    SolverConfig(tol=1e-10), seed=0)
    assert np.allclose(m.eigenvalues, [1.0, 2.0, 3.0], atol=1e-9)
