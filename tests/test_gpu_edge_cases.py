"""Edge cases from the round-1 code review, on the GPU path:
waves of more than 65535 pencils, source_cols=0, more than 16 moments, and
complex duplicates from overlapping contours on a non-Hermitian pencil."""
import numpy as np
import pytest
import scipy.linalg as sla

from conftest import DensePencil, diag_pencil

pytestmark = pytest.mark.gpu

from paper_2511_01927_b200 import Contour, NoEigenvaluesFound, SolverConfig, solve_multi, solve_multi_batch  # noqa: E402
from paper_2511_01927_b200 import solvers as S  # noqa: E402
from paper_2511_01927_b200 import workloads as W  # noqa: E402
from paper_2511_01927_b200.contours import contains  # noqa: E402


def circle(center, radius, count=1):
    return Contour(shape="circle", center=complex(center), radius=radius, expected_count=count)


def test_more_than_65535_pencils_split_into_waves():
    """4200 GEPs x 1 contour x 16 nodes = 67200 pencils: two waves, every
    result equal to its own solve."""
    rng = np.random.default_rng(5)
    ps = [diag_pencil(np.sort(rng.uniform(0.5, 10.0, 16)) + np.arange(16)) for _ in range(4200)]
    cons = []
    for p in ps:
        d = np.diag(p.a)
        cons.append([circle(0.5 * (d[2] + d[4]), 0.5 * (d[4] - d[2]) + 0.25 * min(d[5] - d[4], d[2] - d[1]), 3)])
    cfg = SolverConfig(n_q=16, source_cols=8, n_moments=4)
    assert len(S._waves([S._Contour(0, c[0], cfg, 0, 16) for c in cons], 16, 1 << 60)) == 2
    out = solve_multi_batch(ps, cons, cfg)
    for p, m in zip(ps, out):
        d = np.diag(p.a)
        assert m.errors[0] is None
        assert np.allclose(m.results[0].eigenvalues, d[2:5], rtol=1e-10)


def test_source_cols_zero_is_no_eigenvalues_found():
    """The reference: V has 0 columns -> RankZeroError in the truncation ->
    loop break -> NoEigenvaluesFound, isolated by solve_multi (solvers.py:186-214)."""
    p = diag_pencil([1.0, 2.0, 3.0, 10.0])
    cs = [circle(2.0, 1.5, 3), circle(10.0, 1.0, 1)]
    m = solve_multi(p, cs, SolverConfig(source_cols=0))
    assert all(r is None for r in m.results)
    assert all(isinstance(e, NoEigenvaluesFound) for e in m.errors)
    with pytest.raises(NoEigenvaluesFound):
        S.cirr_solve(p, cs[0], SolverConfig(source_cols=0))


def test_more_than_16_moments():
    """The reference accepts any n_moments >= 1; the moment kernel runs 16 per launch."""
    a, b = W.config1_matrices(seed=0, n=128)
    ev = np.sort(sla.eigh(a, b, eigvals_only=True))
    c = circle(0.5 * (ev[3] + ev[7]), 0.5 * (ev[7] - ev[3]) + 0.3 * min(ev[8] - ev[7], ev[3] - ev[2]), 5)
    p = DensePencil(a, b, True)
    m4 = solve_multi(p, [c], SolverConfig(source_cols=4, n_moments=4))
    m20 = solve_multi(p, [c], SolverConfig(source_cols=4, n_moments=20))
    assert np.allclose(m20.eigenvalues, ev[3:8], rtol=1e-9)
    assert np.allclose(m20.eigenvalues, m4.eigenvalues, rtol=1e-9)


def test_overlapping_ellipses_nonhermitian_no_duplicates():
    """Two overlapping ellipses on a dense non-Hermitian pencil: the union holds
    every eigenvalue inside either contour exactly once (complex dedupe)."""
    a, b = W.config4_matrices(seed=1, n=256)
    truth = sla.eigvals(a, b)
    e1 = Contour(shape="ellipse", center=0.45 + 0j, semi_re=0.3, semi_im=0.15, expected_count=8)
    e2 = Contour(shape="ellipse", center=0.65 + 0j, semi_re=0.3, semi_im=0.15, expected_count=8)
    m = solve_multi(DensePencil(a, b, False), [e1, e2], SolverConfig(n_q=32, source_cols=24, n_moments=4))
    inside = truth[[contains(e1, z) or contains(e2, z) for z in truth]]
    union = m.eigenvalues
    assert len(union) == len(inside)
    for z in inside:
        assert np.sum(np.abs(union - z) <= 1e-8 * abs(z)) == 1
