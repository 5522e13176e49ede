"""Labelled variants (not the path of record): conjugate-pair halving.

SURVEY.md finding 9: for real A, B and a node set closed under conjugation,
M(conj z)^-1 R = conj(M(z)^-1 conj R), so only the upper-half nodes need a
factorisation.  The variant must return the same eigenpairs as the path of
record (same counts, eigenvalues to 1e-9 relative, residuals <= tol) with
half the factorisations.
"""
import dataclasses

import numpy as np
import pytest
import scipy.linalg as sla

from conftest import DensePencil

pytestmark = pytest.mark.gpu

from paper_2511_01927_b200 import Contour, SolverConfig, feast_solve, solve_multi  # noqa: E402
from paper_2511_01927_b200 import workloads as W  # noqa: E402
from paper_2511_01927_b200.contours import contains  # noqa: E402


def _match(got, ref):
    used = np.zeros(len(got), dtype=bool)
    worst = 0.0
    for v in ref:
        d = np.where(used, np.inf, np.abs(got - v))
        j = int(np.argmin(d))
        used[j] = True
        worst = max(worst, d[j] / abs(v))
    return worst


def _counted(c, ev):
    return dataclasses.replace(c, expected_count=int(sum(contains(c, complex(v)) for v in ev)))


def _pair_run(a, b, contours, cfg_kw, solver="cirr", hermitian=False):
    p = DensePencil(a, b, hermitian=hermitian)
    base = solve_multi(p, contours, SolverConfig(**cfg_kw), solver=solver)
    half = solve_multi(p, contours, SolverConfig(conjugate_pairs=True, **cfg_kw), solver=solver)
    return base, half


def _same(base, half, n_q):
    for rb, rh in zip(base.results, half.results):
        assert rb is not None and rh is not None
        assert len(rb.eigenvalues) == len(rh.eigenvalues)
        assert _match(rh.eigenvalues, rb.eigenvalues) <= 1e-9
        assert rh.residuals.max() <= 1e-10
        assert rh.stats.n_factorizations == n_q // 2
        assert rb.stats.n_factorizations == n_q


def test_conjugate_pairs_config4_shape():
    n = 768
    a, b = W.config4_matrices(seed=5, n=n)
    ev = sla.eigvals(a, b)
    cs = []
    for cen in (0.5, -0.5):
        c = Contour(shape="ellipse", center=complex(cen, 0.0), semi_re=0.3, semi_im=0.15)
        cs.append(_counted(c, ev))
    base, half = _pair_run(a, b, cs, dict(n_q=64, source_cols=32, n_moments=8))
    _same(base, half, 64)
    for c, r in zip(cs, half.results):
        assert len(r.eigenvalues) == c.expected_count


def test_conjugate_pairs_hermitian_circles():
    wl = W.config1(seed=0)
    base, half = _pair_run(wl.a, wl.b, wl.contours[:3], dict(n_q=wl.n_q, source_cols=wl.source_cols,
                                                            n_moments=wl.n_moments), hermitian=True)
    _same(base, half, wl.n_q)


def test_conjugate_pairs_feast_complex_block():
    # FEAST's iterates are complex after the first pass: [U | conj U] solves
    a, b = W.config4_matrices(seed=2, n=384)
    ev = sla.eigvals(a, b)
    c = _counted(Contour(shape="circle", center=0.4 + 0j, radius=0.25), ev)
    cfg = dict(n_q=32, source_cols=2 * c.expected_count + 8)
    p = DensePencil(a, b, hermitian=False)
    rb = feast_solve(p, c, SolverConfig(**cfg))
    rh = feast_solve(p, c, SolverConfig(conjugate_pairs=True, **cfg))
    assert len(rh.eigenvalues) == len(rb.eigenvalues) == c.expected_count
    assert _match(rh.eigenvalues, rb.eigenvalues) <= 1e-9
    assert rh.stats.n_factorizations == 16


def test_conjugate_pairs_falls_back_off_axis():
    # centre off the real axis: nodes are not conjugate-closed -> full node set
    a, b = W.config4_matrices(seed=1, n=256)
    ev = sla.eigvals(a, b)
    c = _counted(Contour(shape="circle", center=0.3 + 0.2j, radius=0.3), ev)
    base, half = _pair_run(a, b, [c], dict(n_q=32))
    assert half.results[0].stats.n_factorizations == 32
    assert _match(half.results[0].eigenvalues, base.results[0].eigenvalues) <= 1e-12


def test_early_exit_keeps_the_converged_pairs():
    # SURVEY.md finding 8: spurious inside Ritz values keep config-4-like
    # problems at max_refine; stopping once the converged set is stable returns
    # the same converged eigenpairs with fewer passes
    n = 768
    a, b = W.config4_matrices(seed=5, n=n)
    ev = sla.eigvals(a, b)
    cs = [_counted(Contour(shape="ellipse", center=complex(cen, 0.0), semi_re=0.3, semi_im=0.15), ev)
          for cen in (0.5, -0.5)]
    p = DensePencil(a, b, hermitian=False)
    kw = dict(n_q=64, source_cols=32, n_moments=8)
    base = solve_multi(p, cs, SolverConfig(**kw))
    early = solve_multi(p, cs, SolverConfig(early_exit=True, **kw))
    for c, rb, re_ in zip(cs, base.results, early.results):
        assert len(re_.eigenvalues) == len(rb.eigenvalues) == c.expected_count
        assert _match(re_.eigenvalues, rb.eigenvalues) <= 1e-9
        assert re_.residuals.max() <= 1e-10
        assert re_.stats.iterations <= rb.stats.iterations
