"""The pipelined engine (one host thread + high-priority stream per contour,
bulk work on one low-priority stream) must return what the single-stream
batched loop returns: same counts, eigenvalues to rounding, same stats."""
import dataclasses

import numpy as np
import pytest
import scipy.linalg as sla

from conftest import DensePencil

pytestmark = pytest.mark.gpu

from paper_2511_01927_b200 import Contour, SolverConfig, solve_multi  # noqa: E402
from paper_2511_01927_b200 import solvers as S  # noqa: E402
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


def _run(pencil, cs, cfg, pipeline, monkeypatch):
    monkeypatch.setattr(S, "_PIPELINE", pipeline)
    return solve_multi(pencil, cs, cfg)


def test_pipelined_equals_batched_nonhermitian(monkeypatch):
    a, b = W.config4_matrices(seed=4, n=640)
    ev = sla.eigvals(a, b)
    cs = []
    for cen in (0.5, -0.5, 0.0):
        c = Contour(shape="ellipse", center=complex(cen, 0.0), semi_re=0.25, semi_im=0.15)
        cs.append(dataclasses.replace(c, expected_count=int(sum(contains(c, complex(v)) for v in ev))))
    p = DensePencil(a, b, hermitian=False)
    cfg = SolverConfig(n_q=32, source_cols=24, n_moments=4)
    mb = _run(p, cs, cfg, False, monkeypatch)
    mp = _run(p, cs, cfg, True, monkeypatch)
    for c, rb, rp in zip(cs, mb.results, mp.results):
        assert rb is not None and rp is not None
        assert len(rp.eigenvalues) == len(rb.eigenvalues) == c.expected_count
        assert _match(rp.eigenvalues, rb.eigenvalues) <= 1e-10
        assert rp.residuals.max() <= 1e-10
        assert rp.stats.n_factorizations == rb.stats.n_factorizations
        assert rp.stats.iterations == rb.stats.iterations


def test_pipelined_isolates_errors(monkeypatch):
    # a contour with nothing inside next to a normal one: per-contour errors stay isolated
    wl = W.config1(seed=0)
    p = DensePencil(wl.a, wl.b, hermitian=True)
    empty = Contour(shape="circle", center=-50.0 + 0j, radius=0.5, expected_count=1)
    cs = [wl.contours[0], empty]
    cfg = SolverConfig(n_q=wl.n_q, source_cols=wl.source_cols, n_moments=wl.n_moments)
    mb = _run(p, cs, cfg, False, monkeypatch)
    mp = _run(p, cs, cfg, True, monkeypatch)
    assert mp.results[1] is None and type(mp.errors[1]).__name__ == type(mb.errors[1]).__name__
    for i in (0,):
        assert len(mp.results[i].eigenvalues) == len(mb.results[i].eigenvalues)
        assert _match(mp.results[i].eigenvalues, mb.results[i].eigenvalues) <= 1e-10
