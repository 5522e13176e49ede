"""Device Krylov scouts against the unmodified
reference `scout` (tests/golden/make_scout_golden.py -> ref_scout.npz), and
the reference's own scouting tests (pkg/tests/test_scouting.py:22-55)."""
import os

import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "ref_scout.npz"))
METHODS = ("lanczos", "arnoldi", "krylov-schur-restarted")


@pytest.fixture(scope="module")
def sc():
    if not torch.cuda.is_available():
        pytest.fail("gpu test without CUDA")
    from paper_2511_01927_b200 import scouting
    return scouting


def _t20():
    n = int(G["t20_n"])
    a = sp.csr_matrix((G["t20_a_data"], G["t20_a_indices"], G["t20_a_indptr"]), shape=(n, n)).toarray()
    b = sp.csr_matrix((G["t20_b_data"], G["t20_b_indices"], G["t20_b_indptr"]), shape=(n, n)).toarray()
    return a.real, b.real


@pytest.mark.parametrize("method", METHODS)
def test_scout_matches_reference(sc, method):
    """Same Ritz values as the reference scout on the same pencil, budget and
    seed: diag(1..100) (full and partial Krylov), thermal20, config 3."""
    diag = (np.diag(np.arange(1.0, 101.0)), np.eye(100))
    est = sc.scout(diag, method, 100, 5, seed=0)
    assert np.allclose(est.ritz_values, np.arange(1.0, 6.0), atol=1e-8)      # test_scouting.py:24-29
    assert np.allclose(est.ritz_values, G[f"diag100_full_{method}"], rtol=1e-10, atol=0)
    est = sc.scout(diag, method, 30, 3, seed=1)
    assert np.abs(est.ritz_values - np.array([1.0, 2.0, 3.0])).max() <= 1e-6  # test_scouting.py:32-37
    assert np.allclose(est.ritz_values, G[f"diag100_part_{method}"], rtol=1e-9, atol=0)
    m = int(G["t20_m"])
    est = sc.scout(_t20(), method, 60, m, seed=2)
    assert est.method == method and est.k_iters == 60 and len(est.ritz_values) == m
    assert np.allclose(est.ritz_values, G[f"t20_{method}"], rtol=1e-9, atol=0)
    from paper_2511_01927_b200 import workloads as W
    est = sc.scout(W.config3_matrices(), method, 100, 32, seed=3)
    assert np.allclose(est.ritz_values, G[f"cfg3_{method}"], rtol=1e-9, atol=0)


def test_scout_errors(sc):
    from paper_2511_01927_b200.errors import ParameterError, SingularShiftError
    a, b = _t20()
    with pytest.raises(ParameterError):
        sc.scout((a, b), "lanczos", 3, 4, seed=0)                          # test_scouting.py:47-49
    with pytest.raises(ParameterError):
        sc.scout((a, b), "power-iteration", 60, 4, seed=0)                 # test_scouting.py:52-54
    z = np.diag(np.array([1.0, 0.0, 2.0]))
    with pytest.raises(SingularShiftError):
        sc.scout((z, np.eye(3)), "lanczos", 3, 1, seed=0)                  # singular A: shift 0 hits an eigenvalue
