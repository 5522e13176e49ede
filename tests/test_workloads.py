"""Input generators for the BASELINE configs."""
import numpy as np
import pytest

from conftest import golden
from paper_2511_01927_b200 import workloads as W


def test_grf_2d_bitwise_reference():
    g = golden("ref_grf.npz")
    for s in range(3):
        assert np.array_equal(W.grf_2d(16, 16, 1.0, 0.5, 0.2, s), g[f"c2_s{s}"])
    assert np.array_equal(W.grf_2d(48, 48, 1.0, 0.5, 0.2, 0), g["c3_s0"])
    assert np.array_equal(W.grf_2d(10, 10, 1.0, 0.1, 0.2, 7), g["t10_s7"])


def test_config1_structure():
    a, b = W.config1_matrices()
    assert a.shape == (512, 512)
    assert np.array_equal(a, a.T) and np.array_equal(b, b.T)
    assert np.count_nonzero(np.triu(a, 2)) == 0
    np.linalg.cholesky(b)


def test_config2_3_spd():
    for a, b in (W.config2_matrices(0), W.config3_matrices()):
        assert np.allclose(a, a.T)
        np.linalg.cholesky(a)
        assert np.count_nonzero(b - np.diag(np.diag(b))) == 0 and (np.diag(b) > 0).all()


def test_config4_small_variant():
    a, b = W.config4_matrices(0, n=64)
    assert a.shape == (64, 64) and not np.allclose(a, a.T)
    assert np.abs(np.diag(b) - 1.0).max() < 0.05 * 5 / 8


def test_config5_small_grid_spd():
    a, b = W.config5_matrices(0, nx=5)
    assert a.shape == (125, 125)
    assert np.array_equal(b, b.T) and np.array_equal(a, a.T)
    w = np.linalg.eigvalsh(b)
    assert w.min() > 0 and w.max() / w.min() < 1e3


def test_contour_fixtures_match_generators():
    import json
    o1 = golden("oracle_config1.npz")
    c = json.loads(str(o1["contours"]))[0]
    wl = W.config1()
    assert abs(c["center"][0] - wl.contours[0].center.real) < 1e-9 * abs(c["center"][0])
    assert c["expected_count"] == 33


def test_largest_gap_cut():
    eigs = np.array([1.0, 2.0, 3.0, 3.1, 10.0, 11.0, 12.0])
    assert W.largest_gap_cut(eigs, 3) == 4
