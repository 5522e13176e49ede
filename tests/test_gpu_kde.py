"""Device KDE contour construction against the
unmodified reference (tests/golden/make_kde_golden.py -> ref_kde.npz,
ref_thermal.npz) and the reference's own KDE tests
(pkg/tests/test_contours.py:33-138)."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "ref_kde.npz"))


@pytest.fixture(scope="module")
def K():
    if not torch.cuda.is_available():
        pytest.fail("gpu test without CUDA")
    from paper_2511_01927_b200 import kde
    return kde


def _pred(K, v):
    return K.SpectrumPrediction(values=np.asarray(v, dtype=float))


def test_kde_eval_matches_reference(K):
    got = K.kde_eval(G["kde_ts"], G["kde_eigs"], float(G["kde_coef"]))
    ref = G["kde_out"]
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()


def test_reference_kde_unit_cases(K):
    assert K.kde_sparsity(0.0, 1.0, [0.5], 7.0, 0.5) == pytest.approx(1.0)
    assert K.kde_sparsity(0.0, 1.0, [], 10.0, 0.3) == 0.0
    assert K.kde_sparsity(0.0, 1.0, [0.0, 1.0], 10.0, 0.5) == pytest.approx(2.0 * np.exp(-2.5), rel=1e-14)
    assert K.find_cut(0.0, 1.0, [0.0, 1.0], 10.0) == pytest.approx(0.5, abs=1e-8)
    assert K.find_cut(0.3, 0.7, [0.3, 0.7], 25.0) == pytest.approx(0.5, abs=1e-8)
    got = K.find_cut(0.0, 1.0, [0.1, 0.2, 0.9], 10.0)
    assert got == pytest.approx(0.5998453835765787, abs=1e-6) and 0.2 < got < 0.9
    from paper_2511_01927_b200.errors import CutUndefinedError, EmptyPredictionError, ParameterError
    with pytest.raises(CutUndefinedError):
        K.find_cut(0.0, 1.0, [0.5], 10.0)
    with pytest.raises(EmptyPredictionError):
        K.SpectrumPrediction(values=np.array([]))
    with pytest.raises(ParameterError):
        K.construct_contours(_pred(K, [1.0, 2.0]), n_min=5, n_max=2)


def test_reference_partition_cases(K):
    values = np.linspace(0.0, 1.0, 30)
    _, cs = K.construct_contours(_pred(K, values))
    assert len(cs) == 1 and cs[0].expected_count == 30
    values = np.concatenate([np.linspace(0.0, 1.0, 30), np.linspace(9.0, 10.0, 30)])
    part, cs = K.construct_contours(_pred(K, values), n_min=10, n_max=50, w=10.0)
    assert len(cs) == 2 and 1.0 < part.intervals[0].end < 9.0
    assert [iv.count for iv in part.intervals] == [30, 30]
    rng = np.random.default_rng(0)
    values = np.sort(rng.uniform(-3.0, 5.0, 120))
    part, cs = K.construct_contours(_pred(K, values), n_min=10, n_max=50)
    assert sum(iv.count for iv in part.intervals) == 120
    for v in values:
        assert any(c.contains(complex(v, 0.0)) for c in cs)
    p1, c1 = K.construct_contours(_pred(K, values))
    p2, c2 = K.construct_contours(_pred(K, values))
    assert p1 == p2 and c1 == c2


@pytest.mark.parametrize("case", [str(c) for c in G["cases"]])
def test_partition_matches_reference(K, case):
    vals = G[f"{case}_values"]
    nmin, nmax, w = G[f"{case}_params"]
    part, cs = K.construct_contours(_pred(K, vals), n_min=int(nmin), n_max=int(nmax), w=float(w))
    ref = G[f"{case}_iv"]
    got = np.array([[iv.start, iv.end, iv.count] for iv in part.intervals])
    assert got.shape == ref.shape
    assert np.array_equal(got[:, 2], ref[:, 2])                      # same counts
    span = vals[-1] - vals[0]
    assert np.abs(got[:, :2] - ref[:, :2]).max() <= 1e-9 * span      # same cuts (golden-section 1e-10 width)
    assert all(c.source == "kde" and c.shape == "circle" for c in cs)


def test_thermal20_contours_match_reference(K):
    T = np.load(os.path.join(HERE, "golden", "ref_thermal.npz"))
    ref = json.loads(str(T["t20_kde_contours"]))
    _, cs = K.construct_contours(_pred(K, T["t20_kde_truth"]), n_min=1, n_max=50)
    assert len(cs) == len(ref)
    for c, r in zip(cs, ref):
        assert c.expected_count == r["expected_count"]
        cr = r["center"]
        cre = cr[0] if isinstance(cr, (list, tuple)) else (cr["re"] if isinstance(cr, dict) else complex(cr).real)
        assert abs(c.center.real - cre) <= 1e-9 * abs(cre) and abs(c.radius - r["radius"]) <= 1e-9 * r["radius"]
