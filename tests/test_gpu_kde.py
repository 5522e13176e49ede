"""Device KDE density under the reference's OWN contour
construction: `patch.install(cieig)` points `cieig.contours.kde_eval`
(contours.py:20, called at :191) at `cirr_kde_eval`, and the unmodified
`construct_contours` / `find_cut` / `kde_sparsity` (contours.py:175-320) run on
it. Checked against the reference's numba outputs (tests/golden/
make_kde_golden.py -> ref_kde.npz, ref_thermal.npz) and the reference's own
KDE unit cases (pkg/tests/test_contours.py:33-138)."""
import json
import os

import numpy as np
import pytest

from conftest import reference_cieig

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "ref_kde.npz"))


@pytest.fixture(scope="module")
def C():
    """cieig.contours with the device density patched in."""
    if not torch.cuda.is_available():
        pytest.fail("gpu test without CUDA")
    cieig = reference_cieig()
    from paper_2511_01927_b200 import kde

    calls = []
    kde.install(cieig)
    orig = cieig.contours.kde_eval
    cieig.contours.kde_eval = lambda *a: calls.append(1) or orig(*a)
    yield cieig.contours
    assert calls, "the reference did not evaluate its density through the device kernel"
    cieig.contours.kde_eval = orig
    kde.uninstall(cieig)


def _pred(C, v):
    return C.SpectrumPrediction(values=np.asarray(v, dtype=float))


def test_kde_eval_matches_reference():
    if not torch.cuda.is_available():
        pytest.fail("gpu test without CUDA")
    from paper_2511_01927_b200 import kde_eval
    got = kde_eval(G["kde_ts"], G["kde_eigs"], float(G["kde_coef"]))
    ref = G["kde_out"]
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()
    assert kde_eval(np.zeros(0), G["kde_eigs"], 1.0).shape == (0,)
    assert np.array_equal(kde_eval(np.array([0.5, 1.0]), np.zeros(0), 1.0), [0.0, 0.0])


def test_patch_routes_contours_density():
    cieig = reference_cieig()
    from paper_2511_01927_b200 import kde, patch
    patch.install(cieig)
    try:
        assert cieig.contours.kde_eval is kde.kde_eval
    finally:
        patch.uninstall(cieig)
    assert cieig.contours.kde_eval is not kde.kde_eval


def test_reference_kde_unit_cases(C):
    assert C.kde_sparsity(0.0, 1.0, [0.5], 7.0, 0.5) == pytest.approx(1.0)
    assert C.kde_sparsity(0.0, 1.0, [], 10.0, 0.3) == 0.0
    assert C.kde_sparsity(0.0, 1.0, [0.0, 1.0], 10.0, 0.5) == pytest.approx(2.0 * np.exp(-2.5), rel=1e-14)
    assert C.find_cut(0.0, 1.0, [0.0, 1.0], 10.0) == pytest.approx(0.5, abs=1e-8)
    assert C.find_cut(0.3, 0.7, [0.3, 0.7], 25.0) == pytest.approx(0.5, abs=1e-8)
    got = C.find_cut(0.0, 1.0, [0.1, 0.2, 0.9], 10.0)
    assert got == pytest.approx(0.5998453835765787, abs=1e-6) and 0.2 < got < 0.9


def test_reference_partition_cases(C):
    values = np.linspace(0.0, 1.0, 30)
    _, cs = C.construct_contours(_pred(C, values))
    assert len(cs) == 1 and cs[0].expected_count == 30
    values = np.concatenate([np.linspace(0.0, 1.0, 30), np.linspace(9.0, 10.0, 30)])
    part, cs = C.construct_contours(_pred(C, values), n_min=10, n_max=50, w=10.0)
    assert len(cs) == 2 and 1.0 < part.intervals[0].end < 9.0
    assert [iv.count for iv in part.intervals] == [30, 30]
    rng = np.random.default_rng(0)
    values = np.sort(rng.uniform(-3.0, 5.0, 120))
    part, cs = C.construct_contours(_pred(C, values), n_min=10, n_max=50)
    assert sum(iv.count for iv in part.intervals) == 120
    for v in values:
        assert any(c.contains(complex(v, 0.0)) for c in cs)


@pytest.mark.parametrize("case", [str(c) for c in G["cases"]])
def test_partition_matches_reference(C, case):
    vals = G[f"{case}_values"]
    nmin, nmax, w = G[f"{case}_params"]
    part, cs = C.construct_contours(_pred(C, vals), n_min=int(nmin), n_max=int(nmax), w=float(w))
    ref = G[f"{case}_iv"]
    got = np.array([[iv.start, iv.end, iv.count] for iv in part.intervals])
    assert got.shape == ref.shape
    assert np.array_equal(got[:, 2], ref[:, 2])                      # same counts
    span = vals[-1] - vals[0]
    assert np.abs(got[:, :2] - ref[:, :2]).max() <= 1e-9 * span      # same cuts (golden-section 1e-10 width)
    assert all(c.source == "kde" and c.shape == "circle" for c in cs)


def test_thermal20_contours_match_reference(C):
    T = np.load(os.path.join(HERE, "golden", "ref_thermal.npz"))
    ref = json.loads(str(T["t20_kde_contours"]))
    _, cs = C.construct_contours(_pred(C, T["t20_kde_truth"]), n_min=1, n_max=50)
    assert len(cs) == len(ref)
    for c, r in zip(cs, ref):
        assert c.expected_count == r["expected_count"]
        d = c.to_json_dict()
        assert d["center"] == pytest.approx(r["center"], rel=1e-9)
        assert abs(c.radius - r["radius"]) <= 1e-9 * r["radius"]
