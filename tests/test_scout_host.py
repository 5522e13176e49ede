"""Host arithmetic of the scouts (scout_contour, calibrate_margin), mirroring
the reference's pkg/tests/test_scouting.py:57-95 (no GPU needed)."""
import numpy as np
import pytest

from paper_2511_01927_b200.errors import EmptyPredictionError, ParameterError, ParameterWarning
from paper_2511_01927_b200.scouting import RitzEstimate, calibrate_margin, scout_contour


def _ritz(values):
    return RitzEstimate(method="lanczos", k_iters=60, ritz_values=np.asarray(values, dtype=float), elapsed=0.0)


class _Truth:
    def __init__(self, eigs):
        self.eigenvalues = np.asarray(eigs, dtype=float)


def test_scout_contour_margin_arithmetic():
    c = scout_contour(_ritz([1.0, 5.0]), 1.2)
    assert c.re_min == pytest.approx(0.6)
    assert c.re_max == pytest.approx(5.4)
    assert c.shape == "rect" and c.source == "scout" and c.expected_count == 2
    assert (c.im_max - c.im_min) == pytest.approx((c.re_max - c.re_min) / 5.0)


def test_scout_contour_identity_margin():
    c = scout_contour(_ritz([1.0, 5.0]), 1.0)
    assert c.re_min == 1.0 and c.re_max == 5.0


def test_scout_contour_degenerate_span_warns():
    with pytest.warns(ParameterWarning):
        c = scout_contour(_ritz([2.0, 2.0]), 1.2)
    assert c.re_min < 2.0 < c.re_max


def test_scout_contour_rejects():
    with pytest.raises(ParameterError):
        scout_contour(_ritz([1.0, 2.0]), 0.9)
    with pytest.raises(EmptyPredictionError):
        scout_contour(_ritz([]), 1.2)


def test_calibrate_margin_already_contained():
    assert calibrate_margin(_ritz([1.0, 5.0]), _Truth([2.0, 3.0])) == 1.0


def test_calibrate_margin_one_sided_overshoot():
    mf = calibrate_margin(_ritz([1.0, 5.0]), _Truth([1.0, 5.2]))
    c = scout_contour(_ritz([1.0, 5.0]), mf)
    assert c.re_max >= 5.2
    c_prev = scout_contour(_ritz([1.0, 5.0]), mf - 0.01)
    assert c_prev.re_max < 5.2
    with pytest.raises(ParameterError):
        calibrate_margin(_ritz([1.0, 5.0]), _Truth([2.0]), step=0.0)
