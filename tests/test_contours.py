"""Quadrature/contour restatement vs the reference (contours.py:327-363) and
its KATs (pkg/tests/test_contours.py:146-199)."""
import numpy as np
import pytest

from conftest import golden
from paper_2511_01927_b200.contours import (
    Contour, contains, contour_params, contours_from_json, contours_to_json, moment_frame, quadrature_for)
from paper_2511_01927_b200.errors import ParameterError


def circle(c, r, k=0):
    return Contour(shape="circle", center=complex(c), radius=r, expected_count=k)


def test_circle_rule_bitwise_reference():
    g = golden("ref_kats.npz")
    for nq in (4, 8, 32):
        r = quadrature_for(circle(0.3, 1.7), nq)
        assert np.array_equal(r.nodes, g[f"quad_circle_{nq}_nodes"])
        assert np.array_equal(r.weights, g[f"quad_circle_{nq}_weights"])


def test_rect_rule_bitwise_reference():
    g = golden("ref_kats.npz")
    r = quadrature_for(Contour(shape="rect", re_min=-1.0, re_max=2.0, im_min=-0.5, im_max=0.75), 16)
    assert np.array_equal(r.nodes, g["quad_rect_16_nodes"])
    assert np.array_equal(r.weights, g["quad_rect_16_weights"])


def test_centred_pole_sums_to_one():
    r = quadrature_for(circle(0.0, 1.0), 32)
    assert abs(np.sum(r.weights / (r.nodes - 0.0)) - 1.0) <= 1e-14


@pytest.mark.parametrize("nq", [4, 8, 32])
def test_weights_sum_to_zero(nq):
    assert abs(quadrature_for(circle(0.0, 1.0), nq).weights.sum()) <= 1e-14


def test_outside_pole_decays():
    for nq in (8, 16, 32):
        r = quadrature_for(circle(0.0, 1.0), nq)
        assert abs(np.sum(r.weights / (r.nodes - 2.0))) <= 10 * 0.5**nq


def test_parameter_errors():
    with pytest.raises(ParameterError):
        quadrature_for(circle(0.0, 1.0), 7)
    with pytest.raises(ParameterError):
        quadrature_for(Contour(shape="rect", re_min=0, re_max=1, im_min=0, im_max=1), 6)
    with pytest.raises(ParameterError):
        Contour(shape="ellipse", semi_re=0.0, semi_im=1.0)
    with pytest.raises(ParameterError):
        Contour(shape="triangle")


def test_ellipse_reduces_to_circle():
    e = Contour(shape="ellipse", center=0.5 + 0j, semi_re=0.7, semi_im=0.7)
    c = circle(0.5, 0.7)
    re_, rc = quadrature_for(e, 16), quadrature_for(c, 16)
    assert np.allclose(re_.nodes, rc.nodes, atol=1e-15) and np.allclose(re_.weights, rc.weights, atol=1e-15)


@pytest.mark.parametrize("pole,inside", [(0.5 + 0.05j, True), (0.75, True), (0.5 + 0.3j, False), (0.95, False)])
def test_ellipse_resolvent_filter(pole, inside):
    e = Contour(shape="ellipse", center=0.5 + 0j, semi_re=0.3, semi_im=0.15)
    r = quadrature_for(e, 64)
    val = np.sum(r.weights / (r.nodes - pole))
    assert abs(val - (1.0 if inside else 0.0)) < 1e-6
    assert contains(e, pole) is inside


def test_json_round_trip_and_params():
    cs = [circle(1.0, 2.0, 3), Contour(shape="ellipse", center=-0.5 + 0j, semi_re=0.3, semi_im=0.15),
          Contour(shape="rect", re_min=0, re_max=1, im_min=-1, im_max=1)]
    assert contours_from_json(contours_to_json(cs)) == cs
    assert contour_params(cs[1]) == (1, -0.5, 0.0, 0.3, 0.15)
    assert moment_frame(cs[0]) == (1.0 + 0j, 2.0)
    assert moment_frame(cs[1]) == (-0.5 + 0j, 0.3)
