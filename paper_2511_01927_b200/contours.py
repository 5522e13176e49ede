"""Contour geometry and quadrature for the CIRR stage.

Restates the reference's ``Contour``/``QuadratureRule``/``quadrature_for``
(cieig/contours.py:26-137, 327-363) and adds the ellipse shape BASELINE
config 4 needs (the reference rejects unknown shapes at contours.py:40-50).
Reference ``Contour`` objects are accepted anywhere a contour is expected
(duck-typed on ``shape``/``center``/``radius``/rect bounds).
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np

from .errors import ParameterError


@dataclass(frozen=True)
class Contour:
    """Closed integration path: circle, axis-aligned rect, or ellipse."""

    shape: str  # "circle" | "rect" | "ellipse"
    center: complex = 0.0 + 0.0j  # circle / ellipse
    radius: float = 0.0  # circle
    re_min: float = 0.0  # rect
    re_max: float = 0.0
    im_min: float = 0.0
    im_max: float = 0.0
    semi_re: float = 0.0  # ellipse semi-axis along Re
    semi_im: float = 0.0  # ellipse semi-axis along Im
    expected_count: int = 0
    source: str = "manual"

    def __post_init__(self):  # contours.py:40-50 (+ ellipse)
        if self.shape == "circle":
            if self.radius <= 0:
                raise ParameterError("circle radius must be positive")
        elif self.shape == "rect":
            if self.re_min >= self.re_max or self.im_min >= self.im_max:
                raise ParameterError("rect bounds must be ordered")
            if self.source == "scout" and self.aspect_ratio() > 5.0 + 1e-12:
                raise ParameterError("scout rect aspect ratio must be <= 5")
        elif self.shape == "ellipse":
            if self.semi_re <= 0 or self.semi_im <= 0:
                raise ParameterError("ellipse semi-axes must be positive")
        else:
            raise ParameterError(f"unknown contour shape {self.shape!r}")

    def aspect_ratio(self) -> float:
        if self.shape == "circle":
            return 1.0
        if self.shape == "ellipse":
            return max(self.semi_re, self.semi_im) / min(self.semi_re, self.semi_im)
        w = self.re_max - self.re_min
        h = self.im_max - self.im_min
        return max(w, h) / min(w, h)

    def contains(self, z: complex, slack: float = 0.0) -> bool:
        return contains(self, z, slack)

    def area(self) -> float:
        if self.shape == "circle":
            return float(np.pi * self.radius**2)
        if self.shape == "ellipse":
            return float(np.pi * self.semi_re * self.semi_im)
        return (self.re_max - self.re_min) * (self.im_max - self.im_min)

    def to_json_dict(self) -> dict:  # contours.py:78-95 (+ ellipse)
        if self.shape == "circle":
            return {"shape": "circle", "center": [self.center.real, self.center.imag],
                    "radius": self.radius, "expected_count": self.expected_count,
                    "source": self.source}
        if self.shape == "ellipse":
            return {"shape": "ellipse", "center": [self.center.real, self.center.imag],
                    "semi_re": self.semi_re, "semi_im": self.semi_im,
                    "expected_count": self.expected_count, "source": self.source}
        return {"shape": "rect", "re_min": self.re_min, "re_max": self.re_max,
                "im_min": self.im_min, "im_max": self.im_max,
                "expected_count": self.expected_count, "source": self.source}

    @classmethod
    def from_json_dict(cls, d: dict) -> "Contour":
        common = dict(expected_count=int(d.get("expected_count", 0)),
                      source=d.get("source", "manual"))
        if d["shape"] == "circle":
            return cls(shape="circle", center=complex(d["center"][0], d["center"][1]),
                       radius=float(d["radius"]), **common)
        if d["shape"] == "ellipse":
            return cls(shape="ellipse", center=complex(d["center"][0], d["center"][1]),
                       semi_re=float(d["semi_re"]), semi_im=float(d["semi_im"]), **common)
        return cls(shape="rect", re_min=float(d["re_min"]), re_max=float(d["re_max"]),
                   im_min=float(d["im_min"]), im_max=float(d["im_max"]), **common)


def contours_to_json(contours) -> str:
    return json.dumps({"contours": [c.to_json_dict() for c in contours]})


def contours_from_json(text: str):
    return [Contour.from_json_dict(d) for d in json.loads(text)["contours"]]


def contains(c, z: complex, slack: float = 0.0) -> bool:
    """Strict interior test (contours.py:59-66); ellipse: ((x-c)/a)^2+(y/b)^2<1."""
    z = complex(z)
    if c.shape == "circle":
        return abs(z - c.center) < c.radius + slack
    if c.shape == "ellipse":
        dr = (z.real - c.center.real) / (c.semi_re + slack)
        di = (z.imag - complex(c.center).imag) / (c.semi_im + slack)
        return dr * dr + di * di < 1.0
    return (c.re_min - slack < z.real < c.re_max + slack
            and c.im_min - slack < z.imag < c.im_max + slack)


def contains_many(c, zs, slack: float = 0.0) -> np.ndarray:
    """contains() over an array, elementwise with the same float64 arithmetic:
    Python's abs(complex) is libm hypot, which np.hypot matches bit for bit
    (np.abs of complex128 does not: it differs in the last ulp for ~1/3 of
    values, enough to flip a boundary decision)."""
    z = np.asarray(zs, dtype=np.complex128)
    if c.shape == "circle":
        d = z - complex(c.center)
        return np.hypot(d.real, d.imag) < c.radius + slack
    if c.shape == "ellipse":
        dr = (z.real - complex(c.center).real) / (c.semi_re + slack)
        di = (z.imag - complex(c.center).imag) / (c.semi_im + slack)
        return dr * dr + di * di < 1.0
    return ((c.re_min - slack < z.real) & (z.real < c.re_max + slack)
            & (c.im_min - slack < z.imag) & (z.imag < c.im_max + slack))


def contains_rows(contours: list, zs: np.ndarray, counts) -> np.ndarray:
    """contains_many for many contours at once: row b of zs (first counts[b]
    entries) against contours[b]; the same float64 arithmetic per element."""
    z = np.asarray(zs, dtype=np.complex128)
    nb, k = z.shape
    out = np.zeros((nb, k), dtype=bool)
    valid = np.arange(k)[None, :] < np.asarray(counts)[:, None]
    shapes = np.array([c.shape for c in contours])
    for shape in set(shapes.tolist()):
        rows = np.flatnonzero(shapes == shape)
        cs = [contours[r] for r in rows]
        zz = z[rows]
        cen = np.array([complex(c.center) for c in cs]) if shape != "rect" else None
        if shape == "circle":
            d = zz - cen[:, None]
            m = np.hypot(d.real, d.imag) < np.array([c.radius for c in cs])[:, None]
        elif shape == "ellipse":
            dr = (zz.real - cen.real[:, None]) / np.array([c.semi_re for c in cs])[:, None]
            di = (zz.imag - cen.imag[:, None]) / np.array([c.semi_im for c in cs])[:, None]
            m = dr * dr + di * di < 1.0
        else:
            lo_r = np.array([c.re_min for c in cs])[:, None]
            hi_r = np.array([c.re_max for c in cs])[:, None]
            lo_i = np.array([c.im_min for c in cs])[:, None]
            hi_i = np.array([c.im_max for c in cs])[:, None]
            m = (lo_r < zz.real) & (zz.real < hi_r) & (lo_i < zz.imag) & (zz.imag < hi_i)
        out[rows] = m
    return out & valid


@dataclass(frozen=True)
class QuadratureRule:
    """sum_j w_j f(z_j) approximates (1/2 pi i) \\oint f(z) dz (contours.py:127-137)."""

    nodes: np.ndarray
    weights: np.ndarray

    @property
    def n_q(self) -> int:
        return len(self.nodes)


_UNIT_NODES: dict = {}


def _unit_nodes(n_q: int):
    """exp(i theta_j), cos theta_j, sin theta_j of the midpoint rule (read-only,
    memoised per n_q: the same arrays bit for bit, made once instead of per
    contour -- config 2 builds 512 rules per batch)."""
    v = _UNIT_NODES.get(n_q)
    if v is None:
        theta = 2.0 * np.pi * (np.arange(n_q) + 0.5) / n_q
        v = (np.exp(1j * theta), np.cos(theta), np.sin(theta))
        for a in v:
            a.setflags(write=False)
        _UNIT_NODES[n_q] = v
    return v


def quadrature_for(contour, n_q: int = 32) -> QuadratureRule:
    """Nodes/weights normalised so sum_j w_j/(z_j - c) -> 1 for an enclosed pole.

    Circle: midpoint trapezoid (contours.py:336-342).  Rect: Gauss-Legendre,
    n_q/4 per edge (contours.py:343-363).  Ellipse: midpoint trapezoid on
    z(t) = c + a cos t + i b sin t with w_j = z'(t_j)/(i n_q); identical to the
    circle rule when a == b.
    """
    if n_q < 4 or n_q % 2 != 0:
        raise ParameterError("n_q must be even and >= 4")
    if contour.shape in ("circle", "ellipse"):
        rot, ct, st = _unit_nodes(n_q)
        if contour.shape == "circle":
            return QuadratureRule(nodes=contour.center + contour.radius * rot,
                                  weights=contour.radius * rot / n_q)
        a, b = contour.semi_re, contour.semi_im
        return QuadratureRule(nodes=contour.center + (a * ct + 1j * b * st),
                              weights=(b * ct + 1j * a * st) / n_q)
    if n_q % 4 != 0:
        raise ParameterError("rect contours need n_q divisible by 4")
    per_edge = n_q // 4
    gl_x, gl_w = np.polynomial.legendre.leggauss(per_edge)
    corners = [complex(contour.re_min, contour.im_min), complex(contour.re_max, contour.im_min),
               complex(contour.re_max, contour.im_max), complex(contour.re_min, contour.im_max)]
    nodes, weights = [], []
    for k in range(4):  # counterclockwise edges
        p0, p1 = corners[k], corners[(k + 1) % 4]
        half = 0.5 * (p1 - p0)
        mid = 0.5 * (p1 + p0)
        nodes.append(mid + gl_x * half)
        weights.append(gl_w * half / (2.0j * np.pi))
    return QuadratureRule(nodes=np.concatenate(nodes), weights=np.concatenate(weights))


def moment_frame(contour) -> tuple[complex, float]:
    """(gamma, rho) for the centred, scaled moments ((z - gamma)/rho)^m.

    Circle: centre and radius; ellipse: centre and max semi-axis; rect: centre
    and max half-side.  Rescaling each moment block leaves span(S) unchanged
    (finding 1) but keeps the stacked block conditioned.
    """
    if contour.shape == "circle":
        return complex(contour.center), float(contour.radius)
    if contour.shape == "ellipse":
        return complex(contour.center), float(max(contour.semi_re, contour.semi_im))
    g = complex(0.5 * (contour.re_min + contour.re_max), 0.5 * (contour.im_min + contour.im_max))
    return g, float(max(0.5 * (contour.re_max - contour.re_min),
                        0.5 * (contour.im_max - contour.im_min)))


def contour_params(contour) -> tuple[int, float, float, float, float]:
    """(shape_code, p0, p1, p2, p3) for the device containment test.

    circle: (0, cr, ci, r, 0); ellipse: (1, cr, ci, a, b); rect: (2, re_min,
    re_max, im_min, im_max).
    """
    if contour.shape == "circle":
        c = complex(contour.center)
        return 0, c.real, c.imag, float(contour.radius), 0.0
    if contour.shape == "ellipse":
        c = complex(contour.center)
        return 1, c.real, c.imag, float(contour.semi_re), float(contour.semi_im)
    return 2, float(contour.re_min), float(contour.re_max), float(contour.im_min), float(contour.im_max)
