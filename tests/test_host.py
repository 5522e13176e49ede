"""Host-side logic of the drop-in (no GPU needed)."""
import ast
import os

import numpy as np
import pytest

from paper_2511_01927_b200 import solvers as S
from paper_2511_01927_b200.contours import Contour
from paper_2511_01927_b200.errors import DeviceError, ParameterError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_solver_config_validation():
    with pytest.raises(ParameterError):
        S.SolverConfig(n_q=2)
    with pytest.raises(ParameterError):
        S.SolverConfig(tol=0.0)
    assert S.SolverConfig().cols_for(3) == 8 and S.SolverConfig().cols_for(10) == 20
    assert S.SolverConfig(source_cols=5).cols_for(100) == 5


def test_sidecar_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    block = rng.standard_normal((7, 3)) + 1j * rng.standard_normal((7, 3))
    path = tmp_path / "v.bin"
    S.write_eigenvectors(path, block)
    assert path.stat().st_size == 16 + 7 * 3 * 16
    assert np.array_equal(S.read_eigenvectors(path), block)


def _res(vals, resid, c=None):
    return S.EigenResult(np.array(vals), np.zeros((2, len(vals))), np.array(resid), c, S.SolveStats())


def test_dedupe_keeps_smaller_residual():
    rs = [_res([1.0, 2.0], [1e-12, 5e-11]), _res([2.0 + 1e-12, 3.0], [1e-13, 1e-12])]
    S._dedupe(rs)
    assert list(rs[0].eigenvalues) == [1.0]
    assert len(rs[1].eigenvalues) == 2


def test_dedupe_complex_values():
    rs = [_res([0.5 + 0.1j, -0.5 + 0.0j], [1e-12, 1e-12]), _res([0.5 + 0.1j + 1e-13], [1e-11])]
    S._dedupe(rs)
    assert len(rs[0].eigenvalues) == 2 and len(rs[1].eigenvalues) == 0


def test_moment_coefficients_match_oracle():
    from oracle.cirr import moment_frame as ofr, quadrature as oq
    e = Contour(shape="ellipse", center=0.5 + 0j, semi_re=0.3, semi_im=0.15)
    c = S._Contour(0, e, S.SolverConfig(n_q=64, n_moments=8), 0, 10)
    nodes, w = oq(e, 64)
    g, r = ofr(e)
    assert np.array_equal(c.nodes, nodes) and (c.gamma, c.rho) == (g, r)
    coef = c.coef(8)
    for j in (0, 17, 63):
        zp, zeta = 1.0 + 0j, (nodes[j] - g) / r
        for m in range(8):
            assert coef[j, m] == w[j] * zp
            zp *= zeta


def test_waves_group_whole_contours():
    cs = [S._Contour(i, Contour(shape="circle", center=0j, radius=1.0), S.SolverConfig(n_q=32), 0, 100)
          for i in range(5)]
    from paper_2511_01927_b200 import _lib
    per = 100 * 100 * 16 + _lib.call("cirr_diag_inv_bytes", 100, 1) + _lib.call("cirr_zgetrf_ws_bytes", 100, 1)
    waves = S._waves(cs, 100, budget_bytes=per * 64)
    assert [len(w) for w in waves] == [2, 2, 1]


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2511_01927_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            tree = ast.parse(open(os.path.join(pkg, fn)).read())
            for node in ast.walk(tree):
                if isinstance(node, ast.Import):
                    assert not any(a.name.split(".")[0] == "oracle" for a in node.names), fn
                if isinstance(node, ast.ImportFrom) and node.module:
                    assert node.module.split(".")[0] != "oracle", fn


def test_no_cuda_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(DeviceError):
        S.cirr_solve(type("P", (), {"a": np.eye(2), "b": np.eye(2), "hermitian": True})(),
                     Contour(shape="circle", center=1 + 0j, radius=0.5))


def test_conjugate_pair_selection():
    """Conjugate-pair variant: upper-half nodes factor, lower half mirrors."""
    from paper_2511_01927_b200.solvers import SolverConfig, _Contour
    from paper_2511_01927_b200 import Contour

    cfg = SolverConfig(n_q=32, conjugate_pairs=True)
    for c in (Contour(shape="circle", center=1.5 + 0j, radius=0.7),
              Contour(shape="ellipse", center=-0.5 + 0j, semi_re=0.3, semi_im=0.15)):
        st = _Contour(0, c, cfg, 0, 10)
        assert st.half and len(st.fidx) == 16
        z = st.nodes
        assert np.all(z[st.fidx].imag > 0)
        for j in range(32):
            src = z[st.fidx[st.mate[j]]]
            assert abs(src - (z[j] if z[j].imag > 0 else np.conj(z[j]))) <= 1e-13
    assert not _Contour(0, Contour(shape="circle", center=0.2 + 0.3j, radius=0.5), cfg, 0, 10).half
    assert not _Contour(0, Contour(shape="circle", center=1.0 + 0j, radius=0.5),
                        SolverConfig(n_q=32), 0, 10).half


def test_solve_multi_batch_validates_before_upload():
    """solve_multi_batch argument checks run before any device work (so they
    hold without a GPU): solver name, one contour list and one seed per pencil."""
    from paper_2511_01927_b200.errors import DimensionError
    a = np.eye(4)
    c = Contour(shape="circle", center=1 + 0j, radius=0.5)
    pen = [(a, a), (a, a)]
    assert S.solve_multi_batch([], [[c]]) == []
    with pytest.raises(ParameterError):
        S.solve_multi_batch(pen, [[c], [c]], solver="lanczos")
    with pytest.raises(DimensionError):
        S.solve_multi_batch(pen, [[c]])
    with pytest.raises(DimensionError):
        S.solve_multi_batch(pen, [[c], [c]], seeds=[0])


def test_contains_many_matches_contains():
    """The vectorised inside test makes the same decisions as contains() on
    boundary-hugging values of every shape."""
    from paper_2511_01927_b200.contours import contains, contains_many
    rng = np.random.default_rng(7)
    shapes = [Contour(shape="circle", center=0.3 + 0.1j, radius=0.7),
              Contour(shape="ellipse", center=-0.5 + 0j, semi_re=0.3, semi_im=0.15),
              Contour(shape="rect", re_min=-1.0, re_max=2.0, im_min=-0.5, im_max=0.25)]
    for c in shapes:
        th = rng.uniform(0, 2 * np.pi, 400)
        z = np.concatenate([c.center + 1.2 * (rng.standard_normal(400) + 1j * rng.standard_normal(400)),
                            (complex(getattr(c, "center", 0.5 - 0.125j)) + (1 + rng.uniform(-1e-15, 1e-15, 400))
                             * np.exp(1j * th) * getattr(c, "radius", getattr(c, "semi_re", 1.5)))])
        for slack in (0.0, 1e-3):
            got = contains_many(c, z, slack)
            want = np.array([contains(c, v, slack) for v in z])
            assert np.array_equal(got, want)


def test_single_moment_coefficients_bitwise():
    """The moments == 1 fast path equals the sequential-power loop bit for bit."""
    for shape in ("circle", "ellipse"):
        c = Contour(shape=shape, center=0.5 - 0.25j, radius=0.3, semi_re=0.3, semi_im=0.15)
        st = S._Contour(0, c, S.SolverConfig(n_q=64, n_moments=8), 0, 10)
        fast = st._coef(1)
        loop = np.empty((len(st.nodes), 1), dtype=np.complex128)
        for j, w in enumerate(st.weights):
            loop[j, 0] = w * (1.0 + 0.0j)
        assert np.array_equal(fast.view(np.float64), loop.view(np.float64))
        assert np.array_equal(np.ascontiguousarray(fast[:, 0]).view(np.float64),
                              np.ascontiguousarray(st._coef(4)[:, 0]).view(np.float64))


def test_dedupe_complex_conjugate_pairs_from_overlapping_contours():
    """a lexicographic sort does not bring near-equal complex values
    together; two overlapping contours each finding a conjugate pair must end
    with one copy of each value, the smaller-residual one."""
    a, b = 0.5 + 0.1j, 0.5 - 0.1j
    eps = 1e-13
    rs = [_res([a, b + eps * 1j, 0.9 + 0j], [1e-12, 3e-12, 1e-12]),
          _res([b, a + eps, 0.1 + 0j], [1e-12, 5e-12, 1e-12])]
    S._dedupe(rs)
    union = np.concatenate([r.eigenvalues for r in rs])
    assert len(union) == 4
    for v in (a, b, 0.9, 0.1):
        assert np.sum(np.abs(union - v) <= 1e-10) == 1
    assert a in rs[0].eigenvalues and b in rs[1].eigenvalues     # the smaller residuals survive


def test_dedupe_complex_same_contour_never_dropped():
    rs = [_res([0.5 + 0.1j, 0.5 + 0.1j + 1e-14], [1e-12, 1e-12])]
    rs.append(_res([2.0 + 0j], [1e-12]))
    S._dedupe(rs)
    assert len(rs[0].eigenvalues) == 2


class _FakeContour:
    def __init__(self, p):
        self.fidx = np.arange(p)
        self.nodes = np.zeros(p)


def test_waves_cap_pencils_per_wave():
    """batch indices ride on grid.y/z (<= 65535); a wave never holds
    more pencils, whatever the byte budget."""
    cs = [_FakeContour(16) for _ in range(4200)]          # 67200 pencils
    waves = S._waves(cs, 16, 1 << 60)
    assert len(waves) == 2
    assert all(sum(len(c.fidx) for c in w) <= S._MAX_WAVE_PENCILS for w in waves)
    assert sum(len(w) for w in waves) == 4200
    # the byte budget counts the factor, its diagonal inverses and LU workspace
    per = 64 * 64 * 16
    assert len(S._waves([_FakeContour(32), _FakeContour(32)], 64, 64 * per + 1)) == 2


def test_contains_rows_equals_contains_many():
    """The batched containment of a Rayleigh-Ritz round equals contains_many
    per contour (same arithmetic), for every shape, honouring the counts."""
    from paper_2511_01927_b200.contours import contains_many, contains_rows
    rng = np.random.default_rng(7)
    cs = [Contour(shape="circle", center=0.1 + 0.2j, radius=0.5),
          Contour(shape="ellipse", center=-0.3 + 0j, semi_re=0.4, semi_im=0.2),
          Contour(shape="rect", re_min=-0.5, re_max=0.5, im_min=-0.1, im_max=0.3),
          Contour(shape="circle", center=1.0 + 0j, radius=0.25)]
    z = rng.uniform(-1.2, 1.2, (4, 50)) + 1j * rng.uniform(-0.6, 0.6, (4, 50))
    counts = [50, 17, 0, 33]
    got = contains_rows(cs, z, counts)
    for b, c in enumerate(cs):
        ref = contains_many(c, z[b])
        ref[counts[b]:] = False
        assert np.array_equal(got[b], ref)


def test_solver_config_arith_option():
    from paper_2511_01927_b200 import SolverConfig
    from paper_2511_01927_b200.errors import ParameterError
    assert SolverConfig().arith is None and SolverConfig(arith="f64").arith == "f64"
    with pytest.raises(ParameterError):
        SolverConfig(arith="fp16")
