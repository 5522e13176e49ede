"""Drop-in test: the UNMODIFIED reference pipeline (cieig, installed under
baseline/_ref) running its own bench strategies and CLI with the GPU CIRR
path patched in (paper_2511_01927_b200.patch), against the same pipeline on
its own CPU solver."""
import json
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
if not os.path.isdir(os.path.join(REF, "cieig")):
    pytest.skip("reference package not installed under baseline/_ref", allow_module_level=True)
sys.path.insert(0, REF)

import cieig  # noqa: E402
import cieig.bench as rb  # noqa: E402
import cieig.cli as rcli  # noqa: E402
import cieig.problems as rp  # noqa: E402

from paper_2511_01927_b200 import patch  # noqa: E402


@pytest.fixture(scope="module")
def thermal():
    p = rp.assemble_thermal(rp.grf_sample(rp.Grid2D(20, 20), 1.0, 0.1, 0.2, seed=11), 1.0)
    return p, rp.dense_ground_truth(p, rp.target_count(p.n) * 4)


@pytest.mark.parametrize("strategy", ["oracle-kde", "scout-lanczos", "random"])
def test_bench_strategy_dropin(thermal, strategy):
    pencil, truth = thermal
    cfg = rb.BenchConfig()
    cpu = rb.run_strategy(pencil, truth, strategy, 1e-10, cfg, seed=0)
    patch.install(cieig)
    try:
        calls = []
        orig = cieig.bench.solve_multi
        cieig.bench.solve_multi = lambda *a, **k: calls.append(1) or orig(*a, **k)
        gpu = rb.run_strategy(pencil, truth, strategy, 1e-10, cfg, seed=0)
        cieig.bench.solve_multi = orig
    finally:
        patch.uninstall(cieig)
    assert calls, "bench did not route through the patched solve_multi"
    assert gpu.missed == cpu.missed
    assert gpu.found == cpu.found


def test_solvers_cirr_solve_patched_errors(thermal):
    pencil, truth = thermal
    from cieig.contours import Contour
    far = Contour(shape="circle", center=complex(1e6), radius=1.0, expected_count=1)
    patch.install(cieig)
    try:
        m = cieig.solvers.solve_multi(pencil, [far], cieig.solvers.SolverConfig())
        assert isinstance(m.errors[0], cieig.errors.NoEigenvaluesFound)
        with pytest.raises(cieig.errors.NoEigenvaluesFound):
            cieig.solvers.cirr_solve(pencil, far)
        assert cieig.solvers.cirr_solve is not patch._ORIG["solvers.cirr_solve"]
    finally:
        patch.uninstall(cieig)


def test_cli_solve_dropin(tmp_path):
    ds = tmp_path / "ds"
    assert rcli.main(["gen", "--problem", "thermal", "--grid", "12", "--seed", "1", "--out", str(ds)]) == 0
    assert rcli.main(["truth", "--in", str(ds)]) == 0
    cont = tmp_path / "c.json"
    assert rcli.main(["contour", "--in", str(ds), "--strategy", "kde", "--out", str(cont)]) == 0
    out_cpu, out_gpu = tmp_path / "cpu.json", tmp_path / "gpu.json"
    vec = tmp_path / "v.bin"
    assert rcli.main(["solve", "--in", str(ds), "--contours", str(cont), "--out", str(out_cpu)]) == 0
    patch.install(cieig)
    try:
        assert rcli.main(["solve", "--in", str(ds), "--contours", str(cont), "--out", str(out_gpu),
                          "--vectors", str(vec)]) == 0
    finally:
        patch.uninstall(cieig)
    a = json.load(open(out_cpu))["eigenvalues"]
    b = json.load(open(out_gpu))["eigenvalues"]
    assert len(a) == len(b) and np.allclose(a, b, rtol=1e-9)
    assert vec.stat().st_size > 16


def test_feast_dropin(thermal):
    pencil, truth = thermal
    from cieig.contours import Contour
    c = Contour(shape="circle", center=complex(0.5 * (truth.eigenvalues[0] + truth.eigenvalues[3])),
                radius=0.5 * (truth.eigenvalues[4] - truth.eigenvalues[0]) + 1e-9 * truth.eigenvalues[4],
                expected_count=4)
    cfg = cieig.solvers.SolverConfig(tol=1e-9)
    cpu = cieig.solvers.solve_multi(pencil, [c], cfg, solver="feast", seed=0)
    patch.install(cieig)
    try:
        gpu = cieig.solvers.solve_multi(pencil, [c], cfg, solver="feast", seed=0)
        r = cieig.solvers.feast_solve(pencil, c, cfg, seed=0)
        assert isinstance(r, cieig.solvers.EigenResult)
    finally:
        patch.uninstall(cieig)
    assert len(gpu.eigenvalues) == len(cpu.eigenvalues)
    assert np.allclose(gpu.eigenvalues, cpu.eigenvalues, rtol=1e-8)
