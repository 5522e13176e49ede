"""Dataset ingestion: Matrix Market + meta.json as the
reference writes them.  Fixtures: tests/golden/dataset_thermal8 (written by the
unmodified reference's problems.write_dataset) and ref_dataset.npz (its dense
matrices, truth, and the reference's FormatError text for malformed files),
both made by tests/golden/make_golden.py."""
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden
from paper_2511_01927_b200 import FormatError, read_dataset, read_matrix_market, write_dataset

FIX = os.path.join(GOLDEN, "dataset_thermal8")


def test_reads_reference_dataset_bitwise():
    ref = golden("ref_dataset.npz")
    ds = read_dataset(FIX)
    assert np.array_equal(ds.pencil.a.toarray(), ref["a"])
    assert np.array_equal(ds.pencil.b.toarray(), ref["b"])
    assert np.array_equal(ds.truth_eigenvalues, ref["truth"])
    assert ds.truth_m == len(ref["truth"])
    assert np.array_equal(ds.field["values"], ref["field"])
    assert ds.pencil.problem_id == str(ref["problem_id"])
    assert ds.pencil.hermitian and ds.grid == (8, 8)


@pytest.mark.parametrize("name", ["empty", "header", "field", "symmetry", "nosize", "size", "entry", "range",
                                  "more", "fewer", "complexbad"])
def test_malformed_files_raise_like_the_reference(tmp_path, name):
    ref = golden("ref_dataset.npz")
    fp = tmp_path / "m.mtx"
    fp.write_text(str(ref[f"bad_{name}_text"]))
    with pytest.raises(FormatError) as ei:
        read_matrix_market(str(fp))
    assert str(ei.value) == str(ref[f"bad_{name}_msg"])


@pytest.mark.parametrize("name", ["sym", "herm", "skew", "int"])
def test_symmetric_storage_is_expanded(tmp_path, name):
    ref = golden("ref_dataset.npz")
    fp = tmp_path / "m.mtx"
    fp.write_text(str(ref[f"sym_{name}_text"]))
    assert np.array_equal(read_matrix_market(str(fp)).toarray(), ref[f"sym_{name}_dense"])


def test_round_trip(tmp_path):
    ds = read_dataset(FIX)
    out = tmp_path / "copy"
    write_dataset(str(out), ds.pencil.a, ds.pencil.b, ds.pencil.problem_id, ds.grid, ds.field, ds.truth_eigenvalues)
    back = read_dataset(str(out))
    assert np.array_equal(back.pencil.a.toarray(), ds.pencil.a.toarray())
    assert np.array_equal(back.pencil.b.toarray(), ds.pencil.b.toarray())
    assert np.array_equal(back.truth_eigenvalues, ds.truth_eigenvalues)


def test_missing_files(tmp_path):
    with pytest.raises(FormatError, match="missing dataset file A.mtx"):
        read_dataset(str(tmp_path))
    (tmp_path / "A.mtx").write_text((open(os.path.join(FIX, "A.mtx")).read()))
    (tmp_path / "B.mtx").write_text((open(os.path.join(FIX, "B.mtx")).read()))
    (tmp_path / "meta.json").write_text("{bad json")
    with pytest.raises(FormatError, match="bad meta.json"):
        read_dataset(str(tmp_path))


@pytest.mark.gpu
def test_solve_reference_dataset_on_gpu():
    from paper_2511_01927_b200 import Contour, SolverConfig, cirr_solve

    ds = read_dataset(FIX)
    t = ds.truth_eigenvalues
    c = Contour(shape="circle", center=complex(0.5 * (t[0] + t[3]), 0.0), radius=0.5 * (t[3] - t[0]) + 0.4 *
                min(t[1] - t[0], t[4] - t[3]), expected_count=4)
    r = cirr_solve(ds.pencil, c, SolverConfig(n_q=32, source_cols=16, n_moments=4))
    assert len(r.eigenvalues) == 4
    assert np.abs(np.sort(r.eigenvalues.real) - t[:4]).max() <= 1e-8 * t[3]
    assert r.residuals.max() <= 1e-10
