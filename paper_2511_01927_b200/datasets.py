"""Pencil ingestion from the reference's on-disk dataset format, and back.

SURVEY.md 8(f) row 2: a dataset directory holds ``A.mtx``, ``B.mtx`` (Matrix
Market coordinate files) and ``meta.json`` (problem id, grid, coefficient
field, optional ground truth) -- the layout of ``problems.py:292-353``
(write_dataset / read_dataset) with the Matrix Market reader/writer of
``sparse.py:137-228``.  Reading one gives a pencil object that
``solve_multi``/``cirr_solve`` upload to HBM directly (dense, as the GPU path
stores every pencil), so ``cieig solve``/``bench`` datasets drive the GPU path
without the reference installed.

Error behaviour follows the reference: every malformed input raises
``FormatError`` with the offending 1-based line number where one exists.
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from .errors import FormatError

_FIELDS = ("real", "complex", "integer")
_SYMMETRIES = ("general", "symmetric", "hermitian", "skew-symmetric")


def read_matrix_market(path) -> sp.csr_matrix:
    """Coordinate-format Matrix Market file -> complex CSR (sparse.py:155-228).

    Fields real/complex/integer; symmetry general/symmetric/hermitian/
    skew-symmetric (the stored triangle is mirrored, conjugated or negated).
    """
    with open(path) as fh:
        lines = fh.read().splitlines()
    if not lines:
        raise FormatError("empty file", line=1)
    head = lines[0].split()
    if len(head) != 5 or head[0] != "%%MatrixMarket" or head[1].lower() != "matrix" \
            or head[2].lower() != "coordinate":
        raise FormatError("bad Matrix Market header", line=1)
    fld, sym = head[3].lower(), head[4].lower()
    if fld not in _FIELDS:
        raise FormatError(f"unsupported field {fld!r}", line=1)
    if sym not in _SYMMETRIES:
        raise FormatError(f"unsupported symmetry {sym!r}", line=1)
    ln = 1
    while ln < len(lines) and (lines[ln].startswith("%") or not lines[ln].strip()):
        ln += 1
    if ln >= len(lines):
        raise FormatError("missing size line", line=len(lines))
    try:
        n_rows, n_cols, nnz = (int(t) for t in lines[ln].split())
    except ValueError:
        raise FormatError("bad size line", line=ln + 1) from None
    ii = np.empty(nnz, dtype=np.int64)
    jj = np.empty(nnz, dtype=np.int64)
    vv = np.empty(nnz, dtype=np.complex128)
    cnt = 0
    for pos in range(ln + 1, len(lines)):
        raw = lines[pos].strip()
        if not raw or raw.startswith("%"):
            continue
        if cnt >= nnz:
            raise FormatError("more entries than declared", line=pos + 1)
        tok = raw.split()
        try:
            i, j = int(tok[0]) - 1, int(tok[1]) - 1
            v = complex(float(tok[2]), float(tok[3])) if fld == "complex" else complex(float(tok[2]), 0.0)
        except (ValueError, IndexError):
            raise FormatError("bad entry line", line=pos + 1) from None
        if not (0 <= i < n_rows and 0 <= j < n_cols):
            raise FormatError("index out of range", line=pos + 1)
        ii[cnt], jj[cnt], vv[cnt] = i, j, v
        cnt += 1
    if cnt != nnz:
        raise FormatError(f"expected {nnz} entries, found {cnt}", line=len(lines))
    if sym != "general":
        off = ii != jj
        mv = vv[off]
        if sym == "hermitian":
            mv = np.conj(mv)
        elif sym == "skew-symmetric":
            mv = -mv
        ii, jj, vv = np.concatenate([ii, jj[off]]), np.concatenate([jj, ii[off]]), np.concatenate([vv, mv])
    return sp.coo_matrix((vv, (ii, jj)), shape=(n_rows, n_cols)).tocsr()


def write_matrix_market(path, m, field: str = "complex") -> None:
    """1-based coordinate file, general symmetry, 17 significant digits
    (sparse.py:137-152)."""
    if field not in ("real", "complex"):
        raise FormatError(f"unsupported field {field!r}")
    coo = (m if sp.issparse(m) else sp.coo_matrix(np.asarray(m))).tocoo()
    with open(path, "w") as fh:
        fh.write(f"%%MatrixMarket matrix coordinate {field} general\n")
        fh.write(f"{coo.shape[0]} {coo.shape[1]} {coo.nnz}\n")
        for i, j, v in zip(coo.row, coo.col, coo.data):
            v = complex(v)
            if field == "real":
                fh.write(f"{i + 1} {j + 1} {v.real:.17g}\n")
            else:
                fh.write(f"{i + 1} {j + 1} {v.real:.17g} {v.imag:.17g}\n")


@dataclass
class DatasetPencil:
    """A, B as read from disk (complex CSR); ``solve_multi`` accepts it like the
    reference's ``MatrixPencil`` (problems.py:348-350 marks these Hermitian
    with positive-definite B)."""

    a: sp.csr_matrix
    b: sp.csr_matrix
    hermitian: bool = True
    b_positive_definite: bool = True
    problem_id: str = ""

    @property
    def n(self) -> int:
        return self.a.shape[0]


@dataclass
class Dataset:
    pencil: DatasetPencil
    grid: tuple = (0, 0)
    field: dict = field(default_factory=dict)
    truth_eigenvalues: np.ndarray | None = None
    truth_m: int | None = None


def read_dataset(path) -> Dataset:
    """A.mtx + B.mtx + meta.json (problems.py:318-353)."""
    files = {name: os.path.join(path, name) for name in ("A.mtx", "B.mtx", "meta.json")}
    for name, fp in files.items():
        if not os.path.exists(fp):
            raise FormatError(f"missing dataset file {name}")
    a = read_matrix_market(files["A.mtx"])
    b = read_matrix_market(files["B.mtx"])
    try:
        with open(files["meta.json"]) as fh:
            meta = json.load(fh)
    except json.JSONDecodeError as exc:
        raise FormatError(f"bad meta.json: {exc.msg}", line=exc.lineno) from exc
    try:
        grid = (int(meta["grid"]["nx"]), int(meta["grid"]["ny"]))
        fm = meta["field"]
        fld = {"values": np.asarray(fm["values"], dtype=float), "mean": float(fm["mean"]),
               "variance": float(fm["variance"]), "length_scale": float(fm["length_scale"]),
               "seed": int(fm["seed"])}
        pid = str(meta["problem_id"])
    except (KeyError, TypeError) as exc:
        raise FormatError(f"meta.json missing key: {exc}") from exc
    truth = meta.get("truth")
    return Dataset(pencil=DatasetPencil(a=a, b=b, problem_id=pid), grid=grid, field=fld,
                   truth_eigenvalues=None if truth is None else np.asarray(truth["eigenvalues"], dtype=float),
                   truth_m=None if truth is None else int(truth["m"]))


def write_dataset(path, a, b, problem_id: str, grid=(0, 0), field_meta: dict | None = None,
                  truth_eigenvalues=None) -> None:
    """Inverse of read_dataset (problems.py:292-315)."""
    os.makedirs(path, exist_ok=True)
    write_matrix_market(os.path.join(path, "A.mtx"), a)
    write_matrix_market(os.path.join(path, "B.mtx"), b)
    fm = dict(field_meta or {})
    meta = {
        "problem_id": problem_id,
        "grid": {"nx": int(grid[0]), "ny": int(grid[1])},
        "field": {"mean": fm.get("mean", 0.0), "variance": fm.get("variance", 0.0),
                  "length_scale": fm.get("length_scale", 0.0), "seed": fm.get("seed", 0),
                  "values": np.asarray(fm.get("values", []), dtype=float).tolist()},
        "truth": None if truth_eigenvalues is None else {
            "m": len(truth_eigenvalues), "eigenvalues": np.asarray(truth_eigenvalues, dtype=float).tolist()},
    }
    with open(os.path.join(path, "meta.json"), "w") as fh:
        json.dump(meta, fh)
