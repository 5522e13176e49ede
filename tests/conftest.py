import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")  # SURVEY 0 finding 5: threaded OpenBLAS is pathological here

import numpy as np  # noqa: E402
import pytest  # noqa: E402

try:  # numpy may already be loaded by a plugin: clamp the BLAS pool at runtime too
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)
except Exception:  # pragma: no cover
    pass

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libcirr.so")
    config.addinivalue_line("markers", "slow: full-size BASELINE configs (minutes)")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def csr_dense(g, prefix):
    import scipy.sparse as sp
    n = int(g[prefix.split("_")[0] + "_n"])
    m = sp.csr_matrix((g[prefix + "_data"], g[prefix + "_indices"], g[prefix + "_indptr"]), shape=(n, n))
    return m.toarray()


class DensePencil:
    """Minimal pencil object (duck-typed like cieig.MatrixPencil)."""

    def __init__(self, a, b, hermitian=True):
        self.a = np.asarray(a)
        self.b = np.asarray(b)
        self.hermitian = hermitian

    @property
    def n(self):
        return self.a.shape[0]


def diag_pencil(da, db=None):
    a = np.diag(np.asarray(da, dtype=float))
    b = np.eye(len(da)) if db is None else np.diag(np.asarray(db, dtype=float))
    return DensePencil(a, b, True)


@pytest.fixture(scope="session")
def thermal():
    g = golden("ref_thermal.npz")
    return {
        "t10": DensePencil(csr_dense(g, "t10_a").real, csr_dense(g, "t10_b").real),
        "t20": DensePencil(csr_dense(g, "t20_a").real, csr_dense(g, "t20_b").real),
        "g": g,
    }


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_cieig():
    """The unmodified reference package staged under baseline/_ref by
    __graft_entry__.build() (copied from /root/reference/pkg/src/cieig when
    that exists; the copy travels to the GPU box). Skips when absent."""
    if not os.path.isfile(os.path.join(REF_DIR, "cieig", "solvers.py")):
        try:
            import __graft_entry__
            __graft_entry__.stage_reference()
        except Exception:  # pragma: no cover
            pass
    if not os.path.isfile(os.path.join(REF_DIR, "cieig", "solvers.py")):
        pytest.skip("reference package not staged under baseline/_ref (run __graft_entry__.build())")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import cieig
    import cieig.bench  # noqa: F401
    import cieig.cli  # noqa: F401
    import cieig.contours  # noqa: F401
    import cieig.problems  # noqa: F401
    import cieig.solvers  # noqa: F401
    return cieig
