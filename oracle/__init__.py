"""CPU oracle for the CIRR contour-integral stage -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import anything from this package, and only as
the checker or the timed CPU baseline.  The product path
(``paper_2511_01927_b200``) never imports it and has no CPU fallback.

Parity is pinned: ``tests/test_oracle_pin.py`` checks the restatement (in its
``reference`` mode) against golden vectors produced by the unmodified
reference package (``tests/golden/make_golden.py`` imports
``/root/reference/pkg/src/cieig`` in the build container) and against the
reference's own known-answer tests (``pkg/tests/test_solvers.py:30-142``,
``test_linalg.py:29-170``, ``test_contours.py:146-199``).
"""

from .cirr import (  # noqa: F401
    OracleConfig,
    apply_projector,
    cirr_solve,
    contains,
    feast_solve,
    orthonormalize,
    quadrature,
    rank_truncate_svd,
    residuals,
    solve_multi,
)
