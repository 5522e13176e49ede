"""Drop the GPU CIRR path into an unmodified reference pipeline (cieig).

    import cieig
    from paper_2511_01927_b200 import patch
    patch.install(cieig)          # bench / cli / solvers now solve on the B200
    ...
    patch.uninstall(cieig)

Patch points:
  * ``cieig.solvers.cirr_solve`` -- looked up at call time by the reference's
    own ``solve_multi`` (solvers.py:319), so per-contour callers are rerouted;
  * ``cieig.solvers.solve_multi``, ``cieig.bench.solve_multi`` (bench.py:23,
    used at 144) and ``cieig.cli.solve_multi`` (cli.py:41, used at 194) -- the
    name-imported copies, replaced so a call batches every contour through one
    device pass;
  * ``cieig.contours.kde_eval`` (imported by name at contours.py:20, looked up
    at call time at :191) -- the density of the reference's own KDE contour
    construction, evaluated on the device (kde.py).

Results come back as the reference's own ``EigenResult`` / ``SolveStats`` /
``MultiResult`` objects and errors as the reference's own exception classes,
so reference code that catches ``cieig.errors.*`` keeps working.  FEAST
(``solver="feast"``) runs on the same device path.
"""

from __future__ import annotations

from . import errors as E
from . import kde as K
from . import solvers as S

_ORIG: dict = {}

_ERR_NAMES = ("SingularShiftError", "RankZeroError", "IndefiniteBError", "NoEigenvaluesFound",
              "ConvergenceError", "DimensionError", "ParameterError")


def _to_ref_error(cieig, exc):
    """Map one of our exceptions onto the reference class of the same name."""
    rerr = cieig.errors
    name = type(exc).__name__
    if name == "SingularShiftError":
        return rerr.SingularShiftError(exc.shift, node_index=exc.node_index)
    if name == "ConvergenceError":
        return rerr.ConvergenceError(exc.best_residual)
    if name in _ERR_NAMES:
        return getattr(rerr, name)(str(exc))
    return exc


def _to_ref_result(cieig, r):
    rs = cieig.solvers
    stats = rs.SolveStats(n_linear_solves=r.stats.n_linear_solves, n_factorizations=r.stats.n_factorizations,
                          iterations=r.stats.iterations, elapsed=r.stats.elapsed)
    return rs.EigenResult(eigenvalues=r.eigenvalues, eigenvectors=r.eigenvectors, residuals=r.residuals,
                          contour=r.contour, stats=stats)


def gpu_cirr_solve_for(cieig):
    def cirr_solve(pencil, contour, cfg=None, seed: int = 0):
        try:
            return _to_ref_result(cieig, S.cirr_solve(pencil, contour, cfg, seed=seed))
        except E.CieigError as exc:
            raise _to_ref_error(cieig, exc) from exc

    cirr_solve.__doc__ = "B200 CIRR (paper_2511_01927_b200) behind the reference signature (solvers.py:165)."
    return cirr_solve


def gpu_feast_solve_for(cieig):
    def feast_solve(pencil, contour, cfg=None, seed: int = 0):
        try:
            return _to_ref_result(cieig, S.feast_solve(pencil, contour, cfg, seed=seed))
        except E.CieigError as exc:
            raise _to_ref_error(cieig, exc) from exc

    feast_solve.__doc__ = "B200 FEAST behind the reference signature (solvers.py:230)."
    return feast_solve


def gpu_solve_multi_for(cieig):
    def solve_multi(pencil, contours, cfg=None, solver: str = "cirr", seed: int = 0):
        try:
            m = S.solve_multi(pencil, contours, cfg, solver=solver, seed=seed)
        except E.CieigError as exc:
            raise _to_ref_error(cieig, exc) from exc
        rs = cieig.solvers
        results = [None if r is None else _to_ref_result(cieig, r) for r in m.results]
        errs = [None if e is None else _to_ref_error(cieig, e) for e in m.errors]
        agg = rs.SolveStats(n_linear_solves=m.stats.n_linear_solves, n_factorizations=m.stats.n_factorizations,
                            iterations=m.stats.iterations, elapsed=m.stats.elapsed)
        return rs.MultiResult(results=results, errors=errs, stats=agg)

    solve_multi.__doc__ = "B200 batched solve_multi behind the reference signature (solvers.py:312)."
    return solve_multi


def install(cieig) -> None:
    """Reroute the reference's CIRR entry points to the GPU path."""
    import cieig.bench  # noqa: F401
    import cieig.cli  # noqa: F401
    import cieig.solvers  # noqa: F401

    if _ORIG:
        return
    _ORIG["solvers.cirr_solve"] = cieig.solvers.cirr_solve
    _ORIG["solvers.feast_solve"] = cieig.solvers.feast_solve
    _ORIG["solvers.solve_multi"] = cieig.solvers.solve_multi
    _ORIG["bench.solve_multi"] = cieig.bench.solve_multi
    _ORIG["cli.solve_multi"] = cieig.cli.solve_multi
    sm = gpu_solve_multi_for(cieig)
    cieig.solvers.cirr_solve = gpu_cirr_solve_for(cieig)
    cieig.solvers.feast_solve = gpu_feast_solve_for(cieig)
    cieig.solvers.solve_multi = sm
    cieig.bench.solve_multi = sm
    cieig.cli.solve_multi = sm
    K.install(cieig)


def uninstall(cieig) -> None:
    if not _ORIG:
        return
    cieig.solvers.cirr_solve = _ORIG.pop("solvers.cirr_solve")
    cieig.solvers.feast_solve = _ORIG.pop("solvers.feast_solve")
    cieig.solvers.solve_multi = _ORIG.pop("solvers.solve_multi")
    cieig.bench.solve_multi = _ORIG.pop("bench.solve_multi")
    cieig.cli.solve_multi = _ORIG.pop("cli.solve_multi")
    K.uninstall(cieig)
