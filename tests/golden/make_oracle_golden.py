"""Full-size BASELINE-config fixtures from the restated CPU oracle + dense truth.

Run in the build container (minutes to ~30 min for config 4's QZ truth):

    OPENBLAS_NUM_THREADS=8 python tests/golden/make_oracle_golden.py [1 2 3 4 5]

For each config it stores the contours (JSON), the oracle's per-contour
eigenvalues / residuals / iterations / ranks, and the dense-truth eigenvalues
strictly inside each contour (scipy.linalg.eigh for the Hermitian configs,
scipy.linalg.eig for config 4) with the minimum distance of any eigenvalue to
each boundary.  The GPU parity tests compare against these without needing
the oracle's minutes of CPU time on the GPU box.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np
import scipy.linalg as sla

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import oracle  # noqa: E402
from oracle.cirr import OracleConfig, Pencil  # noqa: E402
from paper_2511_01927_b200 import workloads as W  # noqa: E402
from paper_2511_01927_b200.contours import contains  # noqa: E402


def boundary_q(c, lam):
    if c.shape == "circle":
        return np.abs(lam - c.center) / c.radius
    return np.sqrt(((lam.real - c.center.real) / c.semi_re) ** 2 + ((lam.imag - c.center.imag) / c.semi_im) ** 2)


def solve(wl, truth, tag, out, threads_note="", lu="dense"):
    p = Pencil(wl.a, wl.b, wl.hermitian)
    cfg = OracleConfig(n_q=wl.n_q, source_cols=wl.source_cols, n_moments=wl.n_moments, lu=lu)
    t = time.perf_counter()
    m = oracle.solve_multi(p, wl.contours, cfg, seed=0)
    el = time.perf_counter() - t
    out[f"{tag}contours"] = np.array(json.dumps([c.to_json_dict() for c in wl.contours]))
    out[f"{tag}oracle_seconds"] = np.array(el)
    for i, (c, r, e) in enumerate(zip(wl.contours, m.results, m.errors)):
        inside = np.array([v for v in truth if contains(c, v)])
        q = boundary_q(c, truth)
        out[f"{tag}c{i}_truth"] = np.sort(inside) if inside.size else inside
        out[f"{tag}c{i}_min_boundary_dist"] = np.array(np.abs(q - 1.0).min())
        out[f"{tag}c{i}_err"] = np.array("" if e is None else type(e).__name__)
        if r is not None:
            out[f"{tag}c{i}_eigs"] = r.eigenvalues
            out[f"{tag}c{i}_res"] = r.residuals
            out[f"{tag}c{i}_iters"] = np.array(r.iterations)
            out[f"{tag}c{i}_ranks"] = np.array(r.ranks)
            print(f"{tag}c{i}: {len(r.eigenvalues)} found / {inside.size} truth, iters {r.iterations}, "
                  f"ranks {r.ranks}, max res {r.residuals.max():.2e}, min |q-1| {np.abs(q - 1).min():.2e}",
                  flush=True)
        else:
            print(f"{tag}c{i}: error {e!r} / {inside.size} truth", flush=True)
    print(f"{tag} oracle {el:.1f}s {threads_note}", flush=True)


def config1():
    wl = W.config1()
    truth = W.sorted_real_eigs(wl.a, wl.b)
    out = {}
    solve(wl, truth, "", out)
    np.savez_compressed(os.path.join(HERE, "oracle_config1.npz"), **out)


def config2(n_gep=256):
    out = {"n_gep": np.array(n_gep)}
    for s in range(n_gep):
        a, b = W.config2_matrices(s)
        truth = np.sort(sla.eigh(a, b, eigvals_only=True))
        wl = W.config2_gep(s, eigs=truth)
        solve(wl, truth, f"s{s}_", out)
    np.savez_compressed(os.path.join(HERE, "oracle_config2.npz"), **out)


def config3():
    a, b = W.config3_matrices()
    truth = np.sort(sla.eigh(a, b, eigvals_only=True))
    wl = W.config3(eigs=truth)
    out = {}
    solve(wl, truth, "", out)
    np.savez_compressed(os.path.join(HERE, "oracle_config3.npz"), **out)


def config4():
    wl = W.config4()
    t = time.perf_counter()
    cache = os.path.join("/tmp", "config4_truth.npy")
    if os.path.exists(cache):
        truth = np.load(cache)
    else:
        truth = sla.eig(wl.a, wl.b, right=False)
        np.save(cache, truth)
    print(f"config4 truth {time.perf_counter() - t:.1f}s", flush=True)
    out = {}
    solve(wl, truth, "", out)
    np.savez_compressed(os.path.join(HERE, "oracle_config4.npz"), **out)


def config5():
    a, b = W.config5_matrices()
    truth = np.sort(sla.eigh(a, b, eigvals_only=True, subset_by_index=[150, 500]))
    full_idx = np.arange(150, 501)
    # contour placement needs l_1..l_460 indices; build a padded array with the subset in place
    eigs = np.full(501, np.nan)
    eigs[full_idx] = truth
    wl = W.config5(eigs=eigs)
    out = {}
    # 7-point stencils: SuperLU (the reference's own factorisation) is far
    # faster than a dense LU here; the moments are still the centred ones
    solve(wl, truth, "", out, lu="superlu")
    np.savez_compressed(os.path.join(HERE, "oracle_config5.npz"), **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["1", "2", "3", "4", "5"]
    for w in which:
        globals()[f"config{w}"]()
