"""Golden vectors for the device KDE contour construction (SURVEY.md 8(f)
row 4) from the UNMODIFIED reference `cieig.contours.construct_contours`
(contours.py:230-320) and `kde_eval` (kernels.py:58-67, numba build).

Run in the build container only (imports /root/reference/pkg/src):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_kde_golden.py

Output: ref_kde.npz -- for case c: c_values (sorted predictions), c_nmin,
c_nmax, c_w, c_iv (intervals: start, end, count); kde_ts/kde_eigs/kde_coef/
kde_out for a direct kde_eval check.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from cieig.contours import SpectrumPrediction, construct_contours  # noqa: E402
from cieig.kernels import kde_eval  # noqa: E402


def main():
    out = {}
    cases = []
    for seed, m, nmin, nmax, w in ((0, 120, 10, 50, 10.0), (1, 500, 10, 50, 10.0), (2, 2000, 20, 80, 10.0),
                                   (3, 300, 5, 30, 25.0), (4, 64, 1, 12, 10.0)):
        rng = np.random.default_rng(seed)
        # clustered spectra: a few dense groups plus a uniform background
        vals = np.concatenate([rng.normal(c, 0.3, m // 4) for c in rng.uniform(-10, 10, 3)]
                              + [rng.uniform(-12, 12, m - 3 * (m // 4))])
        vals = np.sort(vals)
        part, _ = construct_contours(SpectrumPrediction(values=vals), n_min=nmin, n_max=nmax, w=w)
        name = f"case{seed}"
        cases.append(name)
        out[f"{name}_values"] = vals
        out[f"{name}_params"] = np.array([nmin, nmax, w])
        out[f"{name}_iv"] = np.array([[iv.start, iv.end, iv.count] for iv in part.intervals])
        print(name, len(part.intervals), "intervals", flush=True)
    out["cases"] = np.array(cases)
    rng = np.random.default_rng(9)
    ts = np.linspace(-5.0, 5.0, 3001)
    eigs = np.sort(rng.uniform(-6.0, 6.0, 2500))
    out["kde_ts"], out["kde_eigs"], out["kde_coef"] = ts, eigs, np.array(3.7)
    out["kde_out"] = kde_eval(ts, eigs, 3.7)
    np.savez_compressed(os.path.join(HERE, "ref_kde.npz"), **out)


if __name__ == "__main__":
    main()
