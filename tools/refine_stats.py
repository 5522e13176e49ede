"""Dev tool: per-column quality of the refinement-round eigenbasis W0 = Q^H S
on config 4 (how many columns of T = W0^-1 M W0 are already near e_j)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2511_01927_b200 import solvers as S  # noqa: E402
from paper_2511_01927_b200 import _lib  # noqa: E402



def main():
    import torch
    eng_cls = None
    for v in vars(S).values():
        if isinstance(v, type) and hasattr(v, "_refine_eig_g"):
            eng_cls = v
    base = eng_cls._refine_eig_g

    def hook(self, S_st, Q, At, Bt, kdim, kmax, nb, lam, Sv, info):
        n = self.n
        kk = kmax * kmax
        W0h = torch.empty((nb, kmax, kmax), dtype=torch.complex128, device="cuda")
        _lib.call("cirr_gemm", 1, kmax, kmax, n, nb, S._ptr(S_st), n, kmax * n, S._ptr(Q), kmax, n * kmax,
                  S._ptr(W0h), kmax, kk, 1.0, 0, self.stream)
        ks = kdim.cpu().numpy()
        for b in range(nb):
            k = int(ks[b])
            W = W0h[b, :k, :k].conj().T
            W = W / torch.linalg.norm(W, dim=0, keepdim=True)
            M = torch.linalg.solve(Bt[b, :k, :k], At[b, :k, :k])
            T = torch.linalg.solve(W, M @ W)
            d = torch.diagonal(T)
            off = (T - torch.diag(d)).abs()
            c = off.max(dim=0).values.cpu().numpy()
            scale = float(d.abs().max())
            h = [int((c <= t * scale).sum()) for t in (1e-1, 1e-2, 1e-3, 1e-5, 1e-8, 1e-11)]
            print(f"[stats] k={k} scale={scale:.3f} cols with max|T_ij|/scale <= 1e-1,-2,-3,-5,-8,-11: {h}"
                  f" cond(W)={float(torch.linalg.cond(W)):.2e}", flush=True)
        return (yield from base(self, S_st, Q, At, Bt, kdim, kmax, nb, lam, Sv, info))

    eng_cls._refine_eig_g = hook
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from run_config import main as run
    run(4, reps=1)


if __name__ == "__main__":
    main()
