import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_01927_b200 import _lib


def run(a, b, herm):
    nprob, k, _ = a.shape
    A = torch.from_numpy(np.ascontiguousarray(a)).cuda(); B = torch.from_numpy(np.ascontiguousarray(b)).cuda()
    kd = torch.full((nprob,), k, dtype=torch.int32, device="cuda")
    wsb = (_lib.call("cirr_small_eig_ws_bytes", k) + 255) // 256 * 256
    ws = torch.empty(nprob * wsb, dtype=torch.uint8, device="cuda")
    lam = torch.empty((nprob, k), dtype=torch.complex128, device="cuda")
    S = torch.empty((nprob, k, k), dtype=torch.complex128, device="cuda")
    info = torch.empty(nprob, dtype=torch.int32, device="cuda")
    _lib.call("cirr_small_eig", herm, A.data_ptr(), B.data_ptr(), k, k * k, kd.data_ptr(), k, nprob,
              ws.data_ptr(), lam.data_ptr(), S.data_ptr(), k, k * k, info.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    out = []
    for p in range(nprob):
        s = S.cpu().numpy()[p]; l = lam.cpu().numpy()[p]
        r = a[p] @ s - (b[p] @ s) * l[None, :]
        rel = np.linalg.norm(r, axis=0) / (np.linalg.norm(a[p] @ s, axis=0) + np.abs(l) * np.linalg.norm(b[p] @ s, axis=0))
        import scipy.linalg as sla
        w = sla.eigh(a[p], b[p], eigvals_only=True) if herm else None
        out.append((rel.max(), None if w is None else np.abs(np.sort(l.real) - w).max()))
    return out


rng = np.random.default_rng(1)
for k in (6, 64, 120):
    for nprob in (1, 2):
        x = rng.standard_normal((nprob, k, k)) + 1j * rng.standard_normal((nprob, k, k))
        a = x + np.conj(np.transpose(x, (0, 2, 1)))
        y = rng.standard_normal((nprob, k, k)) + 1j * rng.standard_normal((nprob, k, k))
        b1 = np.einsum("bij,bkj->bik", y, np.conj(y)) + k * np.eye(k)
        yy = np.eye(k) + 0.05 * y
        b2 = np.einsum("bij,bkj->bik", yy, np.conj(yy))
        print(k, nprob, "b1", run(a, b1, 1), "b2", run(a, b2, 1), flush=True)
