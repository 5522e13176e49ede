"""max |P A - L U| / (n max|A|) of one dense n = 2048 complex pencil: int8 trailing updates vs all-FP64 (DMMA)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2511_01927_b200 import _lib as lib

n = 2048
rng = np.random.default_rng(2048)
A = rng.standard_normal((1, n, n)) + 1j * rng.standard_normal((1, n, n))
st = torch.cuda.current_stream().cuda_stream


def backward_error(mode):
    lib.call("cirr_set_lu_gemm", mode)
    F = torch.from_numpy(A.copy()).cuda()
    ipiv = torch.empty((1, n), dtype=torch.int32, device="cuda")
    perm = torch.empty((1, n), dtype=torch.int32, device="cuda")
    mp = torch.empty(1, dtype=torch.float64, device="cuda")
    info = torch.empty(1, dtype=torch.int32, device="cuda")
    ws = torch.zeros(lib.call("cirr_zgetrf_ws_bytes", n, 1), dtype=torch.uint8, device="cuda")
    lib.call("cirr_zgetrf_batched", F.data_ptr(), n, n, n * n, 1, ipiv.data_ptr(), perm.data_ptr(), mp.data_ptr(),
             info.data_ptr(), ws.data_ptr(), st)
    torch.cuda.synchronize()
    lu = F[0].cpu().numpy()
    L, U, pa = np.tril(lu, -1) + np.eye(n), np.triu(lu), A[0].copy()
    for i, pi in enumerate(ipiv[0].cpu().numpy()):
        if pi != i:
            pa[[i, pi]] = pa[[pi, i]]
    return np.abs(pa - L @ U).max() / (n * np.abs(A[0]).max())


print("int8 %.3e   fp64 (DMMA) %.3e   (u = %.3e)" % (backward_error(1), backward_error(0), 2.0 ** -53))
