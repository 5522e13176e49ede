"""Phase split (Householder QR / Jacobi SVD / back-application) of one
cirr_orth call on graded moment-like blocks: n x c, nprob problems."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_01927_b200 import _lib  # noqa: E402


def main(n=4096, c=256, nprob=2):
    lib = _lib.load()
    lib.cirr_orth_phases.argtypes = [ctypes.c_void_p]
    rng = np.random.default_rng(0)
    Ws = []
    for p in range(nprob):
        U, _ = np.linalg.qr(rng.standard_normal((n, c)) + 1j * rng.standard_normal((n, c)))
        V, _ = np.linalg.qr(rng.standard_normal((c, c)) + 1j * rng.standard_normal((c, c)))
        s = np.logspace(0, -11.7, c)
        Ws.append(((U * s) @ V.conj().T).T)
    W0 = torch.from_numpy(np.ascontiguousarray(np.stack(Ws))).cuda()
    st = torch.cuda.current_stream().cuda_stream
    sig = torch.empty((nprob, c), dtype=torch.float64, device="cuda")
    order = torch.empty((nprob, c), dtype=torch.int32, device="cuda")
    kept = torch.empty(nprob, dtype=torch.int32, device="cuda")
    Qt = torch.empty((nprob, c, n), dtype=torch.complex128, device="cuda")
    ws = torch.empty(_lib.call("cirr_orth_ws_bytes", c, nprob), dtype=torch.uint8, device="cuda")
    sw = torch.zeros(1, dtype=torch.int32, device="cuda")
    for rep in range(3):
        W = W0.clone()
        torch.cuda.synchronize()
        t = time.perf_counter()
        _lib.call("cirr_orth", W.data_ptr(), n, c * n, n, c, nprob, 1e-12, sig.data_ptr(), order.data_ptr(),
                  kept.data_ptr(), Qt.data_ptr(), n, c * n, ws.data_ptr(), sw.data_ptr(), st)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t) * 1e3
        ph = (ctypes.c_longlong * 4)()
        lib.cirr_orth_phases(ph)
        clk = 1.965e6  # cycles per ms at 1965 MHz
        print(f"n={n} c={c} nprob={nprob}: {ms:.2f} ms  QR {(ph[1]-ph[0])/clk:.2f}  Jacobi {(ph[2]-ph[1])/clk:.2f}  "
              f"back {(ph[3]-ph[2])/clk:.2f} ms  sweeps {sw.item()} kept {kept.cpu().tolist()}", flush=True)


if __name__ == "__main__":
    main(*[int(x) for x in sys.argv[1:]])
