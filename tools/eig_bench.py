"""Time the small projected eigensolvers (K6) and the Jacobi SVD (K4)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_01927_b200 import _lib  # noqa: E402


def t_small(k, herm, nprob=2, reps=3):
    rng = np.random.default_rng(k)
    a = rng.standard_normal((nprob, k, k)) + 1j * rng.standard_normal((nprob, k, k))
    b = np.eye(k) + 0.05 * (rng.standard_normal((nprob, k, k)) + 1j * rng.standard_normal((nprob, k, k)))
    if herm:
        a = a + np.conj(np.transpose(a, (0, 2, 1)))
        b = np.einsum("bij,bkj->bik", b, np.conj(b))
    A = torch.from_numpy(a).cuda(); B = torch.from_numpy(b).cuda()
    kd = torch.full((nprob,), k, dtype=torch.int32, device="cuda")
    wsb = (_lib.call("cirr_small_eig_ws_bytes", k) + 255) // 256 * 256
    ws = torch.empty(nprob * wsb, dtype=torch.uint8, device="cuda")
    lam = torch.empty((nprob, k), dtype=torch.complex128, device="cuda")
    S = torch.empty((nprob, k, k), dtype=torch.complex128, device="cuda")
    info = torch.empty(nprob, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        _lib.call("cirr_small_eig", 1 if herm else 0, A.data_ptr(), B.data_ptr(), k, k * k, kd.data_ptr(), k, nprob,
                  ws.data_ptr(), lam.data_ptr(), S.data_ptr(), k, k * k, info.data_ptr(), st)
        e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    s = S.cpu().numpy()[0]; l = lam.cpu().numpy()[0]
    r = a[0] @ s - (b[0] @ s) * l[None, :]
    rel = np.linalg.norm(r, axis=0) / (np.linalg.norm(a[0] @ s, axis=0) + np.abs(l) * np.linalg.norm(b[0] @ s, axis=0))
    import ctypes
    ph = (ctypes.c_longlong * 16)()
    _lib.call("cirr_small_eig_phases", ctypes.addressof(ph))
    if not herm:
        d = [ph[i + 1] - ph[i] for i in range(6)]
        print("  phases (Mcycles): LU %.2f solve %.2f hess %.2f qr %.2f vec %.2f sort+Zx %.2f" % tuple(x / 1e6 for x in d),
              "sweeps", ph[8], "rotations", ph[9], "cycles/rot %.0f" % (d[3] / max(ph[9], 1)), "win/chain/def Mcyc %.1f %.1f %.1f" % (ph[10]/1e6, ph[11]/1e6, ph[12]/1e6))
    print(f"small_eig herm={herm} k={k} nprob={nprob}: {min(ts):.2f} ms, info={info.cpu().numpy()}, max rel res {rel.max():.1e}", flush=True)


def t_orth(n, c, nprob=2, reps=2):
    rng = np.random.default_rng(c)
    u = np.linalg.qr(rng.standard_normal((n, c)) + 1j * rng.standard_normal((n, c)))[0]
    s = np.logspace(0, -11.5, c)
    m = (u * s) @ np.linalg.qr(rng.standard_normal((c, c)) + 0j)[0]
    W0 = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(m.T, (nprob, c, n)))).cuda()
    st = torch.cuda.current_stream().cuda_stream
    sig = torch.empty((nprob, c), dtype=torch.float64, device="cuda"); order = torch.empty((nprob, c), dtype=torch.int32, device="cuda")
    kept = torch.empty(nprob, dtype=torch.int32, device="cuda"); Qt = torch.empty((nprob, c, n), dtype=torch.complex128, device="cuda")
    ws = torch.empty(_lib.call("cirr_orth_ws_bytes", c, nprob), dtype=torch.uint8, device="cuda"); sw = torch.zeros(1, dtype=torch.int32, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(reps):
        W = W0.clone()
        e0.record()
        _lib.call("cirr_orth", W.data_ptr(), n, c * n, n, c, nprob, 1e-12, sig.data_ptr(), order.data_ptr(), kept.data_ptr(),
                  Qt.data_ptr(), n, c * n, ws.data_ptr(), sw.data_ptr(), st)
        e1.record(); torch.cuda.synchronize()
    import ctypes
    ph = (ctypes.c_longlong * 4)()
    _lib.call("cirr_orth_phases", ctypes.addressof(ph))
    print(f"orth n={n} c={c} nprob={nprob}: {e0.elapsed_time(e1):.2f} ms sweeps={sw.item()} kept={kept.cpu().numpy()} "
          f"QR {(ph[1]-ph[0])/1e6:.2f} Jacobi {(ph[2]-ph[1])/1e6:.2f} Q {(ph[3]-ph[2])/1e6:.2f} Mcycles", flush=True)


if __name__ == "__main__" and len(sys.argv) == 1:
    for k in (120, 256):
        t_small(k, False)
        t_small(k, True)
    t_orth(4096, 256)
    t_orth(4096, 120)


def t_gen_split(k, nprob=2, reps=2):
    import ctypes
    rng = np.random.default_rng(k + 7)
    A = rng.standard_normal((nprob, k, k)) + 1j * rng.standard_normal((nprob, k, k))
    B = np.eye(k) + 0.05 * (rng.standard_normal((nprob, k, k)) + 1j * rng.standard_normal((nprob, k, k)))
    At, Bt = torch.from_numpy(A).cuda(), torch.from_numpy(np.ascontiguousarray(B)).cuda()
    kd = torch.full((nprob,), k, dtype=torch.int32, device="cuda")
    ws = torch.empty(_lib.call("cirr_gen_eig_ws_bytes", k, nprob), dtype=torch.uint8, device="cuda")
    lam = torch.empty((nprob, k), dtype=torch.complex128, device="cuda")
    info = torch.zeros(nprob, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(reps):
        e0.record()
        _lib.call("cirr_gen_eig_values", At.data_ptr(), Bt.data_ptr(), kd.data_ptr(), k, nprob, ws.data_ptr(),
                  lam.data_ptr(), info.data_ptr(), st)
        e1.record(); torch.cuda.synchronize()
    q = (ctypes.c_longlong * 8)()
    _lib.call("cirr_gen_eig_qr_stats", ctypes.addressof(q))
    print(f"gen_eig_values k={k} nprob={nprob}: {e0.elapsed_time(e1):.2f} ms  sweeps {q[0]} rot {q[1]} "
          f"defl {q[2]/1e6:.1f}M chain {q[3]/1e6:.1f}M far {q[4]/1e6:.1f}M cycles", flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "split":
    for k in (120, 256):
        t_gen_split(k)


def t_cholqr2(n, c, nprob=2, reps=3):
    rng = np.random.default_rng(c)
    u = np.linalg.qr(rng.standard_normal((n, c)) + 1j * rng.standard_normal((n, c)))[0]
    m = (u * np.logspace(0, -3, c)) @ np.linalg.qr(rng.standard_normal((c, c)) + 0j)[0]
    W = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(m.T, (nprob, c, n)))).cuda()
    cd = torch.full((nprob,), c, dtype=torch.int32, device="cuda")
    Qt = torch.empty((nprob, c, n), dtype=torch.complex128, device="cuda")
    ws = torch.empty(_lib.call("cirr_orth_cholqr2_ws_bytes", n, c, nprob), dtype=torch.uint8, device="cuda")
    ok = torch.zeros(nprob, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        _lib.call("cirr_orth_cholqr2", W.data_ptr(), n, c * n, n, c, nprob, cd.data_ptr(), 1e5, Qt.data_ptr(), n,
                  c * n, ws.data_ptr(), ok.data_ptr(), st)
        e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(f"cholqr2 n={n} c={c} nprob={nprob}: {min(ts):.2f} ms ok={ok.cpu().numpy()}", flush=True)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "orth":
    for c in (120, 256):
        t_orth(4096, c)
        t_cholqr2(4096, c)
