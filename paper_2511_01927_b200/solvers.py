"""CIRR contour-integral solver on one B200 -- the drop-in for cieig.solvers.

Public API mirrors the reference (cieig/solvers.py:25-377): ``SolverConfig``,
``SolveStats``, ``EigenResult``, ``MultiResult``, ``ProjectorContext``,
``apply_projector``, ``cirr_solve``, ``solve_multi``,
``write_eigenvectors``/``read_eigenvectors``.  Same argument meaning,
defaults, statistics and exceptions.  The arithmetic runs in libcirr.so
(hand-written sm_100a kernels, see include/cirr.h); this module only
orchestrates: it owns device buffers as torch tensors, keeps the reference's
host-side control flow (refinement loop, inside filter, convergence filter,
dedupe) and generates the probe block V with the same numpy call as the
reference so the inputs are bit-identical.

Deviations from the reference (all documented in DESIGN.md section 3):
  * moments are centred and scaled, ((z_j - gamma)/rho)^m (span-preserving);
  * non-Hermitian pencils use a general Rayleigh-Ritz (eig) and complex
    containment; ellipse contours are supported;
  * all contours of a ``solve_multi`` call are batched through K1-K3.
"""

from __future__ import annotations

import functools
import struct
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .contours import QuadratureRule, contains, contains_many, contains_rows, moment_frame, quadrature_for
from .errors import (
    ConvergenceError,
    DeviceError,
    DimensionError,
    IndefiniteBError,
    NoEigenvaluesFound,
    ParameterError,
    RankZeroError,
    SingularShiftError,
)

PIVOT_REL_TOL = 1e-14  # linalg.py:26
_DEBUG = bool(int(__import__("os").environ.get("CIRR_DEBUG", "0")))
# certified CholeskyQR2 basis for refinement blocks (CIRR_CHOLQR=0 forces the SVD path)
_CHOLQR = bool(int(__import__("os").environ.get("CIRR_CHOLQR", "1")))
_CHOLQR_KAPPA = 1e5
# previous-round eigenvalues as QR shift hints (CIRR_QR_HINTS=0 disables)
_QR_HINTS = bool(int(__import__("os").environ.get("CIRR_QR_HINTS", "1")))
# refinement rounds: Newton refinement of the eigenbasis W0 = Q^H S instead of
# the Hessenberg QR (CIRR_EIG_REFINE=0 disables; non-converged problems fall back)
_EIG_REFINE = bool(int(__import__("os").environ.get("CIRR_EIG_REFINE", "1")))
_EIG_REFINE_ITERS = 5
# large batches (>= _INTERLEAVE_MIN contours in a wave) run as _INTERLEAVE
# engines on their own streams, interleaved at their host syncs (CIRR_INTERLEAVE=1: one engine)
_INTERLEAVE = int(__import__("os").environ.get("CIRR_INTERLEAVE", "2"))
_INTERLEAVE_MIN = int(__import__("os").environ.get("CIRR_INTERLEAVE_MIN", "32"))
# banded pencils factor and solve on the band only (CIRR_BAND=0: always the dense ranges)
_BAND = bool(int(__import__("os").environ.get("CIRR_BAND", "1")))


@functools.lru_cache(maxsize=64)
def _band_lu_flops(n: int, kl: int, ku: int) -> float:
    """Algorithmic complex LU flops of an n x n pencil with kl sub- and ku
    superdiagonals: sum over columns of 8 (rows below) (columns right, fill-in
    included); 8 n^3 / 3 for a dense one."""
    c = np.arange(n, dtype=np.float64)
    rest = n - 1.0 - c
    return float(8.0 * np.sum(np.minimum(kl, rest) * np.minimum(kl + ku, rest)))


@functools.lru_cache(maxsize=64)
def _band_solve_unit(n: int, kl: int, ku: int) -> float:
    """Complex flops per right-hand side of one L and one U solve on factors
    of lower / upper bandwidth kl / ku (8 n^2 dense)."""
    i = np.arange(n, dtype=np.float64)
    return float(8.0 * (np.sum(np.minimum(i, kl)) + np.sum(np.minimum(n - 1.0 - i, ku))))


def _band_solve_flops(n: int, kl: int, ku: int, K: int) -> float:
    return K * _band_solve_unit(n, kl, ku)
# launches put the batch (pencils of a wave) on grid.y / grid.z, whose limit
# is 65535: a wave never holds more pencils than that
_MAX_WAVE_PENCILS = 65535
_MOMENT_CHUNK = 16  # cirr_moments handles up to 16 moments per launch (MAXM)



_TORCH_OK = None


def _torch():
    global _TORCH_OK
    if _TORCH_OK is not None:
        return _TORCH_OK
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("CUDA device not available: the CIRR path has no CPU fallback")
    _TORCH_OK = torch
    return torch


class _Cols:
    """Columns [0, k) of entry b of a (batch, n, K) device block, standing in
    for the torch view buf[b, :, :k] where the engine only needs its address,
    shape and strides (a torch view costs ~4 us of Python; config 2 makes two
    per contour per Rayleigh-Ritz round).  tensor() makes the real view."""
    __slots__ = ("buf", "b", "k")

    def __init__(self, buf, b: int, k: int):
        self.buf, self.b, self.k = buf, b, k

    @property
    def shape(self):
        return (self.buf.shape[1], self.k)

    def dim(self) -> int:
        return 2

    def numel(self) -> int:
        return self.buf.shape[1] * self.k

    def stride(self, d: int) -> int:
        return self.buf.stride(1) if d == 0 else 1

    def data_ptr(self) -> int:
        return self.buf.data_ptr() + self.b * self.buf.stride(0) * self.buf.element_size()

    def tensor(self):
        return self.buf[self.b, :, : self.k]

    def cpu(self):
        return self.tensor().cpu()

    def contiguous(self):
        return self.tensor().contiguous()

    def is_contiguous(self) -> bool:
        return self.k == self.buf.shape[2]


# ---------------------------------------------------------------------------
# configuration and result types (solvers.py:25-94)


@dataclass
class SolverConfig:
    n_q: int = 32
    source_cols: int | None = None  # default: max(8, 2 * expected_count)
    n_moments: int = 4
    max_refine: int = 8
    tol: float = 1e-10
    rank_rel_tol: float = 1e-12
    drop_tol: float = 1e-10
    # Labelled variant, not the reference's behaviour (SURVEY.md finding 9):
    # for the real pencils this path holds and a conjugate-symmetric node set,
    # factor only the upper-half nodes and recover the lower half from
    # M(conj z)^-1 R = conj(M(z)^-1 conj R).  Halves K1+K2 work.
    conjugate_pairs: bool = False
    # Labelled variant (SURVEY.md finding 8): stop refining a contour once its
    # converged set (pairs with residual <= tol) is unchanged across two passes.
    early_exit: bool = False
    # Arithmetic of the k = 512 updates of dense factorisations and solves:
    # None keeps the library mode (default int8: exact digit products on the
    # tcgen05 tensor cores, DESIGN.md section 3 item 8; CIRR_LU_GEMM=dmma or
    # cirr_set_lu_gemm(0) change it), "int8" / "f64" set it for this call.
    arith: str | None = None

    def __post_init__(self):
        if self.n_q < 4 or self.n_moments < 1 or self.max_refine < 1:
            raise ParameterError("counts must be >= 1 (n_q >= 4)")
        if self.tol <= 0:
            raise ParameterError("tol must be positive")
        if self.arith not in (None, "int8", "f64"):
            raise ParameterError("arith must be None, 'int8' or 'f64'")

    def cols_for(self, expected_count: int) -> int:
        if self.source_cols is not None:
            return self.source_cols
        return max(8, 2 * expected_count)


def _cfg_view(cfg) -> SolverConfig:
    """Accept a reference SolverConfig (duck-typed) or None."""
    if cfg is None:
        return SolverConfig()
    if isinstance(cfg, SolverConfig):
        return cfg
    return SolverConfig(n_q=cfg.n_q, source_cols=cfg.source_cols, n_moments=cfg.n_moments,
                        max_refine=cfg.max_refine, tol=cfg.tol, rank_rel_tol=cfg.rank_rel_tol,
                        drop_tol=getattr(cfg, "drop_tol", 1e-10),
                        conjugate_pairs=bool(getattr(cfg, "conjugate_pairs", False)),
                        early_exit=bool(getattr(cfg, "early_exit", False)),
                        arith=getattr(cfg, "arith", None))


@dataclass
class SolveStats:
    n_linear_solves: int = 0
    n_factorizations: int = 0
    iterations: int = 0
    elapsed: float = 0.0

    def to_dict(self) -> dict:
        return {"n_linear_solves": self.n_linear_solves, "n_factorizations": self.n_factorizations,
                "iterations": self.iterations, "elapsed": self.elapsed}


@dataclass
class EigenResult:
    eigenvalues: np.ndarray
    eigenvectors: np.ndarray  # (n, k)
    residuals: np.ndarray
    contour: object
    stats: SolveStats

    def to_json_dict(self) -> dict:
        ev = self.eigenvalues
        vals = ev.tolist() if not np.iscomplexobj(ev) else [[v.real, v.imag] for v in ev]
        return {"contour": self.contour.to_json_dict(), "eigenvalues": vals,
                "residuals": self.residuals.tolist(), "stats": self.stats.to_dict()}


@dataclass
class MultiResult:
    results: list
    errors: list
    stats: SolveStats

    @property
    def eigenvalues(self) -> np.ndarray:
        vals = [r.eigenvalues for r in self.results if r is not None]
        return np.sort(np.concatenate(vals)) if vals else np.array([])

    def to_json_dict(self) -> dict:
        ev = self.eigenvalues
        vals = ev.tolist() if not np.iscomplexobj(ev) else [[v.real, v.imag] for v in ev]
        return {"contours": [r.to_json_dict() if r is not None else {"error": str(e)}
                             for r, e in zip(self.results, self.errors)],
                "eigenvalues": vals, "stats": self.stats.to_dict()}


def _as_block(x) -> np.ndarray:  # linalg.py:29-35
    b = np.asarray(x, dtype=np.complex128)
    if b.ndim == 1:
        b = b[:, None]
    if b.ndim != 2:
        raise DimensionError("block must be 2-D")
    return b


def write_eigenvectors(path, block) -> None:  # solvers.py:80-87
    b = _as_block(block)
    with open(path, "wb") as fh:
        fh.write(struct.pack("<QQ", b.shape[0], b.shape[1]))
        fh.write(np.ascontiguousarray(b, dtype="<c16").tobytes())


def read_eigenvectors(path) -> np.ndarray:  # solvers.py:90-94
    with open(path, "rb") as fh:
        n_rows, n_cols = struct.unpack("<QQ", fh.read(16))
        data = np.frombuffer(fh.read(), dtype="<c16")
    return data.reshape(n_rows, n_cols)


# ---------------------------------------------------------------------------
# device pencil


def _dense(m) -> np.ndarray:
    if isinstance(m, np.ndarray):
        return m
    if hasattr(m, "to_dense"):
        return m.to_dense()
    if hasattr(m, "toarray"):
        return m.toarray()
    return np.asarray(m)


_HOST_POOL = None


def _host_pool():
    global _HOST_POOL
    if _HOST_POOL is None:
        from concurrent.futures import ThreadPoolExecutor

        _HOST_POOL = ThreadPoolExecutor(max_workers=8, thread_name_prefix="cirr-stage")
    return _HOST_POOL


def _upload(torch, x: np.ndarray):
    """Host matrix -> device.  Large matrices go through pinned staging (torch's
    caching host allocator) and an async copy: config 4's 134 MB A takes
    1.9 + 2.4 ms that way against 12.6 ms straight from pageable memory (the
    staging copy is the caller's data, so the array may change afterwards)."""
    t = torch.from_numpy(x)
    if x.nbytes >= (1 << 20):
        return t.pin_memory().to("cuda", non_blocking=True)
    return t.to("cuda")


class DevicePencil:
    """A, B resident in HBM, dense and row-major: real float64 when both are
    real (the configs), complex128 when either has a nonzero imaginary part
    (the reference's MatrixPencil holds complex128 CSR values, sparse.py:14-43)."""

    def __init__(self, a, b, hermitian: bool | None = None):
        torch = _torch()
        if isinstance(a, torch.Tensor) and isinstance(b, torch.Tensor):
            self._from_tensors(torch, a, b, hermitian)
            return
        a = np.asarray(_dense(a))
        b = np.asarray(_dense(b))
        if a.ndim != 2 or a.shape[0] != a.shape[1] or a.shape != b.shape:
            raise DimensionError("pencil matrices must be square and equally sized")
        cx = any(np.iscomplexobj(m) and np.abs(m.imag).max(initial=0.0) != 0.0 for m in (a, b))
        self.complex = cx
        dt = np.complex128 if cx else np.float64
        a = np.ascontiguousarray(a if cx else a.real, dtype=dt)
        b = np.ascontiguousarray(b if cx else b.real, dtype=dt)
        self.n = a.shape[0]
        self.a = _upload(torch, a)
        self.b = _upload(torch, b)
        self.hermitian = bool(hermitian) if hermitian else self._device_symmetric()

    @property
    def gemm_kind(self) -> int:
        """cirr_gemm operand kind of A and B: 2 = real float64, 0 = complex128."""
        return 0 if self.complex else 2

    def assemble(self, z, cnt: int, pencils, maxabs, stream):
        """K1: pencils[j] = z[j] B - A for cnt shifts (cirr_assemble / cirr_assemble_c)."""
        n = self.n
        _lib.call("cirr_assemble_c" if self.complex else "cirr_assemble", _ptr(self.a), _ptr(self.b), n, n, _ptr(z),
                  cnt, _ptr(pencils), n, n * n, _ptr(maxabs), stream)

    def _device_symmetric(self, rel_tol: float = 1e-12) -> bool:
        """sparse.py:83-87 applied to A and B on the device (a flag of False or
        None means 'unknown' here, as the reference's default is False)."""
        torch = _torch()
        out = torch.empty((2, 2), dtype=torch.float64, device="cuda")
        st = _stream()
        fn = "cirr_hermitian_c" if self.complex else "cirr_symmetry"
        _lib.call(fn, _ptr(self.a), self.n, self.n, _ptr(out[0]), st)
        _lib.call(fn, _ptr(self.b), self.n, self.n, _ptr(out[1]), st)
        o = out.cpu().numpy()
        return bool(all(o[i, 0] <= rel_tol * max(o[i, 1], 1e-300) for i in range(2)))

    def _from_tensors(self, torch, a, b, hermitian):
        """float64 or complex128 tensors (host, ideally pinned, or device): copied
        with non_blocking H2D; the Hermitian flag must be given or is computed on
        the device."""
        if a.dim() != 2 or a.shape[0] != a.shape[1] or a.shape != b.shape:
            raise DimensionError("pencil matrices must be square and equally sized")
        ok = (torch.float64, torch.complex128)
        if a.dtype not in ok or b.dtype not in ok:
            raise NotImplementedError("tensor pencils must be float64 or complex128")
        self.complex = a.dtype == torch.complex128 or b.dtype == torch.complex128
        dt = torch.complex128 if self.complex else torch.float64
        self.n = a.shape[0]
        self.a = a.to("cuda", non_blocking=True).to(dt).contiguous()
        self.b = b.to("cuda", non_blocking=True).to(dt).contiguous()
        self.hermitian = bool(hermitian) if hermitian else self._device_symmetric()

    @staticmethod
    def bands(dps) -> list:
        """(kl, ku) of each DevicePencil (cached on it): one batched device pass
        over the uncached A and B (cirr_bandwidth_ptrs, grouped by order and
        dtype), one read-back for all of them."""
        todo = [d for d in dps if getattr(d, "_band", None) is None]
        if todo:
            torch = _torch()
            groups: dict = {}
            for d in todo:
                groups.setdefault((d.n, d.complex), []).append(d)
            bufs = []
            for (n, cx), ds in groups.items():
                ptrs = _h2d(np.array([[d.a.data_ptr(), d.b.data_ptr()] for d in ds], dtype=np.int64).reshape(-1))
                buf = _zeros((2 * len(ds), 2), torch.int32)
                _lib.call("cirr_bandwidth_ptrs", _ptr(ptrs), 2 * len(ds), 1 if cx else 0, n, n, _ptr(buf), _stream())
                bufs.append((ds, buf))
            for ds, buf in bufs:
                v = buf.cpu().numpy().reshape(len(ds), 2, 2).max(axis=1)
                for d, (kl, ku) in zip(ds, v.tolist()):
                    d._band = (int(kl), int(ku))
        return [d._band for d in dps]

    @classmethod
    def of(cls, pencil):
        if isinstance(pencil, DevicePencil):
            return pencil
        return cls(pencil.a, pencil.b, getattr(pencil, "hermitian", None))

    @classmethod
    def of_many(cls, pencils) -> list:
        """``[DevicePencil.of(p) for p in pencils]`` with the host pencils of one
        order and dtype staged into one pinned buffer by a few host threads
        (numpy's copies release the GIL) and moved in one async H2D copy.
        Config 2's 256 pencils: 38 ms as 512 pageable copies.  Each matrix
        starts on a 256-byte boundary of the staging buffer."""
        torch = _torch()
        out = [p if isinstance(p, DevicePencil) else None for p in pencils]
        groups: dict = {}
        for i, p in enumerate(pencils):
            if out[i] is not None:
                continue
            if isinstance(p.a, torch.Tensor) or isinstance(p.b, torch.Tensor):
                out[i] = cls.of(p)
                continue
            a = np.asarray(_dense(p.a))
            b = np.asarray(_dense(p.b))
            if a.ndim != 2 or a.shape[0] != a.shape[1] or a.shape != b.shape:
                raise DimensionError("pencil matrices must be square and equally sized")
            cx = any(np.iscomplexobj(m) and np.abs(m.imag).max(initial=0.0) != 0.0 for m in (a, b))
            if not cx:
                a, b = a.real, b.real
            groups.setdefault((a.shape[0], cx), []).append((i, a, b, getattr(p, "hermitian", None)))
        for (n, cx), items in groups.items():
            if len(items) == 1:
                i, a, b, h = items[0]
                out[i] = cls(a, b, h)
                continue
            tdt = torch.complex128 if cx else torch.float64
            esz = 16 if cx else 8
            slot = -(-n * n * esz // 256) * 256 // esz
            buf = torch.empty(len(items) * 2 * slot, dtype=tdt, pin_memory=True)
            view = buf.numpy()

            def fill(js, view=view, items=items, slot=slot, n=n):
                for j in js:
                    _, a, b, _ = items[j]
                    view[(2 * j) * slot:(2 * j) * slot + n * n].reshape(n, n)[...] = a
                    view[(2 * j + 1) * slot:(2 * j + 1) * slot + n * n].reshape(n, n)[...] = b

            nt = min(8, len(items))
            list(_host_pool().map(fill, [range(t, len(items), nt) for t in range(nt)]))
            dev = buf.to("cuda", non_blocking=True)
            for j, (i, _, _, h) in enumerate(items):
                d = cls.__new__(cls)
                d.complex = cx
                d.n = n
                d.a = dev[(2 * j) * slot:(2 * j) * slot + n * n].view(n, n)
                d.b = dev[(2 * j + 1) * slot:(2 * j + 1) * slot + n * n].view(n, n)
                d.hermitian = bool(h) if h else d._device_symmetric()
                out[i] = d
        return out


def _is_symmetric(m: np.ndarray, rel_tol: float = 1e-12) -> bool:  # sparse.py:83-87
    scale = max(float(np.abs(m).max()) if m.size else 0.0, 1e-300)
    return float(np.abs(m - m.T).max(initial=0.0)) <= rel_tol * scale


class StageTimer:
    """CUDA-event timing of engine stages on the launching stream (bench.py).

    ``with timer.stage("lu"):`` brackets the enqueue of a stage; ``totals()``
    (after a synchronize) returns milliseconds per stage name summed over
    every bracket, plus per-stage work counters the engine adds.
    """

    def __init__(self):
        self.events = []
        self.work = {}

    def stage(self, name):
        timer = self

        class _Ctx:
            def __enter__(self_inner):
                torch = _torch()
                self_inner.e0 = torch.cuda.Event(enable_timing=True)
                self_inner.e1 = torch.cuda.Event(enable_timing=True)
                self_inner.e0.record()

            def __exit__(self_inner, *exc):
                self_inner.e1.record()
                timer.events.append((name, self_inner.e0, self_inner.e1))
                return False

        return _Ctx()

    def add(self, name, amount):
        self.work[name] = self.work.get(name, 0) + amount

    def totals(self) -> dict:
        out = {}
        for name, e0, e1 in self.events:
            out[name] = out.get(name, 0.0) + e0.elapsed_time(e1)
        return out

    def reset(self):
        self.events.clear()
        self.work.clear()


_TIMER: StageTimer | None = None


class NodeShard:
    """One GEP split over ranks by quadrature node: rank r
    factors and solves the nodes r, r + world, ... of every contour, the moment
    blocks are summed over the ranks once per pass (``allreduce(tensor, op)``,
    op in {"sum", "min"}, in place on a device tensor), and every rank then
    runs the same Rayleigh-Ritz on identical data.  Installed per thread by
    ``dist.solve_multi_node_sharded``."""

    def __init__(self, rank: int, world: int, allreduce):
        if world < 1 or not 0 <= rank < world:
            raise ParameterError("bad rank/world for the node shard")
        self.rank, self.world, self.allreduce = rank, world, allreduce


_SHARD = __import__("threading").local()


def _node_shard():
    sh = getattr(_SHARD, "value", None)
    return sh if sh is not None and sh.world > 1 else None


def set_node_shard(shard):
    """Install (or clear, with None) the calling thread's NodeShard; returns the previous one."""
    prev = getattr(_SHARD, "value", None)
    _SHARD.value = shard
    return prev


def set_stage_timer(timer: StageTimer | None) -> None:
    global _TIMER
    _TIMER = timer


class _NoStage:
    def __enter__(self):
        return None

    def __exit__(self, *exc):
        return False


def _stage(name):
    return _TIMER.stage(name) if _TIMER is not None else _NoStage()


def _work(name, amount):
    if _TIMER is not None:
        _TIMER.add(name, amount)


def _stream():
    torch = _torch()
    return ctypes_ptr(torch.cuda.current_stream().cuda_stream)


def ctypes_ptr(v) -> int:
    return int(v)


def _ptr(t) -> int:
    return t.data_ptr()


def _zeros(shape, dtype=None):
    """A zero-filled device tensor: torch allocates, libcirr zero-fills (a
    stream-ordered memset, no PyTorch kernel on the path)."""
    torch = _torch()
    t = torch.empty(shape, dtype=dtype or torch.complex128, device="cuda")
    if t.numel():
        _lib.call("cirr_zero", _ptr(t), t.numel() * t.element_size(), _stream())
    return t


def _piece(src, d: int, c0: int = 0, conj: bool = False, rows: int | None = None, cols: int | None = None,
           dst_ld: int = 0):
    """Descriptor of one 2-D complex block (a row-major view with unit column
    stride) for _gather: its rows x cols elements go to entry d, column c0
    (row pitch dst_ld, default the destination's)."""
    if src.dim() == 1:
        src = src[None, :]
    r, c = src.shape
    ld = src.stride(0) if r > 1 else c
    if c > 1 and src.stride(1) != 1:
        raise DeviceError("gather source must have unit column stride")
    return (src.data_ptr(), ld, r if rows is None else rows, c if cols is None else cols, d, c0, 1 if conj else 0,
            dst_ld)


def _gather(pieces: list, dst):
    """Copy the pieces into dst with one libcirr launch per 65535 pieces
    (cirr_gather_blocks).  dst is (entries x rows x cols) and a piece's index
    names its entry, or 2-D (rows x cols) and the index names its first row."""
    if not pieces:
        return dst
    ld = dst.stride(-2)
    sd = dst.stride(0)
    for a in range(0, len(pieces), 65535):
        part = pieces[a:a + 65535]
        desc = _h2d(np.asarray(part, dtype=np.int64).reshape(-1))
        mx = max(p_[2] * p_[3] for p_ in part)
        _lib.call("cirr_gather_blocks", len(part), _ptr(desc), mx, _ptr(dst), ld, sd, _stream())
    return dst


def _h2d(x: np.ndarray):
    """Host array -> device tensor, stream-ordered on the current stream with no
    host synchronisation, so enqueueing never waits for earlier GPU work of
    that stream.  Small arrays (the engine's index arrays, coefficients and
    descriptors) go straight from pageable memory: cudaMemcpyAsync stages them
    and returns without a device sync (6 us on the B200 boxes, against 12 us
    for pin_memory()); larger ones through pinned staging."""
    torch = _torch()
    x = np.ascontiguousarray(x)
    if x.nbytes <= 65536:
        return torch.from_numpy(x).to("cuda", non_blocking=True)
    return torch.from_numpy(x).pin_memory().to("cuda", non_blocking=True)


def _drain(gen):
    """Run an engine generator to completion and return its value.  The
    engine's phases are generators that yield just before each blocking
    device-to-host read: alone they run straight through (this), and two
    engines on their own streams can be interleaved (_interleave) so one's
    host work overlaps the other's queued GPU work."""
    while True:
        try:
            next(gen)
        except StopIteration as e:
            return e.value


# ---------------------------------------------------------------------------
# the engine: factor + solve + moments for a set of contours


class _Contour:
    def __init__(self, idx, contour, cfg: SolverConfig, seed: int, n: int, complex_pencil: bool = False):
        self.idx = idx
        self.contour = contour
        rule = quadrature_for(contour, cfg.n_q)
        self.nodes = np.asarray(rule.nodes, dtype=np.complex128)
        self.weights = np.asarray(rule.weights, dtype=np.complex128)
        self.all_nodes = self.nodes
        self.node_ids = np.arange(len(self.nodes))     # position of each kept node in the full rule
        sh = _node_shard()
        if sh is not None:
            if len(self.nodes) < sh.world:
                raise ParameterError(f"n_q = {len(self.nodes)} nodes cannot be split over {sh.world} ranks")
            self.node_ids = np.arange(sh.rank, len(self.nodes), sh.world)
            self.nodes = self.nodes[self.node_ids]
            self.weights = self.weights[self.node_ids]
        self.gamma, self.rho = moment_frame(contour)
        self.ncols = cfg.cols_for(getattr(contour, "expected_count", 0))
        self.seed = seed
        self.stats = SolveStats()
        self.error = None
        self.result = None
        self.t0 = time.perf_counter()
        # solver state
        self.lam = self.res = None
        self.best_res = np.inf
        self.x_dev = None  # inside Ritz vectors on device (n x kin)
        self.done = False
        # factored nodes (all of them unless the conjugate-pair variant applies)
        self.half = False
        self.fidx = np.arange(len(self.nodes))
        if cfg.conjugate_pairs and not complex_pencil:
            self._pair()      # M(conj z) = conj(M(z)) needs real A and B

    def _pair(self):
        """fidx = upper-half nodes; mate[j] = position in fidx of conj(z_j)."""
        z = self.nodes
        N = len(z)
        up = np.flatnonzero(z.imag > 0)
        if N % 2 or len(up) * 2 != N:
            return
        scale = max(float(np.abs(z).max()), 1e-300)
        mate = np.full(N, -1)
        for r, j in enumerate(up):
            mate[j] = r
            k = int(np.argmin(np.abs(z - np.conj(z[j]))))
            if abs(z[k] - np.conj(z[j])) > 1e-13 * scale or z[k].imag >= 0 or mate[k] >= 0:
                return
            mate[k] = r
        if np.any(mate < 0):
            return
        self.half, self.fidx, self.mate = True, up, mate

    def settled(self, lam: np.ndarray, res: np.ndarray, tol: float) -> bool:
        """Early-exit variant: True when the converged set (residual <= tol)
        is unchanged from the previous pass (same count, eigenvalues equal to
        1e-10 relative, matched nearest-neighbour) and reaches the contour's
        expected_count; without an expected count the set must be unchanged
        over three passes.  On config 4 a stable set short of the count still
        gains pairs later, so stability alone would drop eigenpairs."""
        conv = np.asarray(lam)[np.asarray(res) <= tol]
        hist = getattr(self, "_conv_hist", [])
        self._conv_hist = (hist + [conv])[-3:]
        need = 2 if getattr(self.contour, "expected_count", 0) > 0 else 3
        if len(self._conv_hist) < need or len(conv) == 0:
            return False
        scale = max(float(np.abs(conv).max()), 1e-300)
        for prev in self._conv_hist[-need:-1]:
            if len(prev) != len(conv):
                return False
            d = np.abs(conv[:, None] - prev[None, :])
            if max(float(d.min(axis=1).max()), float(d.min(axis=0).max())) > 1e-10 * scale:
                return False
        return len(conv) >= getattr(self.contour, "expected_count", 0)

    def coef(self, moments: int) -> np.ndarray:
        """c[j, m] = w_j zeta_j^m with zeta_j = (z_j - gamma)/rho (sequential powers;
        made once per moment count, read-only)."""
        cache = self.__dict__.setdefault("_coef_cache", {})
        if moments not in cache:
            cache[moments] = self._coef(moments)
        return cache[moments]

    def _coef(self, moments: int) -> np.ndarray:
        if moments == 1:  # w_j * (1+0j): exact products, so numpy's multiply gives the loop's bits
            return (self.weights * (1.0 + 0.0j))[:, None].copy()
        return _coef_rows(self.nodes, self.weights, self.gamma, self.rho, moments)


def _coef_batch(cs: list, moments: int) -> np.ndarray:
    """The stacked moment coefficients of several contours (rows in node
    order, contour after contour): _Contour._coef over all of them at once
    (the same real arithmetic, so the same bits)."""
    if len(cs) == 1:
        return cs[0].coef(moments)
    w = np.concatenate([c.weights for c in cs])
    if moments == 1:
        return (w * (1.0 + 0.0j))[:, None].copy()
    z = np.concatenate([c.nodes for c in cs])
    cnt = [len(c.nodes) for c in cs]
    gamma = np.repeat(np.array([c.gamma for c in cs], dtype=np.complex128), cnt)
    rho = np.repeat(np.array([c.rho for c in cs], dtype=np.float64), cnt)
    return _coef_rows(z, w, gamma, rho, moments)


def _coef_rows(z, w, gamma, rho, moments: int) -> np.ndarray:
    # zp_0 = 1, zp_m = zp_{m-1} * zeta and c = w zp with every complex product
    # written out in real arithmetic (rounded products, then the sum): the bits
    # of the scalar loop (numpy's vectorised complex multiply contracts to FMA
    # and differs in the last ulp)
    zeta = (z - gamma) / rho
    zr, zi = zeta.real, zeta.imag
    wr, wi = w.real, w.imag
    out = np.empty((len(z), moments), dtype=np.complex128)
    pr, pi = np.ones(len(z)), np.zeros(len(z))
    for m in range(moments):
        out[:, m].real = wr * pr - wi * pi
        out[:, m].imag = wr * pi + wi * pr
        pr, pi = pr * zr - pi * zi, pr * zi + pi * zr
    return out


def _pad_stack(blocks: list, dim: int, width: int):
    """Stack 2-D complex device blocks into (len, ...) zero-padded to `width`
    along their axis `dim` (0 or 1): one zero fill and one cirr_gather_blocks
    launch for the whole list."""
    shape = list(blocks[0].shape)
    shape[dim] = width
    out = _zeros([len(blocks)] + shape)
    return _gather([_piece(b, i) for i, b in enumerate(blocks) if b.numel()], out)


_SOURCE_CACHE: dict = {}


def _source_block(seed: int, n: int, ncols: int) -> np.ndarray:
    """default_rng(seed).standard_normal((n, ncols)) (solvers.py:178-180),
    memoised: many contours of a batch share a seed (solve_multi's seed + i)."""
    key = (int(seed), int(n), int(ncols))
    v = _SOURCE_CACHE.get(key)
    if v is None:
        if len(_SOURCE_CACHE) >= 64:
            _SOURCE_CACHE.pop(next(iter(_SOURCE_CACHE)))
        v = np.random.default_rng(seed).standard_normal((n, ncols))
        v.setflags(write=False)
        _SOURCE_CACHE[key] = v
    return v


class _Engine:
    """Batched CIRR over the contours of one wave (factors stay resident).

    Every contour normally belongs to one pencil ``dp``; under
    ``solve_multi_batch`` each contour carries its own (``_Contour.dp``, same
    n, dtype and Hermitian flag), and the per-pencil products gather A and B
    per contour."""

    def __init__(self, dp: DevicePencil, cstates: list, cfg: SolverConfig):
        self.torch = _torch()
        self.dp = dp
        self.cs = cstates
        self.cfg = cfg
        self.n = dp.n
        self.multi = any(getattr(c, "dp", dp) is not dp for c in cstates)
        self.dinv = None            # diagonal-block inverses: allocated and made on first use
        self.ozbuf = None           # int8 digit slices of the factors (blocked solves), made on first use

    def _dp_of(self, ci: int) -> DevicePencil:
        return getattr(self.cs[ci], "dp", None) or self.dp

    def _mats(self, cis: list):
        """(A, B, batch stride) for the pencils of contours cis in order: the
        shared pencil with stride 0, else (A address array, B address array,
        None) for cirr_gemm_ptrs (no stacked copies)."""
        dps = [self._dp_of(ci) for ci in cis]
        if all(d is dps[0] for d in dps):
            return dps[0].a, dps[0].b, 0
        key = tuple(cis)
        cache = self.__dict__.setdefault("_mat_ptrs", {})
        if key not in cache:
            cache[key] = (_h2d(np.array([d.a.data_ptr() for d in dps], dtype=np.int64)),
                          _h2d(np.array([d.b.data_ptr() for d in dps], dtype=np.int64)), None)
        return cache[key]

    def _gemm_mats(self, M, N, K, batch, mat, stride, Bt, ldb, sB, C, ldc, sC):
        """C[b] = mat[b] @ Bt[b] with mat from _mats (shared, or address array)."""
        kind = self.dp.gemm_kind
        if stride is None:
            _lib.call("cirr_gemm_ptrs", kind, M, N, K, batch, _ptr(mat), K, _ptr(Bt), ldb, sB, _ptr(C), ldc, sC, 1.0,
                      0, self.stream)
        else:
            _lib.call("cirr_gemm", kind, M, N, K, batch, _ptr(mat), K, stride, _ptr(Bt), ldb, sB, _ptr(C), ldc, sC,
                      1.0, 0, self.stream)

    def _pencil_runs(self, a: int, b: int):
        """Maximal ranges [lo, hi) of pencils a..b-1 that share one DevicePencil."""
        runs = []
        for ci in range(len(self.cs)):
            lo, hi = max(self.node_off[ci], a), min(self.node_off[ci + 1], b)
            if lo >= hi:
                continue
            d = self._dp_of(ci)
            if runs and runs[-1][2] is d and runs[-1][1] == lo:
                runs[-1][1] = hi
            else:
                runs.append([lo, hi, d])
        return runs

    @property
    def stream(self) -> int:
        """The launching stream: torch's current stream of the calling thread."""
        return _stream()

    # -- K1 + K2 -----------------------------------------------------------
    def _alloc_factors(self):
        torch, n = self.torch, self.n
        self.node_off = [0]
        for c in self.cs:
            self.node_off.append(self.node_off[-1] + len(c.fidx))
        P = self.node_off[-1]
        self.P = P
        self.pencils = torch.empty((P, n, n), dtype=torch.complex128, device="cuda")
        self.maxabs = torch.empty(P, dtype=torch.float64, device="cuda")
        self.ipiv = torch.empty((P, n), dtype=torch.int32, device="cuda")
        self.perm = torch.empty((P, n), dtype=torch.int32, device="cuda")
        self.minpiv = torch.empty(P, dtype=torch.float64, device="cuda")
        self.info = torch.empty(P, dtype=torch.int32, device="cuda")
        self.lbw = _zeros(P, torch.int32)
        # the wave's band: the widest of its pencils (dense: n - 1, n - 1)
        n = self.n
        if _BAND:
            bands = DevicePencil.bands([self._dp_of(ci) for ci in range(len(self.cs))])
            self.kl = min(n - 1, max(b_[0] for b_ in bands))
            self.ku = min(n - 1, max(b_[1] for b_ in bands))
        else:
            self.kl = self.ku = n - 1
        self.klL, self.kuU = n - 1, n - 1   # factor bandwidths, known after the factor read-back
        self._dinv_per_pencil = int(_lib.call("cirr_diag_inv_bytes", n, 1))
        self.contour_of = _h2d(
            np.concatenate([np.full(len(c.fidx), i, dtype=np.int32) for i, c in enumerate(self.cs)]))

    def _factor_range(self, a: int, b: int, nodes: np.ndarray):
        """Enqueue K1 + K2 for pencils
        a..b-1 (shifts `nodes`) on the current stream, as one batched call: the
        panel steps are latency-bound per launch, so one launch over every
        pencil of the wave costs the same as one over a single contour."""
        torch, n = self.torch, self.n
        cnt = b - a
        if cnt == 0:
            return
        z = _h2d(nodes)
        with _stage("assemble"):
            runs = self._pencil_runs(a, b)
            if len(runs) > 2 and not self.dp.complex:
                # many GEPs (solve_multi_batch): one launch over all of them
                ap = np.concatenate([np.full(hi - lo, d.a.data_ptr(), dtype=np.int64) for lo, hi, d in runs])
                bp = np.concatenate([np.full(hi - lo, d.b.data_ptr(), dtype=np.int64) for lo, hi, d in runs])
                ptrs = _h2d(np.stack([ap, bp]))
                _lib.call("cirr_assemble_ptrs", _ptr(ptrs[0]), _ptr(ptrs[1]), n, n, _ptr(z), cnt,
                          _ptr(self.pencils[a]), n, n * n, _ptr(self.maxabs[a:]), self.stream)
            else:
                for lo, hi, d in runs:
                    d.assemble(z[lo - a:], hi - lo, self.pencils[lo], self.maxabs[lo:], self.stream)
        _work("assemble_bytes", cnt * n * n * 16 + 2 * n * n * 8)
        kl, ku = self.kl, self.ku
        with _stage("lu"):
            lws = torch.empty(int(_lib.call("cirr_zgetrf_ws_bytes", n, cnt)), dtype=torch.uint8, device="cuda")
            # banded pencils (the stencil configs): the LU on the band only,
            # bitwise the dense factors; lbw collects L's bandwidth after pivoting
            _lib.call("cirr_zgetrf_band", _ptr(self.pencils[a]), n, n, n * n, cnt, kl, ku, _ptr(self.ipiv[a]),
                      _ptr(self.perm[a]), _ptr(self.minpiv[a:]), _ptr(self.info[a:]), _ptr(self.lbw[a:]),
                      _ptr(lws), self.stream)
        _work("lu_flops", cnt * _band_lu_flops(n, kl, ku))

    def _diag_inverses(self, a: int, b: int):
        with _stage("dinv"):
            _lib.call("cirr_diag_inverses", _ptr(self.pencils[a]), self.n, self.n, self.n * self.n, b - a,
                      _ptr(self.dinv) + a * self._dinv_per_pencil, self.stream)

    def factor(self, sources: bool = False):
        """K1 + K2 for the wave, then the singular-shift test (one read-back).
        sources: also enqueue the CIRR source blocks B V before that read-back,
        so their host-side generation overlaps the factorisation."""
        return _drain(self.factor_g(sources))

    def factor_g(self, sources: bool = False):
        self._alloc_factors()
        self._factor_range(0, self.P, np.concatenate([c.nodes[c.fidx] for c in self.cs]))
        if sources:
            self._src = self.source_blocks(list(range(len(self.cs))))
        yield
        # one read-back for every contour of the wave; linalg.py:68-70 on all
        # pencils at once, the first failing node of each contour reported
        maxabs, minpiv, info, lbw = (t.cpu().numpy() for t in (self.maxabs, self.minpiv, self.info, self.lbw))
        n = self.n
        self.klL = min(n - 1, max(self.kl, int(lbw.max(initial=0))))
        self.kuU = min(n - 1, self.kl + self.ku)
        if _DEBUG:
            print(f"[cirr] band kl={self.kl} ku={self.ku} -> factors klL={self.klL} kuU={self.kuU} (n={n})", flush=True)
        bad = (info != 0) | ~(minpiv >= PIVOT_REL_TOL * np.maximum(maxabs, 1e-300))
        for ci, c in enumerate(self.cs):
            c.stats.n_factorizations = len(c.fidx)
        seen = set()
        sh = _node_shard()
        first = np.full(len(self.cs), np.iinfo(np.int64).max, dtype=np.int64)   # first failing node, full-rule index
        for j in np.flatnonzero(bad):
            ci = int(np.searchsorted(self.node_off, j, side="right")) - 1
            if ci in seen:
                continue
            seen.add(ci)
            c = self.cs[ci]
            jn = int(c.fidx[j - self.node_off[ci]])
            first[ci] = int(c.node_ids[jn])
        if sh is not None:   # every rank must drop the same contours: the smallest failing node over the ranks
            ft = _h2d(first)
            sh.allreduce(ft, "min")
            first = ft.cpu().numpy()
        for ci, c in enumerate(self.cs):
            if first[ci] != np.iinfo(np.int64).max:
                g = int(first[ci])
                c.error = SingularShiftError(complex(c.all_nodes[g]), node_index=g)
                c.done = True

    # -- K3: solve all pencils of the listed contours against per-contour RHS
    def apply(self, active: list, rhs: dict, moments: int, real_rhs: bool = False) -> dict:
        """rhs[ci] = device (n x K_ci) complex block (already multiplied by B).
        Returns St[ci] = device ((moments*K) x n) transposed moment block.
        real_rhs: the blocks are known to be real (conjugate-pair variant: the
        mirrored nodes then need no extra columns).  No host synchronisation."""
        torch, n = self.torch, self.n
        K = max(rhs[ci].shape[1] for ci in active)
        if K == 0:
            return {ci: torch.empty((0, n), dtype=torch.complex128, device="cuda") for ci in active}
        nset = len(active)
        # solve width per contour: conjugate-pair contours with a complex
        # block solve [R | conj R] on their upper-half factors
        ks, cplx_rhs = [], []
        for ci in active:
            kc = rhs[ci].shape[1]
            cx = self.cs[ci].half and not real_rhs
            cplx_rhs.append(cx)
            ks.append(2 * kc if cx else kc)
        Ks = max(ks)
        r0 = rhs[active[0]]
        if nset == 1 and not cplx_rhs[0] and r0.is_contiguous():
            R = (r0.tensor() if isinstance(r0, _Cols) else r0).unsqueeze(0)   # the block itself
        else:  # one gather launch (+ a zero fill when widths differ)
            R = _zeros((nset, n, Ks)) if any(k_ < Ks for k_ in ks) else torch.empty(
                (nset, n, Ks), dtype=torch.complex128, device="cuda")
            pieces = []
            for s, ci in enumerate(active):
                kc = rhs[ci].shape[1]
                if kc:
                    pieces.append(_piece(rhs[ci], s))
                    if cplx_rhs[s]:
                        pieces.append(_piece(rhs[ci], s, kc, conj=True))
            _gather(pieces, R)
        pen_idx, spos = [], [0]
        offs = [0]
        for s, ci in enumerate(active):
            a, b = self.node_off[ci], self.node_off[ci + 1]
            pen_idx.append((a, b))
            spos.append(spos[-1] + (b - a))
            offs.append(offs[-1] + len(self.cs[ci].nodes))
        coefs = _coef_batch([self.cs[ci] for ci in active], moments)
        Psolve, Ptot = spos[-1], offs[-1]
        Ysol = torch.empty((Psolve, n, Ks), dtype=torch.complex128, device="cuda")
        rhs_of = _h2d(np.repeat(np.arange(nset, dtype=np.int32), [b - a for a, b in pen_idx]))
        coef = _h2d(coefs)
        off_t = _h2d(np.asarray(offs, dtype=np.int32))
        St = torch.empty((nset, moments * K, n), dtype=torch.complex128, device="cuda")
        # solve contour ranges; ranges that are adjacent in the pencil buffer go
        # in one batched call (rhs_of picks each pencil's block), so the small
        # diagonal-block GEMMs of the blocked solve get twice the tiles per launch
        runs = []
        for s, (a, b) in enumerate(pen_idx):
            if runs and runs[-1][1] == a:
                runs[-1][1] = b
            else:
                runs.append([a, b])
        # the moment accumulation runs inside the solve call (cirr_zgetrs_moments)
        # unless the conjugate-pair variant must first expand the solved nodes
        fused = Psolve == Ptot and Ks == K and moments <= _MOMENT_CHUNK
        with _stage("solve"):
            dinv = self._dinv(Ks)
            dptr = _ptr(dinv) if dinv is not None else 0
            if dinv is not None:
                self._oz_slices(Ks)
            if len(runs) > 1:
                # scattered contours (refinement passes of a multi-pencil batch):
                # one gathered call over their factors instead of one per run
                pen_of = _h2d(np.concatenate([np.arange(a, b, dtype=np.int32) for a, b in pen_idx]))
                base, pen_ptr, fac_args = self.pencils, _ptr(pen_of), (_ptr(self.perm), dptr)
            else:
                a, b = runs[0]
                base, pen_ptr = self.pencils[a], 0
                fac_args = (_ptr(self.perm[a]), _ptr(dinv) + a * self._dinv_per_pencil if dinv is not None else 0)
            # one entry for the fused (moments), gathered and plain solves, cut
            # to the factors' band (bitwise the dense solves)
            mom = (_ptr(coef), moments, _ptr(off_t), nset, _ptr(St), n, moments * K * n) if fused else \
                (0, 0, 0, 0, 0, 0, 0)
            _lib.call("cirr_zgetrs_band", _ptr(base), n, n, n * n, self.P, pen_ptr, Psolve, fac_args[0], _ptr(R), Ks,
                      n * Ks, _ptr(rhs_of), Ks, _ptr(Ysol), Ks, n * Ks, fac_args[1], *mom, self.klL, self.kuU,
                      self.stream)
        _work("solve_flops", Psolve * _band_solve_flops(n, self.klL, self.kuU, Ks))
        _work("solve_flops_exec", _band_solve_unit(n, self.klL, self.kuU) * sum((b - a) * k
                                                                             for (a, b), k in zip(pen_idx, ks)))
        _work("moment_flops", Ptot * 8.0 * n * K * moments)
        if fused:
            del Ysol
        else:
            if Psolve == Ptot and Ks == K:
                Y = Ysol
            else:  # conjugate-pair variant: expand to every node in quadrature order
                Y = torch.zeros((Ptot, n, K), dtype=torch.complex128, device="cuda")
                with _stage("solve"):
                    for s, ci in enumerate(active):
                        c = self.cs[ci]
                        kc = rhs[ci].shape[1]
                        N = len(c.nodes)
                        if c.half:
                            up = np.zeros(N, dtype=bool)
                            up[c.fidx] = True
                            src = spos[s] + c.mate
                            cj = (~up).astype(np.int32)
                            col0 = np.where(up, 0, kc if cplx_rhs[s] else 0)
                        else:
                            src, cj, col0 = spos[s] + np.arange(N), np.zeros(N, np.int32), np.zeros(N)
                        meta = _h2d(np.stack([src, col0, cj]).astype(np.int32))
                        _lib.call("cirr_copy_cols", _ptr(Ysol), Ks, n * Ks, _ptr(meta[0]), _ptr(meta[1]),
                                  _ptr(meta[2]), n, kc, N, _ptr(Y[offs[s]]), K, n * K, self.stream)
                del Ysol
            with _stage("moments"):
                if moments <= _MOMENT_CHUNK:
                    _lib.call("cirr_moments", _ptr(Y), K, n * K, n, K, _ptr(coef), moments, _ptr(off_t), nset,
                              _ptr(St), n, moments * K * n, self.stream)
                else:  # the reference takes any n_moments >= 1: 16 moments per launch
                    cf = coefs
                    for m0 in range(0, moments, _MOMENT_CHUNK):
                        mc = min(_MOMENT_CHUNK, moments - m0)
                        cpart = _h2d(np.ascontiguousarray(cf[:, m0:m0 + mc]))
                        _lib.call("cirr_moments", _ptr(Y), K, n * K, n, K, _ptr(cpart), mc, _ptr(off_t), nset,
                                  _ptr(St[:, m0 * K:]), n, moments * K * n, self.stream)
            del Y
        sh = _node_shard()
        if sh is not None:   # the one data-path exchange of the node split: sum the partial moment blocks
            with _stage("allreduce"):
                sh.allreduce(St, "sum")
        for s, ci in enumerate(active):
            self.cs[ci].stats.n_linear_solves += len(self.cs[ci].fidx) * ks[s]
        out, pieces, rows = {}, [], 0
        for s, ci in enumerate(active):
            kc = rhs[ci].shape[1]
            if kc == K:
                out[ci] = St[s]
            elif moments == 1:  # the zero rows of a narrower block are a suffix
                out[ci] = St[s, :kc]
            else:  # drop the zero rows inside each moment block: one gather for all
                for m in range(moments):
                    pieces.append(_piece(St[s, m * K:m * K + kc], rows + m * kc))
                out[ci] = (rows, moments * kc)
                rows += moments * kc
        if pieces:
            flat = torch.empty((rows, n), dtype=torch.complex128, device="cuda")
            _gather(pieces, flat)    # entry index = destination row (stride n)
            for ci, v in out.items():
                if isinstance(v, tuple):
                    out[ci] = flat[v[0]:v[0] + v[1]]
        return out

    def _dinv(self, K: int):
        """Inverses of the 128x128 diagonal blocks of every factor (each
        pencil's slice is contiguous), or None when an n x K solve does not read
        them.  Allocated and made on first use after the factorisation, so a
        wave whose solves never read them (small K on the left-looking kernel)
        never holds the buffer."""
        if not int(_lib.call("cirr_zgetrs_uses_dinv", self.n, K)):
            return None
        if self.dinv is None:
            self.dinv = self.torch.empty(self._dinv_per_pencil * self.P, dtype=self.torch.uint8, device="cuda")
            self._diag_inverses(0, self.P)
        return self.dinv

    def _oz_slices(self, K: int):
        """Digit slices of the factors for the int8 tensor-core trailing
        updates of the blocked solves (cirr_ozaki_split_factors): cut once
        after the factorisation, on the first solve wide enough to take the
        blocked path, when the int8 mode is on, the factors are dense, n is a
        multiple of 512 and the buffer (as large as the factors) fits."""
        if self.ozbuf is not None or K <= 16:
            return
        self.ozbuf = False
        n = self.n
        if not int(_lib.call("cirr_set_lu_gemm", -1)) or self.klL < n - 1 or self.kuU < n - 1:
            return
        nbytes = int(_lib.call("cirr_ozaki_factor_bytes", n, self.P))
        if nbytes == 0 or nbytes + (12 << 30) > _free_hbm():
            return
        with _stage("solve.ozsplit"):
            try:
                self.ozbuf = self.torch.empty(nbytes, dtype=self.torch.uint8, device="cuda")
            except self.torch.cuda.OutOfMemoryError:   # fragmented cache: the solves stay on FP64 DMMA
                self.ozbuf = False
                return
            _lib.call("cirr_ozaki_split_factors", _ptr(self.pencils), n, n, n * n, self.P, _ptr(self.ozbuf),
                      self.stream)

    def _bx(self, c, xi):
        """B X for the inside Ritz vectors: the product kept from the residual
        step when it belongs to this X, else computed."""
        bx = getattr(c, "bx_dev", None)
        c.bx_dev = None
        if bx is not None and bx.shape == xi.shape:
            return bx
        return self.bmul(xi, self.cs.index(c))

    def bmul(self, x, ci: int | None = None):
        """B @ x for a device (n x k) complex block (B of contour ci's pencil)."""
        d = self.dp if ci is None else self._dp_of(ci)
        torch, n = self.torch, self.n
        k = x.shape[1]
        if k > 1 and x.stride(1) != 1:
            x = x.contiguous()
        ldx = x.stride(0) if k > 1 else 1
        out = torch.empty((n, k), dtype=torch.complex128, device="cuda")
        if k:
            _lib.call("cirr_gemm", d.gemm_kind, n, k, n, 1, _ptr(d.b), n, 0, _ptr(x), ldx, 0, _ptr(out), k, 0,
                      1.0, 0, self.stream)
        return out

    def amul(self, x, ci: int | None = None):
        d = self.dp if ci is None else self._dp_of(ci)
        torch, n = self.torch, self.n
        k = x.shape[1]
        if k > 1 and x.stride(1) != 1:
            x = x.contiguous()
        ldx = x.stride(0) if k > 1 else 1
        out = torch.empty((n, k), dtype=torch.complex128, device="cuda")
        if k:
            _lib.call("cirr_gemm", d.gemm_kind, n, k, n, 1, _ptr(d.a), n, 0, _ptr(x), ldx, 0, _ptr(out), k, 0,
                      1.0, 0, self.stream)
        return out

    def source_blocks(self, active: list) -> dict:
        """B V for the seeded source blocks V = default_rng(seed).standard_normal
        ((n, L)).astype(complex) of every active contour (solvers.py:178-182):
        one upload and one batched GEMM when the contours share L."""
        torch, n = self.torch, self.n
        vs = {ci: _source_block(self.cs[ci].seed, n, self.cs[ci].ncols) for ci in active}
        widths = {v.shape[1] for v in vs.values()}
        if not self.multi or len(widths) != 1:
            return {ci: self.bmul(_h2d(vs[ci].astype(complex)), ci) for ci in active}
        k = widths.pop()
        # solve_multi's seeds (seed + i) repeat across the GEPs of a batch:
        # upload each distinct block once and expand on the device
        keys = {}
        for ci in active:
            keys.setdefault(id(vs[ci]), (len(keys), vs[ci]))
        if len(keys) < len(active) and k:
            U = _h2d(np.stack([v for _, v in keys.values()]).astype(complex))
            V = torch.empty((len(active), n, k), dtype=torch.complex128, device="cuda")
            _gather([_piece(U[keys[id(vs[ci])][0]], s) for s, ci in enumerate(active)], V)
        else:
            V = _h2d(np.stack([vs[ci] for ci in active]).astype(complex))
        _, B, stride = self._mats(active)
        out = torch.empty((len(active), n, k), dtype=torch.complex128, device="cuda")
        if k:
            self._gemm_mats(n, k, n, len(active), B, stride, V, k, n * k, out, k, n * k)
        return {ci: out[s] for s, ci in enumerate(active)}

    # -- K4..K7 for one contour --------------------------------------------
    def rayleigh_ritz(self, items: list, feast: bool = False, refine: bool = False) -> dict:
        return _drain(self.rayleigh_ritz_g(items, feast, refine))

    def rayleigh_ritz_g(self, items: list, feast: bool = False, refine: bool = False):
        """K4..K7 for several contours at once (solvers.py:187-198, batched).

        items: [(ci, St)] with St the transposed block of contour ci (its columns
        as rows).  CIRR: rank-truncated SVD basis (linalg.py:107-119); FEAST:
        Gram-Schmidt basis with drop_tol (linalg.py:79-104) and every Ritz vector
        returned (solvers.py:253).  Returns {ci: ("ok", lam_in, x_in_dev,
        res_in, x_all_or_None) | ("none", x_all_or_None) | ("rankzero",) |
        ("indefinite", exc)}."""
        with _stage("rr"):
            out = {}
            self._refine_src = None
            if feast:
                basis = self._basis_cgs2(items, out)
            else:
                basis = yield from self._basis_svd_g(items, out, try_cholqr=refine and _CHOLQR)
            if basis is None:
                return out
            items, Qt, ks = basis
            return (yield from self._rr_core_g(items, Qt, ks, out, all_vectors=feast))

    def _basis_cgs2(self, items: list, out: dict):
        torch, n, cfg, st = self.torch, self.n, self.cfg, self.stream
        for ci, S_ in items:
            if S_.shape[0] == 0:
                out[ci] = ("rankzero",)
        items = [(ci, S_) for ci, S_ in items if S_.shape[0] > 0]
        if not items:
            return None
        nb = len(items)
        cmax = max(S_.shape[0] for _, S_ in items)
        Y = _pad_stack([S_ for _, S_ in items], 0, cmax)
        Qt = _zeros((nb, cmax, n))
        kept = _zeros(nb, torch.int32)
        _lib.call("cirr_orthonormalize", _ptr(Y), n, cmax * n, n, cmax, nb, float(cfg.drop_tol), _ptr(Qt), n,
                  cmax * n, _ptr(kept), st)
        return self._live(items, Qt, kept.cpu().numpy(), out)

    def _live(self, items, Qt, ks, out):
        nb = len(items)
        live = [b for b in range(nb) if ks[b] > 0]
        for b in range(nb):
            if ks[b] == 0:
                out[items[b][0]] = ("rankzero",)
        if not live:
            return None
        kmax = int(ks[live].max())
        if len(live) < nb or kmax < Qt.shape[1]:
            out_q = self.torch.empty((len(live), kmax, Qt.shape[2]), dtype=Qt.dtype, device="cuda")
            Qt = _gather([_piece(Qt[b, :kmax], i) for i, b in enumerate(live)], out_q)
            ks = ks[live]
            items = [items[b] for b in live]
        return items, Qt, ks

    def _basis_svd_g(self, items: list, out: dict, try_cholqr: bool = False):
        torch, n, cfg, st = self.torch, self.n, self.cfg, self.stream
        for ci, S_ in items:
            if S_.shape[0] == 0:
                out[ci] = ("rankzero",)
        items = [(ci, S_) for ci, S_ in items if S_.shape[0] > 0]
        if not items:
            return None
        nb = len(items)
        cmax = max(S_.shape[0] for _, S_ in items)
        W = _pad_stack([S_ for _, S_ in items], 0, cmax)
        if try_cholqr and cmax <= n:
            # refinement blocks are normally far from rank deficient: when
            # ||R||_F ||R^-1||_F <= 1e5 certifies that no singular value is cut
            # (rank_rel_tol <= 1e-12), the CholeskyQR2 basis spans the same
            # space as the kept singular vectors (linalg.py:107-119)
            cdim = _h2d(np.array([S_.shape[0] for _, S_ in items], dtype=np.int32))
            Qt = _zeros((nb, cmax, n))
            ws = torch.empty(int(_lib.call("cirr_orth_cholqr2_ws_bytes", n, cmax, nb)), dtype=torch.uint8,
                             device="cuda")
            ok = _zeros(nb, torch.int32)
            with _stage("rr.orth"):
                _lib.call("cirr_orth_cholqr2", _ptr(W), n, cmax * n, n, cmax, nb, _ptr(cdim), _CHOLQR_KAPPA,
                          _ptr(Qt), n, cmax * n, _ptr(ws), _ptr(ok), st)
            if _DEBUG:
                sv = [torch.linalg.svdvals(S_.T).cpu().numpy() for _, S_ in items]
                print(f"[cirr] cholqr2 ok={ok.cpu().numpy().tolist()} kappa={[float(v[0] / v[-1]) for v in sv]}",
                      flush=True)
            yield
            if cfg.rank_rel_tol * _CHOLQR_KAPPA < 1.0 and bool(ok.cpu().numpy().all()):
                if _DEBUG:
                    print(f"[cirr] orth: c={cmax} nprob={nb} certified CholeskyQR2", flush=True)
                ks = np.array([S_.shape[0] for _, S_ in items], dtype=np.int64)
                # full rank: range(Q) = range(S), so Q^H S is an approximate
                # eigenbasis of the projected pencil (cirr_gen_eig_refine)
                self._refine_src = W
                return self._live(items, Qt, ks, out)
        # K4: one-sided Jacobi on all blocks (zero rows pad to cmax and are dropped)
        sigma = torch.empty((nb, cmax), dtype=torch.float64, device="cuda")
        order = torch.empty((nb, cmax), dtype=torch.int32, device="cuda")
        kept = torch.empty(nb, dtype=torch.int32, device="cuda")
        Qt = _zeros((nb, cmax, n))
        ws = torch.empty(int(_lib.call("cirr_orth_ws_bytes", cmax, nb)), dtype=torch.uint8, device="cuda")
        sweeps = _zeros(1, torch.int32)
        with _stage("rr.orth"):
            _lib.call("cirr_orth", _ptr(W), n, cmax * n, n, cmax, nb, float(cfg.rank_rel_tol), _ptr(sigma),
                      _ptr(order), _ptr(kept), _ptr(Qt), n, cmax * n, _ptr(ws), _ptr(sweeps), st)
        yield
        ks = kept.cpu().numpy()
        if _DEBUG:
            print(f"[cirr] orth: c={cmax} nprob={nb} kept={ks.tolist()} sweeps={int(sweeps.item())}", flush=True)
        return self._live(items, Qt, ks, out)

    def _rr_core_g(self, items, Qt, ks, out, all_vectors: bool):
        torch, n, cfg, st = self.torch, self.n, self.cfg, self.stream
        nb = len(items)
        kmax = int(ks.max())
        # K5: projected pencil  A~ = Q^H A Q, B~ = Q^H B Q
        with _stage("rr.project"):
            Q = torch.empty((nb, n, kmax), dtype=torch.complex128, device="cuda")
            _lib.call("cirr_transpose", 0, _ptr(Qt), n, kmax * n, kmax, n, nb, _ptr(Q), kmax, n * kmax, st)
            AQ = torch.empty((nb, n, kmax), dtype=torch.complex128, device="cuda")
            BQ = torch.empty_like(AQ)
            Am, Bm, mstride = self._mats([ci for ci, _ in items])
            self._gemm_mats(n, kmax, n, nb, Am, mstride, Q, kmax, n * kmax, AQ, kmax, n * kmax)
            self._gemm_mats(n, kmax, n, nb, Bm, mstride, Q, kmax, n * kmax, BQ, kmax, n * kmax)
            del Am, Bm
            At = torch.empty((nb, kmax, kmax), dtype=torch.complex128, device="cuda")
            Bt = torch.empty_like(At)
            kk = kmax * kmax
            _lib.call("cirr_gemm", 1, kmax, kmax, n, nb, _ptr(Qt), n, kmax * n, _ptr(AQ), kmax, n * kmax, _ptr(At), kmax,
                      kk, 1.0, 0, st)
            _lib.call("cirr_gemm", 1, kmax, kmax, n, nb, _ptr(Qt), n, kmax * n, _ptr(BQ), kmax, n * kmax, _ptr(Bt), kmax,
                      kk, 1.0, 0, st)
        # K6: small eigenproblems
        herm = self.dp.hermitian
        kdim = _h2d(ks.astype(np.int32))
        info = _zeros(nb, torch.int32)
        lam = _zeros((nb, kmax))
        Sv = None
        with _stage("rr.eigvals"):
            general_split = (not herm) and kmax <= 256 and not all_vectors
            if general_split and _EIG_REFINE and self._refine_src is not None:
                # refinement round: the block's own columns are near eigenvectors
                Sv = _zeros((nb, kmax, kmax))
                if (yield from self._refine_eig_g(self._refine_src, Q, At, Bt, kdim, kmax, nb, lam, Sv, info)):
                    general_split = False
                    for b, (ci, _) in enumerate(items):
                        self.cs[ci].prev_lam = lam[b, : int(ks[b])]
                else:
                    Sv = None
                    info = _zeros(nb, torch.int32)
            if general_split:
                # eigenvalues first; eigenvectors later only for the inside ones
                gws = torch.empty(int(_lib.call("cirr_gen_eig_ws_bytes", kmax, nb)), dtype=torch.uint8, device="cuda")
                # shift hints: the previous round's projected eigenvalues of each contour
                # (refinement rounds); same eigenvalues to rounding, ~20 % fewer QR sweeps
                prev = [getattr(self.cs[ci], "prev_lam", None) for ci, _ in items]
                if _QR_HINTS and all(p_ is not None for p_ in prev):
                    hld = max(max(int(p_.shape[0]) for p_ in prev), 1)
                    hint = _pad_stack([p_[None, :] for p_ in prev], 1, hld).view(nb, hld)
                    hcnt = _h2d(np.array([min(int(p_.shape[0]), 256) for p_ in prev], dtype=np.int32))
                    _lib.call("cirr_gen_eig_values_hinted", _ptr(At), _ptr(Bt), _ptr(kdim), kmax, nb, _ptr(gws),
                              _ptr(lam), _ptr(info), _ptr(hint), _ptr(hcnt), hld, st)
                else:
                    _lib.call("cirr_gen_eig_values", _ptr(At), _ptr(Bt), _ptr(kdim), kmax, nb, _ptr(gws), _ptr(lam),
                              _ptr(info), st)
                for b, (ci, _) in enumerate(items):
                    self.cs[ci].prev_lam = lam[b, : int(ks[b])]   # a view: lam is this round's own buffer
            elif Sv is None:
                wsb = int(_lib.call("cirr_small_eig_ws_bytes", kmax))
                ews = torch.empty(nb * ((wsb + 255) // 256 * 256), dtype=torch.uint8, device="cuda")
                Sv = _zeros((nb, kmax, kmax))
                _lib.call("cirr_small_eig", 1 if herm else 0, _ptr(At), _ptr(Bt), kmax, kk, _ptr(kdim), kmax, nb,
                          _ptr(ews), _ptr(lam), _ptr(Sv), kmax, kk, _ptr(info), st)
        yield
        infos = info.cpu().numpy()
        lam_h = lam.cpu().numpy()
        # solvers.py:161-162 for every contour of the round in one pass
        inside = contains_rows([self.cs[ci].contour for ci, _ in items], lam_h.real + 0j if herm else lam_h, ks)
        inside[infos != 0] = False
        n_in = inside.sum(axis=1)
        order = np.argsort(~inside, axis=1, kind="stable")   # inside columns first, in index order
        keep_idx = {}
        for b, (ci, _) in enumerate(items):
            if infos[b] > 0:
                msg = "projected B is not positive definite" if herm else "projected B is singular"
                out[ci] = ("indefinite", IndefiniteBError(msg))
            elif infos[b] < 0:
                # this contour's projected QR did not converge: a per-contour
                # ConvergenceError (isolated by solve_multi), not a process error
                out[ci] = ("qrfail", None)
            elif n_in[b] == 0:
                out[ci] = ("none", None)
            else:
                keep_idx[b] = order[b, : n_in[b]]
        X = None
        if all_vectors:
            X = torch.empty((nb, n, kmax), dtype=torch.complex128, device="cuda")
            _lib.call("cirr_gemm", 0, n, kmax, kmax, nb, _ptr(Q), kmax, n * kmax, _ptr(Sv), kmax, kk, _ptr(X), kmax,
                      n * kmax, 1.0, 0, st)
            for b, (ci, _) in enumerate(items):
                if ci in out and out[ci][0] == "none":
                    out[ci] = ("none", X[b, :, : ks[b]])
        if not keep_idx:
            return out
        # K7: X = Q s for the inside columns, A X, B X, residuals
        kin_max = int(n_in.max())
        cnt = np.where(np.isin(np.arange(nb), list(keep_idx)), n_in, 0).astype(np.int32)
        valid = np.arange(kin_max)[None, :] < cnt[:, None]
        idx = np.where(valid, order[:, :kin_max], 0).astype(np.int32)
        lam_in = np.where(valid, np.take_along_axis(lam_h, idx, axis=1), 0)
        idx_t = _h2d(idx)
        cnt_t = _h2d(cnt)
        Xi = _zeros((nb, n, kin_max))
        Sin = _zeros((nb, kmax, kin_max))
        if general_split:
            scr = torch.empty(int(_lib.call("cirr_gen_eig_vec_scratch_bytes", kmax, nb, kin_max)), dtype=torch.uint8,
                              device="cuda")
            _lib.call("cirr_gen_eig_vectors", _ptr(gws), _ptr(kdim), kmax, nb, _ptr(lam), _ptr(idx_t), _ptr(cnt_t),
                      kin_max, _ptr(scr), _ptr(Sin), kin_max, kmax * kin_max, st)
        else:  # the inside columns of the projected eigenvectors
            _lib.call("cirr_gather_cols", _ptr(Sv), kmax, kk, _ptr(idx_t), kin_max, _ptr(cnt_t), kin_max, kmax, nb,
                      _ptr(Sin), kin_max, kmax * kin_max, st)
        _lib.call("cirr_gemm", 0, n, kin_max, kmax, nb, _ptr(Q), kmax, n * kmax, _ptr(Sin), kin_max,
                  kmax * kin_max, _ptr(Xi), kin_max, n * kin_max, 1.0, 0, st)
        # A X = (A Q) s and B X = (B Q) s from the projection products: n x k x k_in
        # instead of n x n x k_in (solvers.py:142-143 computes A X, B X directly;
        # the two agree to rounding)
        AX = torch.empty_like(Xi)
        BX = torch.empty_like(Xi)
        _lib.call("cirr_gemm", 0, n, kin_max, kmax, nb, _ptr(AQ), kmax, n * kmax, _ptr(Sin), kin_max,
                  kmax * kin_max, _ptr(AX), kin_max, n * kin_max, 1.0, 0, st)
        _lib.call("cirr_gemm", 0, n, kin_max, kmax, nb, _ptr(BQ), kmax, n * kmax, _ptr(Sin), kin_max,
                  kmax * kin_max, _ptr(BX), kin_max, n * kin_max, 1.0, 0, st)
        lam_t = _h2d(lam_in)
        res = _zeros((nb, kin_max), torch.float64)
        _lib.call("cirr_residuals", _ptr(AX), _ptr(BX), kin_max, n * kin_max, n, _ptr(lam_t), kin_max, _ptr(cnt_t),
                  kin_max, nb, _ptr(res), kin_max, st)
        yield
        res_h = res.cpu().numpy()
        for b, ix in keep_idx.items():
            ci = items[b][0]
            k_in = len(ix)
            lam_b = lam_h[b, ix]
            if herm:
                lam_b = lam_b.real.copy()
            xall = X[b, :, : ks[b]] if all_vectors else None
            # views into the round's blocks (consumers copy or read them; bmul
            # makes a contiguous copy where a raw pointer is needed)
            out[ci] = ("ok", lam_b, _Cols(Xi, b, k_in), res_h[b, :k_in].copy(), xall)
            self.cs[ci].bx_dev = _Cols(BX, b, k_in)   # B X, the next refinement's right-hand side
        return out

    def _refine_eig_g(self, S_st, Q, At, Bt, kdim, kmax: int, nb: int, lam, Sv, info):
        """K6 for a refinement round: eigenpairs of (A~, B~) by Newton refinement
        of W0 = Q^H S (cirr_gen_eig_refine).  S_st: the certified block (nb x
        kmax x n, the columns of S as rows).  Returns False when any problem did
        not converge (the caller then runs the QR path for the round)."""
        torch, n, st = self.torch, self.n, self.stream
        kk = kmax * kmax
        W0h = torch.empty((nb, kmax, kmax), dtype=torch.complex128, device="cuda")
        # S^H Q = conj(S^T) Q: the rows of S_st conjugated times Q (n x kmax)
        _lib.call("cirr_gemm", 1, kmax, kmax, n, nb, _ptr(S_st), n, kmax * n, _ptr(Q), kmax, n * kmax, _ptr(W0h),
                  kmax, kk, 1.0, 0, st)
        ws = torch.empty(int(_lib.call("cirr_gen_eig_refine_ws_bytes", kmax, nb)), dtype=torch.uint8, device="cuda")
        _lib.call("cirr_gen_eig_refine", _ptr(At), _ptr(Bt), _ptr(kdim), kmax, nb, _ptr(W0h), kmax, kk,
                  _EIG_REFINE_ITERS, _ptr(ws), _ptr(lam), _ptr(Sv), kmax, kk, _ptr(info), st)
        yield
        inf = info.cpu().numpy()
        if _DEBUG:
            import ctypes
            stats = (ctypes.c_int * 16)()
            _lib.call("cirr_gen_eig_refine_stats", ctypes.addressof(stats))
            print(f"[cirr] eig refine k={kmax} nprob={nb} info={inf.tolist()} converged at step "
                  f"{list(stats[:min(nb, 8)])} block columns {list(stats[8:8 + min(nb, 8)])}", flush=True)
        return not bool((inf < 0).any())

    # -- the reference control flow (solvers.py:165-227) for all contours ----
    def run(self, moments: int):
        return _drain(self.run_g(moments))

    def solve_g(self, moments: int):
        """factor + run as one generator (the interleaved batch path)."""
        yield from self.factor_g(sources=True)
        yield from self.run_g(moments)

    def run_g(self, moments: int):
        torch, cfg, n = self.torch, self.cfg, self.n
        active = [i for i, c in enumerate(self.cs) if not c.done]
        if not active:
            return
        src = getattr(self, "_src", None)
        self._src = None
        rhs = {ci: src[ci] for ci in active} if src is not None else self.source_blocks(active)  # solvers.py:178-182
        stacked = self.apply(active, rhs, moments, real_rhs=True)
        it_of = {ci: 0 for ci in active}
        for it in range(cfg.max_refine):
            refine = {}
            for ci in active:
                it_of[ci] = it
            rr = yield from self.rayleigh_ritz_g([(ci, stacked[ci]) for ci in active], refine=it > 0)
            for ci in list(active):
                c = self.cs[ci]
                r = rr[ci]
                if r[0] == "rankzero":
                    active.remove(ci)
                    continue
                if r[0] == "indefinite":
                    c.error = r[1]
                    c.fatal = True
                    active.remove(ci)
                    continue
                if r[0] == "qrfail":
                    c.error = ConvergenceError(c.best_res)
                    c.fatal = True
                    active.remove(ci)
                    continue
                if r[0] == "none":
                    c.lam = None
                    active.remove(ci)
                    continue
                _, lam, xi, res, _ = r
                c.lam, c.x_dev, c.res = lam, xi, res
                rmax = float(res.max())
                c.rmax = rmax
                c.best_res = min(c.best_res, rmax)
                if _DEBUG:
                    print(f"[cirr] contour {ci} it {it}: inside {len(lam)} max res {rmax:.2e}", flush=True)
                if rmax <= cfg.tol or it + 1 >= cfg.max_refine or (
                        cfg.early_exit and c.settled(lam, res, cfg.tol)):
                    active.remove(ci)
                    continue
                refine[ci] = self._bx(c, xi)
            if not refine:
                break
            stacked = self.apply(list(refine.keys()), refine, 1)
            active = list(refine.keys())
        yield from self.fetch_vectors_g()
        for ci, c in enumerate(self.cs):
            if c.done:
                continue
            c.stats.iterations = it_of.get(ci, 0) + 1
            c.stats.elapsed = time.perf_counter() - c.t0
            if getattr(c, "fatal", False):
                continue
            self.finish(c)

    # -- FEAST (solvers.py:230-285) on the same resident factors -------------
    def run_feast(self):
        torch, cfg, n = self.torch, self.cfg, self.n
        active = [i for i, c in enumerate(self.cs) if not c.done]
        u = {}
        for ci in active:
            c = self.cs[ci]
            rng = np.random.default_rng(c.seed)
            u[ci] = torch.from_numpy(rng.standard_normal((n, c.ncols)).astype(complex)).to("cuda")  # 238-240
            c.found_any = False
        it_of = {ci: 0 for ci in active}
        for it in range(cfg.max_refine):
            if not active:
                break
            for ci in active:
                it_of[ci] = it
            stacked = self.apply(active, {ci: self.bmul(u[ci], ci) for ci in active}, 1)  # y = P u (246)
            rr = self.rayleigh_ritz([(ci, stacked[ci]) for ci in active], feast=True)
            nxt = []
            for ci in active:
                c = self.cs[ci]
                r = rr[ci]
                if r[0] == "rankzero":  # 249-250
                    continue
                if r[0] == "indefinite":
                    c.error, c.fatal = r[1], True
                    continue
                if r[0] == "qrfail":
                    c.error, c.fatal = ConvergenceError(c.best_res), True
                    continue
                if r[0] == "none":  # 253-255: u = xs, keep iterating
                    if r[1] is not None:
                        u[ci] = r[1]
                    nxt.append(ci)
                    continue
                _, lam, xi, res, xall = r
                u[ci] = xall
                c.found_any = True
                c.lam, c.x_dev, c.res = lam, xi, res
                c.best_res = min(c.best_res, float(res.max()))
                if res.max() <= cfg.tol:  # 260-261
                    continue
                nxt.append(ci)
            active = nxt
        for ci, c in enumerate(self.cs):
            if c.done:
                continue
            c.stats.iterations = it_of.get(ci, 0) + 1
            c.stats.elapsed = time.perf_counter() - c.t0
            if getattr(c, "fatal", False):
                continue
            if not getattr(c, "found_any", False):
                c.lam = None
            self.finish(c)

    def finish(self, c: _Contour):
        cfg = self.cfg
        if c.lam is None or c.lam.size == 0:  # solvers.py:211-214
            c.error = NoEigenvaluesFound(
                f"no eigenvalues inside contour (expected {getattr(c.contour, 'expected_count', 0)})")
            return
        lam, res = c.lam, c.res
        x = c.__dict__.pop("x_host", None)
        if x is None:
            x = c.x_dev.cpu().numpy()
        rmax = getattr(c, "rmax", None)
        if (float(res.max()) if rmax is None else rmax) > cfg.tol:  # solvers.py:215-219
            conv = res <= cfg.tol
            if not np.any(conv):
                c.error = ConvergenceError(c.best_res)
                return
            lam, x, res = lam[conv], x[:, conv], res[conv]
        order = np.argsort(lam)  # solvers.py:220
        if lam.size < 2 or not np.any(order[1:] < order[:-1]):
            # already in order (the Hermitian eigenvalues come back ascending):
            # the same arrays without three fancy-index copies
            c.result = EigenResult(eigenvalues=lam, eigenvectors=x, residuals=res, contour=c.contour,
                                   stats=c.stats)
            return
        c.result = EigenResult(eigenvalues=lam[order], eigenvectors=x[:, order], residuals=res[order],
                               contour=c.contour, stats=c.stats)

    def fetch_vectors(self):
        return _drain(self.fetch_vectors_g())

    def fetch_vectors_g(self):
        """Every finishing contour's Ritz vectors packed by one gather launch
        and read back with one device-to-host copy (not one per contour)."""
        torch = self.torch
        cs = [c for c in self.cs if not c.done and not getattr(c, "fatal", False)
              and c.lam is not None and getattr(c, "x_dev", None) is not None and c.x_dev.numel()]
        if len(cs) < 2:
            return
        pieces, off = [], 0
        for c in cs:
            r, k = c.x_dev.shape
            pieces.append(_piece(c.x_dev, off, dst_ld=k))   # 1-D destination: entry = element offset
            c._x_off = off
            off += r * k
        flat = torch.empty((off, 1), dtype=torch.complex128, device="cuda")
        _gather(pieces, flat)
        host = torch.empty(off, dtype=torch.complex128, pin_memory=True)
        host.copy_(flat.view(-1), non_blocking=True)
        yield
        torch.cuda.current_stream().synchronize()
        h = host.numpy()
        for c in cs:
            r, k = c.x_dev.shape
            c.x_host = h[c._x_off:c._x_off + r * k].reshape(r, k)

    def free(self):
        if getattr(self, "ozbuf", None) is not None and self.ozbuf is not False and hasattr(self, "pencils"):
            _lib.call("cirr_ozaki_release", _ptr(self.pencils))
        for name in ("pencils", "maxabs", "ipiv", "perm", "minpiv", "info", "dinv", "ozbuf"):
            if hasattr(self, name):
                delattr(self, name)


def _waves(cstates: list, n: int, budget_bytes: int) -> list:
    """Group contours (whole) into waves whose factors fit the HBM budget and
    whose pencil count stays within the launch grid limit (_MAX_WAVE_PENCILS).
    Per factored node: the n x n complex128 factor, its diagonal-block
    inverses (made when a solve reads them) and the LU workspace share."""
    per = n * n * 16 + int(_lib.call("cirr_diag_inv_bytes", n, 1)) + int(_lib.call("cirr_zgetrf_ws_bytes", n, 1))
    waves, cur, cur_bytes, cur_p = [], [], 0, 0
    sh = _node_shard()
    for c in cstates:
        p = len(c.fidx) if sh is None else -(-len(c.all_nodes) // sh.world)
        if p > _MAX_WAVE_PENCILS:
            raise ParameterError(f"n_q = {p} factored nodes per contour exceeds {_MAX_WAVE_PENCILS}")
        need = p * per
        if cur and (cur_bytes + need > budget_bytes or cur_p + p > _MAX_WAVE_PENCILS):
            waves.append(cur)
            cur, cur_bytes, cur_p = [], 0, 0
        cur.append(c)
        cur_bytes += need
        cur_p += p
    if cur:
        waves.append(cur)
    return waves


_FOREIGN_BYTES = {}


def _free_hbm() -> int:
    """Free device memory for this process's buffers: the device total minus
    what other users held at the first call (CUDA context, other processes)
    minus what torch has allocated now.  cudaMemGetInfo runs once per device:
    it took up to ~50 ms per call on the B200 boxes (a config-2 solve is
    ~100 ms), and it also misses the blocks torch's allocator has cached."""
    torch = _torch()
    dev = torch.cuda.current_device()
    if dev not in _FOREIGN_BYTES:
        free, total = torch.cuda.mem_get_info()
        _FOREIGN_BYTES[dev] = (total, max(total - free - torch.cuda.memory_reserved(dev), 0))
    total, foreign = _FOREIGN_BYTES[dev]
    return total - foreign - torch.cuda.memory_allocated(dev)


def _hbm_budget(n: int, cstates: list) -> int:
    free = _free_hbm()
    kmax = max([c.ncols for c in cstates] + [1])
    nodes = sum(len(c.nodes) for c in cstates)
    reserve = 4 << 30
    reserve += nodes * n * kmax * 16 * 8  # solve/moment/refinement blocks
    return max(int(free - reserve), n * n * 16 * 64)


def _run_contours(pencil, contours, cfg, seeds, moments_override=None, solver: str = "cirr"):
    cfg = _cfg_view(cfg)
    dp = DevicePencil.of(pencil)
    cstates = [_Contour(i, c, cfg, s, dp.n, dp.complex) for i, (c, s) in enumerate(zip(contours, seeds))]
    _run_states(dp, cstates, cfg, moments_override, solver)
    return cstates


_STREAMS: dict = {}


def _interleave(engines, moments: int) -> None:
    """Run the engines' solve generators round-robin, each on its own stream:
    while the host does one engine's read-back and bookkeeping, the GPU works
    through the kernels the other engines have queued (a large batch such as
    config 2's 512 contours is otherwise host-bound between its syncs)."""
    torch = _torch()
    cur = torch.cuda.current_stream()
    # the same streams every call: torch's caching allocator keeps blocks per
    # stream, so fresh streams would cudaMalloc the whole wave again
    pool = _STREAMS.setdefault(torch.cuda.current_device(), [])
    while len(pool) < len(engines):
        pool.append(torch.cuda.Stream())
    streams = pool[:len(engines)]
    live = []
    for eng, st in zip(engines, streams):
        st.wait_stream(cur)          # inputs uploaded on the caller's stream
        live.append((eng.solve_g(moments), st))
    try:
        while live:
            nxt = []
            for gen, st in live:
                with torch.cuda.stream(st):
                    try:
                        next(gen)
                        nxt.append((gen, st))
                    except StopIteration:
                        pass
            live = nxt
    finally:
        for st in streams:
            cur.wait_stream(st)
    for eng in engines:
        eng.free()


def _interleave_split(wave: list) -> list:
    """How many engines a wave is split into for _interleave (contiguous runs
    of contours, so each engine's pencils stay adjacent)."""
    k = _INTERLEAVE if len(wave) >= _INTERLEAVE_MIN else 1
    if k <= 1:
        return [wave]
    step = -(-len(wave) // k)
    return [wave[i:i + step] for i in range(0, len(wave), step)]


def _run_states(dp, cstates, cfg, moments_override=None, solver: str = "cirr"):
    arith = getattr(cfg, "arith", None)
    if arith is None:
        return _run_states_mode(dp, cstates, cfg, moments_override, solver)
    prev = int(_lib.call("cirr_set_lu_gemm", 1 if arith == "int8" else 0))   # library-wide while this call runs
    try:
        return _run_states_mode(dp, cstates, cfg, moments_override, solver)
    finally:
        _lib.call("cirr_set_lu_gemm", prev)


def _run_states_mode(dp, cstates, cfg, moments_override=None, solver: str = "cirr"):
    moments = cfg.n_moments if moments_override is None else moments_override
    budget = _hbm_budget(dp.n, cstates)
    sh = _node_shard()
    if sh is not None:   # the ranks must cut the same waves: the smallest budget, the largest node share
        bt = _h2d(np.asarray([budget], dtype=np.int64))
        sh.allreduce(bt, "min")
        budget = int(bt.cpu().numpy()[0])
    for wave in _waves(cstates, dp.n, budget):
        parts = _interleave_split(wave) if solver == "cirr" else [wave]
        if len(parts) > 1:
            _interleave([_Engine(dp, part, cfg) for part in parts], moments)
            continue
        eng = _Engine(dp, wave, cfg)
        if solver == "feast":
            eng.factor()
            eng.run_feast()
        else:
            eng.factor(sources=True)
            eng.run(moments)
        eng.free()
        del eng


# ---------------------------------------------------------------------------
# public entry points


def cirr_solve(pencil, contour, cfg: SolverConfig | None = None, seed: int = 0) -> EigenResult:
    """Moment-based contour-integral Rayleigh-Ritz solve (solvers.py:165-227)."""
    c = _run_contours(pencil, [contour], cfg, [seed])[0]
    if c.error is not None:
        raise c.error
    return c.result


def feast_solve(pencil, contour, cfg: SolverConfig | None = None, seed: int = 0) -> EigenResult:
    """Filtered subspace iteration on the device factors (solvers.py:230-285):
    U <- orthonormalize(P U), Rayleigh-Ritz after each projector application."""
    c = _run_contours(pencil, [contour], cfg, [seed], solver="feast")[0]
    if c.error is not None:
        raise c.error
    return c.result


def solve_multi(pencil, contours, cfg: SolverConfig | None = None, solver: str = "cirr",
                seed: int = 0) -> MultiResult:
    """Every contour solved in one batched device pass (solvers.py:312-339);
    per-contour failures are isolated, IndefiniteBError/DimensionError
    propagate, duplicates across contours keep the smaller residual."""
    if solver not in ("cirr", "feast"):
        raise ParameterError(f"unknown solver {solver!r}")
    t0 = time.perf_counter()
    contours = list(contours)
    cstates = _run_contours(pencil, contours, cfg, [seed + i for i in range(len(contours))], solver=solver)
    return _multi_result(cstates, t0)


def _multi_result(cstates, t0) -> MultiResult:
    """solve_multi's aggregation (solvers.py:325-339) over one pencil's contours."""
    results, errors = [], []
    agg = SolveStats()
    for c in cstates:
        if c.error is not None and not isinstance(
                c.error, (NoEigenvaluesFound, ConvergenceError, SingularShiftError, RankZeroError)):
            raise c.error
        if c.result is not None:
            results.append(c.result)
            errors.append(None)
            agg.n_linear_solves += c.stats.n_linear_solves
            agg.n_factorizations += c.stats.n_factorizations
            agg.iterations += c.stats.iterations
        else:
            results.append(None)
            errors.append(c.error)
    _dedupe(results)
    agg.elapsed = time.perf_counter() - t0
    return MultiResult(results=results, errors=errors, stats=agg)


def solve_multi_batch(pencils, contours, cfg: SolverConfig | None = None, solver: str = "cirr",
                      seeds=None) -> list:
    """``[solve_multi(p, cs, cfg, solver, seed=s) for p, cs, s in ...]`` for
    many independent pencils of one size in one batched device pass: the
    DeepContour dataset regime (BASELINE config 2, 256 GEPs of n=256).  The
    reference solves such a batch one ``solve_multi`` call at a time
    (bench.py:144); here every pencil x contour x node of a wave shares one
    batched LU, one batched solve per pass and one batched Rayleigh-Ritz round.

    ``contours`` is one contour list per pencil (or one list for all);
    ``seeds`` one seed per pencil (default 0, solve_multi's default), contour i
    of a pencil using seed + i as solve_multi does.  Pencils whose dtype or
    Hermitian flag differ run in separate batches.  Per-pencil errors follow
    solve_multi: the four isolated types land in ``MultiResult.errors``, any
    other error propagates."""
    if solver not in ("cirr", "feast"):
        raise ParameterError(f"unknown solver {solver!r}")
    t0 = time.perf_counter()
    cfg = _cfg_view(cfg)
    pencils = list(pencils)
    if not pencils:
        return []
    contours = list(contours)
    if contours and not isinstance(contours[0], (list, tuple)):
        contours = [contours] * len(pencils)
    if len(contours) != len(pencils):
        raise DimensionError("need one contour list per pencil")
    seeds = [0] * len(pencils) if seeds is None else [int(x) for x in seeds]
    if len(seeds) != len(pencils):
        raise DimensionError("need one seed per pencil")
    dps = DevicePencil.of_many(pencils)
    n = dps[0].n
    if any(d.n != n for d in dps):
        raise DimensionError("solve_multi_batch needs pencils of one size")
    per = []
    for g, (d, cs, sd) in enumerate(zip(dps, contours, seeds)):
        st = [_Contour(i, c, cfg, sd + i, n, d.complex) for i, c in enumerate(cs)]
        for c in st:
            c.dp = d
        per.append(st)
    groups: dict = {}
    for g, d in enumerate(dps):
        groups.setdefault((d.complex, d.hermitian), []).append(g)
    for gs in groups.values():
        _run_states(dps[gs[0]], [c for g in gs for c in per[g]], cfg, None, solver)
    return [_multi_result(st, t0) for st in per]


def _dedupe_complex_drops(vals_list) -> dict:
    """Complex eigenvalues (non-Hermitian pencils): a 1-D sort does not put
    near-equal complex values next to each other (conjugate pairs found by two
    overlapping contours share a real part to rounding), so match by distance.
    Candidates are visited by ascending residual (ties in input order); one is
    dropped when a value already kept from a DIFFERENT contour lies within
    1e-8 of the span, so each duplicate cluster keeps its smallest residual,
    as the reference's rule does for real values (solvers.py:342-377)."""
    vals = np.array([v[0] for v in vals_list])
    span = float(np.abs(vals[:, None] - vals[None, :]).max())
    tol = 1e-8 * max(span, 1e-300)
    order = sorted(range(len(vals_list)), key=lambda t: (vals_list[t][1], t))
    kept: list = []
    drop: dict = {}
    for idx in order:
        v, ri = vals_list[idx][0], vals_list[idx][2]
        if any(vals_list[k][2] != ri and abs(v - vals_list[k][0]) <= tol for k in kept):
            drop.setdefault(ri, set()).add(vals_list[idx][3])
        else:
            kept.append(idx)
    return drop


def _dedupe(results) -> None:
    """solvers.py:342-377 (span uses |.| so complex eigenvalues work)."""
    all_vals = [(r.eigenvalues[i], r.residuals[i], ri, i) for ri, r in enumerate(results) if r is not None
                for i in range(len(r.eigenvalues))]
    if len(all_vals) < 2:
        return
    vals = np.array([v[0] for v in all_vals])
    if np.iscomplexobj(vals) and np.any(vals.imag != 0):
        drop = _dedupe_complex_drops(all_vals)
    else:
        span = abs(vals.max() - vals.min())
        tol = 1e-8 * max(span, 1e-300)
        order = np.argsort(vals)
        drop: dict = {}
        prev = order[0]
        for idx in order[1:]:
            if abs(all_vals[idx][0] - all_vals[prev][0]) <= tol and all_vals[idx][2] != all_vals[prev][2]:
                loser = idx if all_vals[idx][1] >= all_vals[prev][1] else prev
                winner = idx if loser is prev else prev
                drop.setdefault(all_vals[loser][2], set()).add(all_vals[loser][3])
                prev = winner
            else:
                prev = idx
    for ri, cols in drop.items():
        r = results[ri]
        keep = np.array([i not in cols for i in range(len(r.eigenvalues))])
        results[ri] = EigenResult(eigenvalues=r.eigenvalues[keep], eigenvectors=r.eigenvectors[:, keep],
                                  residuals=r.residuals[keep], contour=r.contour, stats=r.stats)


class ProjectorContext:
    """One device factorisation per quadrature node (solvers.py:97-130).

    ``apply(block, moments)`` returns [S_0 .. S_{M-1}] with S_m = sum_j w_j
    z_j^m Y_j (raw powers, exactly the reference's definition); ``frame`` =
    (gamma, rho) switches to the centred moments the CIRR path uses.
    """

    def __init__(self, pencil, rule: QuadratureRule, frame=None):
        self._dp = DevicePencil.of(pencil)
        self.pencil = pencil
        self.rule = rule
        self._c = _Contour.__new__(_Contour)
        self._c.nodes = np.asarray(rule.nodes, dtype=np.complex128)
        self._c.weights = np.asarray(rule.weights, dtype=np.complex128)
        self._c.gamma, self._c.rho = frame if frame is not None else (0j, 1.0)
        self._c.stats = SolveStats()
        self._c.error = None
        self._c.done = False
        self._c.half = False
        self._c.fidx = np.arange(len(self._c.nodes))
        self._eng = _Engine(self._dp, [self._c], SolverConfig())
        self._eng.factor()
        if self._c.error is not None:
            raise self._c.error
        self.n_factorizations = len(self._c.nodes)
        self.n_linear_solves = 0

    def apply(self, block, moments: int = 1) -> list:
        torch = _torch()
        v = _as_block(block)
        if v.shape[0] != self._dp.n:
            raise DimensionError("block rows must match pencil dimension")
        k = v.shape[1]
        if k == 0:
            return [np.zeros_like(v) for _ in range(moments)]
        bv = self._eng.bmul(torch.from_numpy(np.ascontiguousarray(v)).to("cuda"))
        before = self._c.stats.n_linear_solves
        St = self._eng.apply([0], {0: bv}, moments)[0]
        self.n_linear_solves += self._c.stats.n_linear_solves - before
        st = St.cpu().numpy()  # (moments*k) x n
        return [st[m * k:(m + 1) * k].T.copy() for m in range(moments)]


def apply_projector(pencil, rule: QuadratureRule, v) -> np.ndarray:
    """Quadrature approximation of the spectral projector applied to v (solvers.py:133-137)."""
    ctx = ProjectorContext(pencil, rule)
    return ctx.apply(_as_block(v), moments=1)[0]
