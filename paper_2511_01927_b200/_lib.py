"""ctypes binding of libcirr.so (the C ABI declared in include/cirr.h).

There is no CPU fallback: if the shared library is missing or CUDA is not
available, every entry point raises ``DeviceError``.  Pointers are raw device
addresses of PyTorch tensors; the stream is torch's current CUDA stream.
"""

from __future__ import annotations

import ctypes
import os

from .errors import DeviceError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CIRR_LIB") or os.path.join(_HERE, "libcirr.so")  # CIRR_LIB: A/B builds (dev)
EINVAL = 100000

_P = ctypes.c_void_p
_I = ctypes.c_int
_L = ctypes.c_longlong
_D = ctypes.c_double

# name -> argtypes (all return int unless listed in _RESTYPE)
SIGNATURES = {
    "cirr_assemble": [_P, _P, _I, _L, _P, _I, _P, _L, _L, _P, _P],
    "cirr_symmetry": [_P, _I, _L, _P, _P],
    "cirr_assemble_c": [_P, _P, _I, _L, _P, _I, _P, _L, _L, _P, _P],
    "cirr_assemble_ptrs": [_P, _P, _I, _L, _P, _I, _P, _L, _L, _P, _P],
    "cirr_hermitian_c": [_P, _I, _L, _P, _P],
    "cirr_zgetrf_batched": [_P, _I, _L, _L, _I, _P, _P, _P, _P, _P, _P],
    "cirr_zgetrf_ws_bytes": [_I, _I],
    "cirr_zgetrf_band": [_P, _I, _L, _L, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P],
    "cirr_bandwidth": [_P, _I, _I, _L, _P, _P],
    "cirr_bandwidth_ptrs": [_P, _I, _I, _I, _L, _P, _P],
    "cirr_zgetrs_band": [_P, _I, _L, _L, _I, _P, _I, _P, _P, _L, _L, _P, _I, _P, _L, _L, _P, _P, _I, _P, _I, _P,
                         _L, _L, _I, _I, _P],
    "cirr_zgetrs_batched": [_P, _I, _L, _L, _I, _P, _P, _L, _L, _P, _I, _P, _L, _L, _P, _P],
    "cirr_zgetrs_gather": [_P, _I, _L, _L, _I, _P, _I, _P, _P, _L, _L, _P, _I, _P, _L, _L, _P, _P],
    "cirr_diag_inv_bytes": [_I, _I],
    "cirr_diag_inverses": [_P, _I, _L, _L, _I, _P, _P],
    "cirr_zgetrs_uses_dinv": [_I, _I],
    "cirr_moments": [_P, _L, _L, _I, _I, _P, _I, _P, _I, _P, _L, _L, _P],
    "cirr_zgetrs_moments": [_P, _I, _L, _L, _I, _P, _I, _P, _P, _L, _L, _P, _I, _P, _L, _L, _P, _P, _I, _P, _I, _P,
                            _L, _L, _P],
    "cirr_orth_ws_bytes": [_I, _I],
    "cirr_orth_phases": [_P],
    "cirr_orth": [_P, _L, _L, _I, _I, _I, _D, _P, _P, _P, _P, _L, _L, _P, _P, _P],
    "cirr_orthonormalize": [_P, _L, _L, _I, _I, _I, _D, _P, _L, _L, _P, _P],
    "cirr_orth_cholqr2_ws_bytes": [_I, _I, _I],
    "cirr_orth_cholqr2": [_P, _L, _L, _I, _I, _I, _P, _D, _P, _L, _L, _P, _P, _P],
    "cirr_gemm": [_I, _I, _I, _I, _I, _P, _L, _L, _P, _L, _L, _P, _L, _L, _D, _I, _P],
    "cirr_small_eig_ws_bytes": [_I],
    "cirr_small_eig": [_I, _P, _P, _L, _L, _P, _I, _I, _P, _P, _P, _L, _L, _P, _P],
    "cirr_small_eig_phases": [_P],
    "cirr_gen_eig_qr_stats": [_P],
    "cirr_gen_eig_ws_bytes": [_I, _I],
    "cirr_gen_eig_vec_scratch_bytes": [_I, _I, _I],
    "cirr_gen_eig_values": [_P, _P, _P, _I, _I, _P, _P, _P, _P],
    "cirr_gen_eig_values_hinted": [_P, _P, _P, _I, _I, _P, _P, _P, _P, _P, _I, _P],
    "cirr_gen_eig_vectors": [_P, _P, _I, _I, _P, _P, _P, _I, _P, _P, _L, _L, _P],
    "cirr_gen_eig_refine_ws_bytes": [_I, _I],
    "cirr_gen_eig_refine_stats": [_P],
    "cirr_gen_eig_refine": [_P, _P, _P, _I, _I, _P, _L, _L, _I, _P, _P, _P, _L, _L, _P, _P],
    "cirr_residuals": [_P, _P, _L, _L, _I, _P, _L, _P, _I, _I, _P, _L, _P],
    "cirr_gather_cols": [_P, _L, _L, _P, _L, _P, _I, _I, _I, _P, _L, _L, _P],
    "cirr_copy_cols": [_P, _L, _L, _P, _P, _P, _I, _I, _I, _P, _L, _L, _P],
    "cirr_transpose": [_I, _P, _L, _L, _I, _I, _I, _P, _L, _L, _P],
    "cirr_kde_eval": [_P, _I, _P, _I, _D, _P, _P],
    "cirr_target_sm": [],
    "cirr_set_coop_ctas": [_I],
    "cirr_set_gemm_ctas": [_I],
    "cirr_set_oom_handler": [_P],
    "cirr_launch_count": [],
    "cirr_gemm_ptrs": [_I, _I, _I, _I, _I, _P, _L, _P, _L, _L, _P, _L, _L, _D, _I, _P],
    "cirr_gather_blocks": [_I, _P, _L, _P, _L, _L, _P],
    "cirr_zero": [_P, _L, _P],
    "cirr_set_lu_gemm": [_I],
    "cirr_ozaki_factor_bytes": [_I, _I],
    "cirr_ozaki_split_factors": [_P, _I, _L, _L, _I, _P, _P],
    "cirr_ozaki_release": [_P],
    "cirr_ozaki_zgemm_sub": [_P, _L, _L, _P, _L, _L, _P, _L, _L, _I, _I, _I, _I, _P],
}
_RESTYPE = {"cirr_ozaki_factor_bytes": _L, "cirr_diag_inv_bytes": _L, "cirr_zgetrf_ws_bytes": _L, "cirr_small_eig_ws_bytes": _L, "cirr_launch_count": _L, "cirr_orth_ws_bytes": _L,
            "cirr_gen_eig_ws_bytes": _L, "cirr_gen_eig_vec_scratch_bytes": _L, "cirr_orth_cholqr2_ws_bytes": _L,
            "cirr_gen_eig_refine_ws_bytes": _L}
_RAW = {"cirr_set_lu_gemm", "cirr_ozaki_factor_bytes", "cirr_zgetrs_uses_dinv", "cirr_set_coop_ctas", "cirr_set_gemm_ctas", "cirr_diag_inv_bytes", "cirr_zgetrf_ws_bytes", "cirr_small_eig_ws_bytes", "cirr_launch_count", "cirr_target_sm", "cirr_orth_ws_bytes",
        "cirr_gen_eig_ws_bytes", "cirr_gen_eig_vec_scratch_bytes", "cirr_orth_cholqr2_ws_bytes",
        "cirr_gen_eig_refine_ws_bytes"}

_lib = None


def load(path: str = LIB_PATH):
    """Load libcirr.so once (raises DeviceError when absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise DeviceError(f"libcirr.so not built at {path}; run `make` (or __graft_entry__.build())")
    lib = ctypes.CDLL(path)
    for name, argt in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argt
        fn.restype = _RESTYPE.get(name, _I)
    _install_oom_handler(lib)
    _lib = lib
    return lib


_OOM_CB = None


def _install_oom_handler(lib):
    """cirr_set_oom_handler: a failed scratch allocation inside libcirr empties
    PyTorch's caching allocator (which may hold the free HBM) and retries."""
    global _OOM_CB
    proto = ctypes.CFUNCTYPE(None)

    def handler():
        try:
            import torch

            torch.cuda.empty_cache()
        except Exception:  # noqa: BLE001 -- a callback must not raise into C
            pass

    _OOM_CB = proto(handler)
    lib.cirr_set_oom_handler.argtypes = [proto]
    lib.cirr_set_oom_handler.restype = None
    lib.cirr_set_oom_handler(_OOM_CB)


def call(name: str, *args):
    """Invoke an entry point and turn a non-zero status into DeviceError."""
    fn = getattr(load(), name)
    rc = fn(*args)
    if name in _RAW:
        return rc
    if rc != 0:
        if rc == EINVAL:
            raise DeviceError(f"{name}: invalid arguments")
        raise DeviceError(f"{name}: CUDA error {rc}")
    return rc
