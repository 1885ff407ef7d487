"""ctypes binding of the C ABI in include/rbws_b200.h.

The shared library ``_rbws_b200.so`` is built in-tree by ``build.py`` (nvcc,
sm_100a).  There is no fallback: if the library is missing or no CUDA device
is present, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_NAME = "_rbws_b200.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

_c_int, _c_int64, _c_double, _vp = ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
_pp = ctypes.POINTER(ctypes.c_void_p)
_ip = ctypes.POINTER(ctypes.c_int)
_dp = ctypes.POINTER(ctypes.c_double)

# name -> argtypes (every function returns int unless listed in _RESTYPES)
SIGNATURES = {
    "rbws_version": [],
    "rbws_last_error": [],
    "rbws_launch_count": [],
    "rbws_fetch": [_vp, _vp, _c_int64, _vp],
    "rbws_hierarchy_create": [_pp, _c_int, _c_int, _c_int, _vp, _vp],
    "rbws_hierarchy_create_stored": [_pp, _c_int, _c_int, _c_int, _vp],
    "rbws_hierarchy_is_stored": [_vp],
    "rbws_hierarchy_term_apply": [_vp, _c_int, _c_int, _c_int, _vp, _vp, _vp],
    "rbws_hierarchy_destroy": [_vp],
    "rbws_hierarchy_levels": [_vp],
    "rbws_hierarchy_cells": [_vp, _c_int],
    "rbws_hierarchy_factors": [_vp, _c_int, _vp, _c_int64],
    "rbws_kron_factors": [_c_int, _c_int, _c_int, _vp, _vp, _c_int, _vp, _c_int64],
    "rbws_batch_create": [_pp, _vp, _c_int, _c_int, _c_double],
    "rbws_batch_destroy": [_vp],
    "rbws_batch_setup": [_vp, _vp, _c_int, _ip, _vp],
    "rbws_batch_set_graph": [_vp, _c_int],
    "rbws_set_kernel_variant": [_c_int, _c_int],
    "rbws_batch_set_smoother": [_vp, _c_int],
    "rbws_smooth": [_vp, _c_int, _c_int, _vp, _vp, _vp],
    "rbws_batch_stored_weights": [_vp],
    "rbws_batch_fused_restrict": [_vp],
    "rbws_batch_pre_scaled": [_vp],
    "rbws_batch_cg_fused": [_vp],
    "rbws_apply": [_vp, _c_int, _vp, _vp, _vp],
    "rbws_jacobi_sweep": [_vp, _c_int, _vp, _vp, _vp, _vp],
    "rbws_restrict": [_c_int, _c_int, _vp, _vp, _vp],
    "rbws_prolong_add": [_c_int, _c_int, _vp, _vp, _vp],
    "rbws_vcycle": [_vp, _vp, _vp, _vp],
    "rbws_mgcg_solve": [_vp, _vp, _c_int64, _vp, _c_double, _c_int, _vp, _vp, _vp, _vp, _vp],
    "rbws_msrbcg_solve": [_vp, _vp, _c_int64, _vp, _c_double, _c_int, _c_int, _vp, _vp, _vp, _vp,
                          _vp, _vp, _vp, _vp, _vp],
    "rbws_mgcg_solve_to_host": [_vp, _vp, _c_int64, _vp, _c_double, _c_int, _vp, _vp, _vp, _vp,
                                _vp, _vp, _c_int64, _vp],
    "rbws_batch_dinv": [_vp, _c_int, _vp, _vp],
    "rbws_level_kernel": [_vp, _c_int, _c_int, _vp, _vp, _vp, _vp],
    "rbws_batch_profile": [_vp, _c_int],
    "rbws_batch_profile_read": [_vp, _vp, _vp, _vp, _c_int],
    "rbws_l1roc_project": [_vp, _vp, _c_int64, _c_int, _vp, _c_int, _vp, _vp],
    "rbws_l1roc_online": [_c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp, _c_int64, _vp, _vp,
                          _vp, _vp, _vp, _vp],
    "rbws_basis_dot": [_c_int64, _c_int, _vp, _c_int64, _c_int, _vp, _c_int64, _vp, _vp],
    "rbws_expand": [_c_int, _c_int, _vp, _c_int64, _c_int, _vp, _vp, _vp],
    "rbws_deim_step": [_c_int, _vp, _c_int64, _c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "rbws_deim_step_fn": [_c_int, _vp, _c_int64, _c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "rbws_dense_solve": [_c_int, _vp, _vp, _vp, _vp, _vp],
    "rbws_comm_unique_id": [_vp],
    "rbws_slab_create": [_pp, _vp, _c_int, _c_int, _vp, _c_int, _c_int, _c_double],
    "rbws_slab_destroy": [_vp],
    "rbws_slab_info": [_vp, _ip, _c_int, _ip, _ip],
    "rbws_slab_setup": [_vp, _vp, _ip, _vp],
    "rbws_slab_load": [_vp, _c_int, _vp, _c_int64, _c_int, _vp],
    "rbws_slab_store": [_vp, _c_int, _vp, _c_int64, _c_int, _vp],
    "rbws_slab_prolong_x": [_vp, _vp, _vp],
    "rbws_slab_solve": [_vp, _c_double, _c_int, _ip, _vp, _vp, _ip, _vp],
    # full-node layout (csrc/planes.cu)
    "rbws_fn_combine": [_c_int, _c_int, _c_int, _vp, _vp, _vp, _vp],
    "rbws_fn_apply": [_c_int, _c_int, _vp, _vp, _vp, _vp, _c_int, _vp],
    "rbws_fn_apply_shared": [_c_int, _c_int, _c_int, _vp, _vp, _vp, _vp, _vp, _c_int, _vp],
    "rbws_fn_band_doubles": [_c_int, _c_int, _c_int],
    "rbws_fn_band_factor": [_c_int, _c_int, _c_int, _vp, _vp, _vp, _vp],
    "rbws_fn_band_solve": [_c_int, _c_int, _c_int, _vp, _vp, _vp, _c_double, _c_int, _vp],
    "rbws_fn_band_transpose": [_c_int, _c_int, _c_int, _vp, _vp, _vp],
    "rbws_fn_band_solve_t": [_c_int, _c_int, _c_int, _vp, _vp, _vp, _vp, _c_double, _c_int, _vp],
    "rbws_fn_plane_gs_sweep": [_c_int, _c_int, _vp, _vp, _vp, _vp, _vp, _c_int, _vp],
    "rbws_fn_restrict": [_c_int, _c_int, _vp, _vp, _vp, _vp],
    "rbws_fn_prolong_add": [_c_int, _c_int, _vp, _vp, _vp, _vp],
    "rbws_fn_point_jacobi": [_c_int, _c_int, _vp, _vp, _vp, _c_double, _vp],
}
_RESTYPES = {"rbws_last_error": ctypes.c_char_p, "rbws_launch_count": ctypes.c_int64,
             "rbws_fn_band_doubles": ctypes.c_int64}


def launch_count() -> int:
    return int(load().rbws_launch_count())

_lib = None


class NativeError(RuntimeError):
    """A C-ABI call failed (message from rbws_last_error)."""


def load(path: str | os.PathLike | None = None):
    """Load (once) and return the ctypes library; raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    # RBWS_LIB: an alternative build of the same library (kernel-variant experiments)
    p = Path(path) if path else Path(os.environ.get("RBWS_LIB") or LIB_PATH)
    if not p.exists():
        raise NativeError(
            f"native library {p} not built; run `python build.py` (nvcc, sm_100a). "
            "There is no CPU fallback.")
    lib = ctypes.CDLL(str(p))
    for name, argtypes in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = _RESTYPES.get(name, ctypes.c_int)
    _lib = lib
    return lib


def call(name: str, *args) -> int:
    """Invoke an entry point; non-zero status raises NativeError."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.rbws_last_error().decode(errors="replace")
        raise NativeError(f"{name} failed: {msg}")
    return rc


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise NativeError("no CUDA device: the RBWS B200 path has no CPU fallback")
    load()


def fetch(t):
    """Small device tensor -> numpy array through rbws_fetch (kernel stores into
    mapped pinned memory; no copy-engine DMA that could queue behind a bulk
    download on another stream).  Synchronises the current stream."""
    import numpy as np
    import torch
    dt = {torch.float64: np.float64, torch.float32: np.float32, torch.int32: np.int32,
          torch.int64: np.int64, torch.bool: np.bool_, torch.uint8: np.uint8}[t.dtype]
    t = t.contiguous()
    out = np.empty(tuple(t.shape), dtype=dt)
    call("rbws_fetch", out.ctypes.data, t.data_ptr(), t.numel() * t.element_size(), stream_ptr())
    return out


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
