"""ctypes binding of libppcg_b200.so (the C ABI declared in include/ppcg_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is present, every
device entry point raises DeviceError.  ``build()`` in __graft_entry__.py (or ``make``)
produces the library in-tree.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import DeviceError, raise_for_status

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PPCG_B200_LIB") or os.path.join(_HERE, "libppcg_b200.so")  # override: A/B builds

_lock = threading.Lock()
_lib = None

c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_dbl = ctypes.c_double
vp = ctypes.c_void_p
PP = ctypes.POINTER(ctypes.c_void_p)

# name -> (restype, argtypes)
_SIGS = {
    "bk_version": (c_int, []),
    "bk_launch_count": (ctypes.c_ulonglong, []),
    "bk_spmm_csr_d": (c_int, [c_i64, vp, vp, vp, c_int, vp, c_i64, vp, c_i64, vp]),
    "bk_spmm_csr_z": (c_int, [c_i64, vp, vp, vp, c_int, vp, c_i64, vp, c_i64, vp]),
    "bk_spmm_set_variant": (c_int, [c_int]),
    "bk_spmm_march_d": (c_int, [c_int, c_int, c_int, c_int, c_int, c_i64, vp, vp, c_int, c_int, c_int, vp, c_i64,
                                vp, c_i64, c_int, vp]),
    "bk_spmm_march_z": (c_int, [c_int, c_int, c_int, c_int, c_int, c_i64, vp, vp, c_int, c_int, c_int, vp, c_i64,
                                vp, c_i64, c_int, vp]),
    "bk_spmm_stencil_d": (c_int, [c_int, c_int, c_int, c_int, c_int, c_i64, vp, c_int, c_int, c_int, vp, c_i64,
                                  vp, c_i64, c_int, vp]),
    "bk_spmm_stencil_z": (c_int, [c_int, c_int, c_int, c_int, c_int, c_i64, vp, c_int, c_int, c_int, vp, c_i64,
                                  vp, c_i64, c_int, vp]),
    "bk_spmm_stencil_set_config": (c_int, [c_int]),
    "bk_subblock_grams_set_waves": (c_int, [c_int]),
    "bk_scale_rows_d": (c_int, [c_i64, c_int, vp, vp, c_i64, vp, c_i64, vp]),
    "bk_gram_ws_bytes": (c_i64, [c_i64, c_int, c_int]),
    "bk_gram_d": (c_int, [c_i64, c_int, c_int, vp, c_i64, vp, c_i64, vp, c_i64, c_int, vp, c_i64, vp]),
    "bk_gram_splits": (c_int, [c_int, c_int]),
    "bk_gram_set_loader": (c_int, [c_int]),
    "bk_gram_set_combo": (c_int, [c_int]),
    "bk_gram_part_d": (c_int, [c_i64, c_int, c_int, vp, c_i64, vp, c_i64, vp, c_i64, c_int, c_int, vp, c_i64,
                               vp]),
    "bk_gram2_part_d": (c_int, [c_i64, c_int, c_int, vp, c_i64, vp, c_i64, vp, c_i64, c_int, c_int, vp, c_i64,
                                vp, c_i64, vp, c_i64, c_int, vp, c_i64, vp]),
    "bk_gram2_d": (c_int, [c_i64, c_int, c_int, vp, c_i64, vp, c_i64, vp, c_i64,
                           c_int, c_int, vp, c_i64, vp, c_i64, vp, c_i64, vp, c_i64, vp]),
    "bk_cplx_gram_combine_d": (c_int, [c_int, c_int, vp, c_i64, vp, c_i64, vp]),
    "bk_subblock_grams_ws_bytes": (c_i64, [c_i64, c_int, c_int, c_int]),
    "bk_subblock_grams_d": (c_int, [c_i64, c_int, c_int, c_int, vp, vp, vp, vp, vp, vp, c_i64, c_i64,
                                    vp, vp, vp, c_i64, vp]),
    "bk_subblock_grams_z": (c_int, [c_i64, c_int, c_int, c_int, vp, vp, vp, vp, vp, vp, c_i64, c_i64,
                                    vp, vp, vp, vp, vp, c_i64, vp]),
    "bk_pencil_max_dim": (c_int, []),
    "bk_pencil_phase_clocks": (c_int, [vp]),
    "bk_pencil_set_eig": (c_int, [c_int]),
    "bk_pencil_ws_bytes": (c_i64, [c_int, c_int, c_int]),
    "bk_block_assemble": (c_int, [c_int, c_int, vp, vp, vp, vp, c_i64, vp, vp, c_i64, vp]),
    "bk_block_coef": (c_int, [c_int, c_int, c_int, c_int, vp, vp, vp, c_i64, vp, vp, vp]),
    "bk_block_stats": (c_int, [c_i64, c_int, c_int, vp, c_i64, vp, c_int, vp]),
    "bk_svals_d": (c_int, [vp, c_int, c_int, vp, c_i64, vp]),
    "bk_svals_z": (c_int, [vp, c_int, c_int, vp, c_i64, vp]),
    "bk_subblock_pencils_z": (c_int, [c_int, c_int, c_int, vp, vp, vp, vp, vp, vp, c_int, vp, c_i64, vp]),
    "bk_pencil_batched_z": (c_int, [c_int, c_int, c_int, vp, vp, c_int, vp, vp, vp, vp, c_i64, vp]),
    "bk_subblock_recombine_z": (c_int, [c_i64, c_int, c_int, c_int, vp, vp, vp, vp, vp, vp, vp,
                                        vp, vp, vp, vp, c_i64, c_i64, vp, vp, vp]),
    "bk_subblock_pencils_d": (c_int, [c_int, c_int, c_int, vp, vp, vp, vp, vp, vp, c_int, vp, c_i64, vp]),
    "bk_pencil_batched_d": (c_int, [c_int, c_int, c_int, vp, vp, c_int, vp, vp, vp, vp, c_i64, vp]),
    "bk_subblock_recombine_d": (c_int, [c_i64, c_int, c_int, c_int, vp, vp, vp, vp, vp, vp, vp,
                                        vp, vp, vp, vp, c_i64, c_i64, vp, vp]),
    "bk_tsgemm_ws_bytes": (c_i64, [c_i64, c_int]),
    "bk_tsgemm_d": (c_int, [c_i64, c_int, c_int, c_dbl, vp, c_i64, vp, c_i64, c_dbl, vp, c_i64, vp,
                            c_i64, vp, c_int, vp]),
    "bk_tsgemm_batched_d": (c_int, [c_int, c_i64, c_int, c_int, c_dbl, PP, c_i64, PP, c_i64, c_dbl,
                                    PP, c_i64, PP, c_i64, vp, c_int, c_int, c_int, vp, vp, c_i64, vp]),
    "bk_cplx_expand_d": (c_int, [c_int, c_int, vp, c_i64, vp, c_i64, vp]),
    "bk_fp64_emu_set": (c_int, [c_int]),
    "bk_fp64_emu_enabled": (c_int, []),
    "bk_ozaki_timing": (c_int, [c_int]),
    "bk_ozaki_kernel_ms": (c_dbl, []),
    "bk_ozaki_gram_ws_bytes": (c_i64, [c_i64, c_int, c_int, c_int, c_int]),
    "bk_ozaki_gram_d": (c_int, [c_i64, c_int, c_int, vp, c_i64, vp, c_i64, vp, c_i64, c_int, vp, c_i64, vp]),
    "bk_ozaki_gram2_ws_bytes": (c_i64, [c_i64, c_int, c_int, c_int]),
    "bk_ozaki_gram2_d": (c_int, [c_i64, c_int, vp, c_i64, c_int, vp, c_i64, vp, c_i64, c_int, vp, c_i64, vp, c_i64,
                                 vp, c_i64, vp]),
    "bk_ozaki_coldigits_bytes": (c_i64, [c_i64, c_int]),
    "bk_ozaki_coldigits_d": (c_int, [c_i64, c_int, vp, c_i64, vp, c_i64, vp]),
    "bk_ozaki_gram_pre_ws_bytes": (c_i64, [c_i64, c_int, c_int, c_int, c_int]),
    "bk_ozaki_gram_pre_d": (c_int, [c_i64, c_int, c_int, vp, c_i64, vp, c_int, c_int, vp, c_i64, vp, c_i64, c_int, vp,
                                    c_i64, vp]),
    "bk_ozaki_gram2_pre_ws_bytes": (c_i64, [c_i64, c_int, c_int, c_int]),
    "bk_ozaki_gram2_pre_d": (c_int, [c_i64, c_int, vp, c_i64, vp, c_int, c_int, c_int, vp, c_i64, vp, c_i64, c_int, vp,
                                     c_i64, vp, c_i64, vp, c_i64, vp]),
    "bk_ozaki_tsgemm_ws_bytes": (c_i64, [c_int, c_i64, c_int, c_int, c_int]),
    "bk_ozaki_tsgemm_d": (c_int, [c_int, c_i64, c_int, c_int, c_dbl, PP, c_i64, PP, c_i64, c_dbl, PP, c_i64, PP,
                                  c_i64, vp, c_int, c_int, c_int, vp, vp, c_i64, vp]),
    "bk_sumsq_ws_bytes": (c_i64, []),
    "bk_sumsq_d": (c_int, [c_i64, c_int, vp, c_i64, vp, vp, c_i64, vp]),
    "bk_small_stats_d": (c_int, [c_int, c_int, vp, c_i64, c_int, vp, vp]),
    "bk_rr_residual_ws_bytes": (c_i64, [c_int]),
    "bk_rr_residual_d": (c_int, [c_i64, c_int, c_int, vp, c_i64, vp, c_i64, vp, vp, vp, c_i64, vp, vp,
                                 c_i64, vp]),
    "bk_copy_cols": (c_int, [c_i64, c_int, c_int, vp, c_i64, c_i64, vp, c_i64, c_i64, vp]),
    "bk_zero_cols": (c_int, [c_i64, c_int, c_int, vp, c_i64, c_i64, vp]),
    "bk_dense_create": (c_int, [PP, vp]),
    "bk_dense_destroy": (c_int, [vp]),
    "bk_dense_set_stream": (c_int, [vp, vp]),
    "bk_chol_upper_floor_d": (c_int, [vp, c_int, vp, c_i64, vp]),
    "bk_chol_upper_floor_z": (c_int, [vp, c_int, vp, c_i64, vp]),
    "bk_tri_inv_upper_d": (c_int, [vp, c_int, vp, c_i64]),
    "bk_tri_inv_upper_z": (c_int, [vp, c_int, vp, c_i64]),
    "bk_rr_pencil_d": (c_int, [vp, c_int, vp, c_i64, vp, c_i64, vp, vp, c_i64, vp]),
    "bk_rr_pencil_z": (c_int, [vp, c_int, vp, c_i64, vp, c_i64, vp, vp, c_i64, vp]),
    "bk_householder_q_d": (c_int, [vp, c_i64, c_int, vp, c_i64, vp]),
    "bk_householder_q_z": (c_int, [vp, c_i64, c_int, vp, c_i64, vp]),
}

EXPORTED = tuple(_SIGS)


def load(require_cuda=True):
    """Load the library (once).  Raises DeviceError when it is missing."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise DeviceError(
                    f"native library not built: {LIB_PATH} is missing (run `make` or "
                    "__graft_entry__.build()); there is no CPU fallback")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    if require_cuda:
        import torch

        if not torch.cuda.is_available():
            raise DeviceError("no CUDA device: the PPCG hot path runs only on the GPU (no CPU fallback)")
    return _lib


def call(name, *args):
    """Invoke a status-returning entry point and raise on failure."""
    lib = load()
    code = getattr(lib, name)(*args)
    raise_for_status(code, name)
    return code


def ptr_array(ptrs):
    arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
    return ctypes.cast(arr, PP), arr
