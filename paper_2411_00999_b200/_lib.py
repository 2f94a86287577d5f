"""ctypes binding of the C ABI in include/gnsb.h (libgnsb.so, built in-tree).

The library is the product: it holds every CUDA kernel.  There is no Python
or CPU fallback — if the shared object is missing this module raises at
import-time use, and on a machine without a GPU every compute entry point
returns GNSB_ECUDA, which is raised as RuntimeError.
"""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libgnsb.so")
# A/B experiments only: GNSB_LIB_VARIANT=<tag> loads lib/libgnsb_<tag>.so (a
# build of the same sources with different compile-time knobs)
if os.environ.get("GNSB_LIB_VARIANT"):
    LIB_PATH = os.path.join(_HERE, "lib", "libgnsb_%s.so" % os.environ["GNSB_LIB_VARIANT"])

GNSB_OK, GNSB_EINVAL, GNSB_ECUDA, GNSB_ENCCL, GNSB_ENOMEM = 0, 1, 2, 3, 4
GNSB_F32, GNSB_BF16, GNSB_F64 = 0, 1, 2
LAYER_EMBEDDING, LAYER_LINEAR, LAYER_LAYERNORM = 0, 1, 2

c_i64 = ctypes.c_int64
c_i32 = ctypes.c_int32
c_f64 = ctypes.c_double
c_vp = ctypes.c_void_p
c_dp = ctypes.POINTER(ctypes.c_double)
c_szp = ctypes.POINTER(ctypes.c_size_t)


class GradStats(ctypes.Structure):
    """gnstk::GradStats (proj/include/gnstk/gns.hpp:16-22)."""

    _fields_ = [
        ("g_big_sqnorm", c_f64),
        ("g_small_sqnorm_mean", c_f64),
        ("b_big", c_i64),
        ("b_small", c_i64),
        ("n_small", c_i64),
    ]


class GnsEstimate(ctypes.Structure):
    """gnstk::GnsEstimate (gns.hpp:26-31)."""

    _fields_ = [("g2", c_f64), ("s", c_f64), ("b_simple", c_f64), ("b_simple_defined", c_i32)]


class EmaState(ctypes.Structure):
    """gnstk::EmaState (gns.hpp:36-40)."""

    _fields_ = [("alpha", c_f64), ("value", c_f64), ("count", c_i64)]


class LnBwdPending(ctypes.Structure):
    """gnsb_ln_bwd_pending (include/gnsb.h): one LayerNorm whose stage 2 is deferred."""

    _fields_ = [("ws", c_vp), ("ws_bytes", ctypes.c_size_t), ("B", c_i64), ("M", c_i64), ("D", c_i64),
                ("dt", c_i32), ("dgamma", c_vp), ("dbeta", c_vp), ("raw_sq_gamma", c_vp), ("raw_sq_beta", c_vp),
                ("sums", c_vp)]


_SIGS = {
    "gnsb_version": (ctypes.c_char_p, []),
    "gnsb_last_error": (ctypes.c_char_p, []),
    "gnsb_ln_fwd": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_f64, c_i32, c_vp]),
    "gnsb_ln_bwd_workspace_size": (c_i32, [c_i64, c_i64, c_i64, c_i32, c_szp]),
    "gnsb_ln_bwd": (
        c_i32,
        [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_i64, c_i64, c_i64, c_i32, c_vp,
         ctypes.c_size_t, c_vp],
    ),
    "gnsb_ln_bwd_rows": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i32, c_vp,
                                 ctypes.c_size_t, c_vp]),
    "gnsb_ln_bwd_reduce": (c_i32, [ctypes.POINTER(LnBwdPending), c_i32, c_i32, c_vp]),
    "gnsb_ln_bwd_geometry": (
        c_i32,
        [c_i64, c_i64, c_i64, c_i32, ctypes.POINTER(c_i32), ctypes.POINTER(c_i32), ctypes.POINTER(c_i32)],
    ),
    "gnsb_sqnorm": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp]),
    "gnsb_linear_pe_workspace_size": (c_i32, [c_i64, c_i64, c_i64, c_i64, c_i32, c_szp]),
    "gnsb_linear_pe_norms": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_i32, c_i32, c_vp,
                                     ctypes.c_size_t, c_vp]),
    "gnsb_linear_bias_pe": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i32, c_vp, ctypes.c_size_t, c_vp]),
    "gnsb_embedding_pe_workspace_size": (c_i32, [c_i64, c_i64, c_i64, c_i64, c_i32, c_szp]),
    "gnsb_embedding_pe": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_i32, c_vp,
                                  ctypes.c_size_t, c_vp, c_vp]),
    "gnsb_nccl_available": (c_i32, []),
    "gnsb_nccl_get_unique_id": (c_i32, [c_vp]),
    "gnsb_nccl_comm_init_rank": (c_i32, [ctypes.POINTER(c_vp), c_i32, c_vp, c_i32]),
    "gnsb_nccl_comm_destroy": (c_i32, [c_vp]),
    "gnsb_exchange_workspace_size": (c_i32, [ctypes.POINTER(c_i64), c_i32, c_szp]),
    "gnsb_exchange_pack": (c_i32, [c_vp, c_i32, ctypes.POINTER(c_i64), c_i32, c_vp, c_vp, ctypes.c_size_t, c_vp]),
    "gnsb_exchange_unpack": (c_i32, [c_vp, c_i32, ctypes.POINTER(c_i64), c_i32, c_vp, c_vp, ctypes.c_size_t, c_vp]),
    "gnsb_allreduce_buckets": (c_i32, [c_vp, c_i32, ctypes.POINTER(c_i64), c_i32, c_vp, c_vp, ctypes.c_size_t, c_vp,
                                       c_vp]),
    "gnsb_linear_gemm_workspace_size": (c_i32, [c_i64, c_i64, c_i32, c_i32, c_szp]),
    "gnsb_linear_fwd": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i32, c_i32, c_vp, ctypes.c_size_t,
                                c_vp]),
    "gnsb_linear_dx": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i32, c_i32, c_vp, ctypes.c_size_t, c_vp]),
    "gnsb_linear_gemm": (c_i32, [c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i32, c_i32, c_vp,
                                 ctypes.c_size_t, c_vp]),
    "gnsb_xent": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_f64, c_i32, c_vp, c_vp]),
    "gnsb_embedding_fwd": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i32, c_vp, c_vp]),
    "gnsb_estimate_g2": (c_i32, [ctypes.POINTER(GradStats), c_dp]),
    "gnsb_estimate_s": (c_i32, [ctypes.POINTER(GradStats), c_dp]),
    "gnsb_make_gns_estimate": (None, [c_f64, c_f64, ctypes.POINTER(GnsEstimate)]),
    "gnsb_ema_update": (c_i32, [ctypes.POINTER(EmaState), c_f64]),
    "gnsb_smoothed_gns": (c_i32, [ctypes.POINTER(EmaState), ctypes.POINTER(EmaState), ctypes.POINTER(GnsEstimate)]),
    "gnsb_aggregate": (c_i32, [ctypes.POINTER(GradStats), ctypes.POINTER(c_i32), c_i32, c_i32, ctypes.POINTER(GradStats)]),
    "gnsb_gns_step": (c_i32, [c_vp, ctypes.POINTER(c_i32), c_i32, c_i64, c_f64, c_vp, c_vp, c_vp, c_vp]),
    "gnsb_flops": (c_i32, [c_i64, c_i64, c_i64, c_i64, c_i32, ctypes.POINTER(c_i64)]),
    "gnsb_io_values": (c_i32, [c_i64, c_i64, c_i64, c_i64, c_i32, ctypes.POINTER(c_i64)]),
    "gnsb_crossover_t": (c_i32, [c_i64, c_i64, c_i32, c_dp]),
    "gnsb_synth_ln": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, ctypes.c_float,
                              ctypes.c_uint64, c_i32, c_vp]),
    "gnsb_synth_linear": (c_i32, [c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_i64, c_i64, ctypes.c_uint64, c_i32, c_vp]),
}

_lib = None
_lock = threading.Lock()


class GnsbCudaError(RuntimeError):
    """A CUDA-side failure reported by libgnsb (GNSB_ECUDA)."""


def lib() -> ctypes.CDLL:
    """Load libgnsb.so (once).  Raises loudly when the extension is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"libgnsb.so not found at {LIB_PATH}: the CUDA extension is not built "
                    "(run `python -c 'import __graft_entry__ as g; g.build()'` or `make lib`)"
                )
            h = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
            _lib = h
    return _lib


def last_error() -> str:
    return lib().gnsb_last_error().decode()


def check(status: int) -> None:
    """Map a gnsb_status to the reference's exception classes."""
    if status == GNSB_OK:
        return
    msg = last_error()
    if status == GNSB_EINVAL:
        raise ValueError(msg)  # the reference throws std::invalid_argument
    raise GnsbCudaError(msg or f"gnsb status {status}")


def exported_symbols() -> list:
    return sorted(_SIGS)
