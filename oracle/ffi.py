"""ctypes access to the CPU checkers (TEST INFRASTRUCTURE ONLY).

  orc  -> oracle/liboracle.so          our fp64 C restatement (oracle.c)
  ref  -> oracle/_ref/libgnstk_ref.so   the unmodified reference library
                                        compiled from /root/reference (optional)

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module.  The product path (paper_2411_00999_b200) never does.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libgnstk_ref.so")

_dp = ctypes.POINTER(ctypes.c_double)
_fp = ctypes.POINTER(ctypes.c_float)
_i64 = ctypes.c_int64


def _p(a):
    if a is None:
        return None
    assert a.flags.c_contiguous
    if a.dtype == np.float64:
        return a.ctypes.data_as(_dp)
    if a.dtype == np.float32:
        return a.ctypes.data_as(_fp)
    raise TypeError(a.dtype)


class Oracle:
    """Our restatement (oracle.c)."""

    def __init__(self, path=ORC_PATH):
        self.h = ctypes.CDLL(path)
        h = self.h
        h.orc_last_error.restype = ctypes.c_char_p
        h.orc_synth_z.restype = ctypes.c_float
        h.orc_synth_z.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        h.orc_synth_ln.argtypes = [_fp, _fp, _fp, _fp, _i64, _i64, _i64, _i64, _i64, ctypes.c_float,
                                   ctypes.c_uint64, ctypes.c_int]
        h.orc_synth_linear.argtypes = [_fp, _fp, _i64, _i64, _i64, _i64, _i64, _i64, ctypes.c_uint64, ctypes.c_int]
        h.orc_layernorm_forward.argtypes = [_dp, _dp, _dp, ctypes.c_double, _i64, _i64, _dp, _dp, _dp]
        h.orc_layernorm_backward.argtypes = [_dp, _dp, _dp, _dp, _i64, _i64, _i64, _dp, _dp, _dp, _dp, _dp, _dp]
        h.orc_layernorm_backward_xmr.argtypes = [_dp, _dp, _dp, _dp, _dp, _i64, _i64, _i64, _dp, _dp, _dp, _dp,
                                                 _dp, _dp]
        h.orc_linear_backward.argtypes = [_dp, _dp, _dp, ctypes.c_int, _i64, _i64, _i64, _i64, _dp, _dp, _dp, _dp,
                                          _dp, _dp]
        h.orc_linear_frobenius.argtypes = [_dp, _dp, _i64, _i64, _i64, _i64, _dp]
        h.orc_embedding_backward.argtypes = [ctypes.POINTER(ctypes.c_int32), _dp, _i64, _i64, _i64, _i64, _dp, _dp,
                                             _dp]
        h.orc_crossover_t.argtypes = [_i64, _i64, ctypes.c_int, _dp]
        h.orc_flops.argtypes = [_i64, _i64, _i64, _i64, ctypes.c_int, ctypes.POINTER(_i64)]
        h.orc_io_values.argtypes = [_i64, _i64, _i64, _i64, ctypes.c_int, ctypes.POINTER(_i64)]
        h.orc_gauss_next.restype = ctypes.c_double
        h.orc_round_bf16.restype = ctypes.c_float
        h.orc_round_bf16.argtypes = [ctypes.c_float]

    def err(self):
        return self.h.orc_last_error().decode()

    # ---------------------------------------------------------------- synth
    def synth_ln(self, B, T, D, b_offset=0, B_div=None, sigma=0.3, stream0=0, bf16=False):
        x = np.empty((B, T, D), np.float32)
        dy = np.empty((B, T, D), np.float32)
        gamma = np.empty(D, np.float32)
        beta = np.empty(D, np.float32)
        self.h.orc_synth_ln(_p(x), _p(dy), _p(gamma), _p(beta), B, T, D, b_offset, B_div or B, sigma, stream0,
                            1 if bf16 else 0)
        return x, dy, gamma, beta

    def synth_linear(self, B, T, K, L, b_offset=0, B_div=None, stream0=10, bf16=False):
        x = np.empty((B, T, K), np.float32)
        dy = np.empty((B, T, L), np.float32)
        self.h.orc_synth_linear(_p(x), _p(dy), B, T, K, L, b_offset, B_div or B, stream0, 1 if bf16 else 0)
        return x, dy

    # --------------------------------------------------------------- layers
    def ln_forward(self, x, gamma, beta, eps=1e-5):
        x = np.ascontiguousarray(x, np.float64)
        D = x.shape[-1]
        rows = x.size // D
        y = np.empty_like(x)
        xhat = np.empty_like(x)
        inv = np.empty(x.shape[:-1], np.float64)
        rc = self.h.orc_layernorm_forward(_p(x), _p(np.ascontiguousarray(gamma, np.float64)),
                                          _p(np.ascontiguousarray(beta, np.float64)), eps, rows, D, _p(y), _p(xhat),
                                          _p(inv))
        if rc:
            raise ValueError(self.err())
        return y, xhat, inv

    def ln_backward(self, xhat, inv_std, g, gamma, mean=None):
        """Reference backward.  With mean given, `xhat` is x and xhat = (x-mean)*inv_std."""
        g = np.ascontiguousarray(g, np.float64)
        B = g.shape[0]
        D = g.shape[-1]
        M = g.size // (B * D) if B and D else 0
        dx = np.empty_like(g)
        dgamma = np.empty(D)
        dbeta = np.empty(D)
        rg = np.empty(B)
        rb = np.empty(B)
        corr = np.empty(2)
        xa = np.ascontiguousarray(xhat, np.float64)
        ia = np.ascontiguousarray(inv_std, np.float64)
        ga = np.ascontiguousarray(gamma, np.float64)
        if mean is None:
            rc = self.h.orc_layernorm_backward(_p(xa), _p(ia), _p(g), _p(ga), B, M, D, _p(dx), _p(dgamma),
                                               _p(dbeta), _p(rg), _p(rb), _p(corr))
        else:
            ma = np.ascontiguousarray(mean, np.float64)
            rc = self.h.orc_layernorm_backward_xmr(_p(xa), _p(ma), _p(ia), _p(g), _p(ga), B, M, D, _p(dx),
                                                   _p(dgamma), _p(dbeta), _p(rg), _p(rb), _p(corr))
        if rc:
            raise ValueError(self.err())
        return dict(dx=dx, dgamma=dgamma, dbeta=dbeta, raw_gamma=rg, raw_beta=rb, corrected=corr)

    def linear_backward(self, x, g, W, bias=None):
        x = np.ascontiguousarray(x, np.float64)
        g = np.ascontiguousarray(g, np.float64)
        W = np.ascontiguousarray(W, np.float64)
        B = x.shape[0]
        K = x.shape[-1]
        L = g.shape[-1]
        M = x.size // (B * K) if B and K else 0
        dW = np.empty((K, L))
        db = np.empty(L)
        rw = np.empty(B)
        rb = np.empty(B)
        corr = np.empty(2)
        dx = np.empty_like(x)
        rc = self.h.orc_linear_backward(_p(x), _p(g), _p(W), 1 if bias is not None else 0, B, M, K, L, _p(dW),
                                        _p(db), _p(rw), _p(rb), _p(corr), _p(dx))
        if rc:
            raise ValueError(self.err())
        out = dict(dW=dW, raw_w=rw, corrected=corr, dx=dx)
        if bias is not None:
            out.update(dbias=db, raw_b=rb)
        return out

    def linear_frobenius(self, x, g):
        x = np.ascontiguousarray(x, np.float64)
        g = np.ascontiguousarray(g, np.float64)
        B, T, K = x.shape
        L = g.shape[-1]
        out = np.empty(B)
        rc = self.h.orc_linear_frobenius(_p(x), _p(g), B, T, K, L, _p(out))
        if rc:
            raise ValueError(self.err())
        return out

    def embedding_backward(self, ids, g, V):
        """layers.cpp:315-368: ids [B, T] int32, g [B, T, D] -> dW [V, D], raw [B], corrected."""
        ids = np.ascontiguousarray(ids, np.int32)
        g = np.ascontiguousarray(g, np.float64)
        B, T, D = g.shape
        dW = np.empty((V, D))
        raw = np.empty(B)
        corr = np.empty(1)
        rc = self.h.orc_embedding_backward(ids.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), _p(g), B, T, V, D,
                                           _p(dW), _p(raw), _p(corr))
        if rc:
            raise ValueError(self.err())
        return dict(dW=dW, raw_w=raw, corrected=float(corr[0]))

    def crossover_t(self, k, l, criterion):
        out = ctypes.c_double()
        rc = self.h.orc_crossover_t(k, l, criterion, ctypes.byref(out))
        if rc:
            raise ValueError(self.err())
        return out.value

    def flops(self, b, t, k, l, method):
        out = (_i64 * 2)()
        if self.h.orc_flops(b, t, k, l, method, out):
            raise ValueError(self.err())
        return out[0], out[1]

    def io_values(self, b, t, k, l, method):
        out = (_i64 * 2)()
        if self.h.orc_io_values(b, t, k, l, method, out):
            raise ValueError(self.err())
        return out[0], out[1]

    def round_bf16(self, v: float) -> float:
        return self.h.orc_round_bf16(v)


class Reference:
    """The unmodified reference library (oracle/_ref/libgnstk_ref.so)."""

    def __init__(self, path=REF_PATH):
        self.h = ctypes.CDLL(path)
        h = self.h
        h.ref_last_error.restype = ctypes.c_char_p
        h.ref_layernorm_forward.argtypes = [_dp, _dp, _dp, ctypes.c_double, _i64, _i64, _dp, _dp, _dp]
        h.ref_layernorm_backward.argtypes = [_dp, _dp, _dp, _dp, _i64, _i64, _i64, _dp, _dp, _dp, _dp, _dp, _dp]
        h.ref_layernorm_backward_threaded.argtypes = [ctypes.c_int, _dp, _dp, _dp, _dp, _i64, _i64, _i64, _dp, _dp,
                                                      _dp, _dp, _dp, _dp]
        h.ref_linear_backward.argtypes = [_dp, _dp, _dp, _dp, _i64, _i64, _i64, _i64, _dp, _dp, _dp, _dp, _dp, _dp]
        h.ref_linear_frobenius.argtypes = [_dp, _dp, _i64, _i64, _i64, _i64, _dp]
        h.ref_gauss_draw.argtypes = [ctypes.c_uint64, _i64, _dp]

    def ln_backward(self, xhat, inv_std, g, gamma, threads=0):
        g = np.ascontiguousarray(g, np.float64)
        B = g.shape[0]
        D = g.shape[-1]
        M = g.size // (B * D)
        dx = np.empty_like(g)
        dgamma = np.empty(D)
        dbeta = np.empty(D)
        rg = np.empty(B)
        rb = np.empty(B)
        corr = np.empty(2)
        args = (_p(np.ascontiguousarray(xhat, np.float64)), _p(np.ascontiguousarray(inv_std, np.float64)), _p(g),
                _p(np.ascontiguousarray(gamma, np.float64)), B, M, D, _p(dx), _p(dgamma), _p(dbeta), _p(rg), _p(rb),
                _p(corr))
        rc = (self.h.ref_layernorm_backward_threaded(threads, *args) if threads else
              self.h.ref_layernorm_backward(*args))
        if rc:
            raise ValueError(self.h.ref_last_error().decode())
        return dict(dx=dx, dgamma=dgamma, dbeta=dbeta, raw_gamma=rg, raw_beta=rb, corrected=corr)

    def ln_forward(self, x, gamma, beta, eps=1e-5):
        x = np.ascontiguousarray(x, np.float64)
        D = x.shape[-1]
        rows = x.size // D
        y = np.empty_like(x)
        xhat = np.empty_like(x)
        inv = np.empty(x.shape[:-1], np.float64)
        rc = self.h.ref_layernorm_forward(_p(x), _p(np.ascontiguousarray(gamma, np.float64)),
                                          _p(np.ascontiguousarray(beta, np.float64)), eps, rows, D, _p(y), _p(xhat),
                                          _p(inv))
        if rc:
            raise ValueError(self.h.ref_last_error().decode())
        return y, xhat, inv

    def gauss(self, seed, n):
        out = np.empty(n)
        self.h.ref_gauss_draw(seed, n, _p(out))
        return out


def oracle() -> Oracle:
    return Oracle()


def reference_available() -> bool:
    return os.path.exists(REF_PATH)


def reference() -> Reference:
    return Reference()
