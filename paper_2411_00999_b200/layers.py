"""LayerNorm forward / simultaneous backward on B200, mirroring the reference API.

Mirrors gnstk's layers API (proj/include/gnstk/layers.hpp:18-80) with the same
names, argument meaning, map keys ("gamma", "beta"), correction convention
(corrected = (sum_b raw / B) * B^2, raw kept per example) and error behaviour
(ValueError carrying the reference's "layers: ..." message where the
reference throws std::invalid_argument).  Tensors are torch CUDA tensors;
every computation runs in libgnsb.so (include/gnsb.h).  There is no CPU path.

Differences from the fp64 reference, by design:
  * rows may be fp32, bf16 or fp64; statistics are fp32 (fp64 for fp64 rows);
    norm outputs are fp64;
  * the forward additionally caches (x, mean) so the backward reads x once
    instead of a materialised xhat; a reference-style cache holding only
    (normalized, inv_std) is accepted too.
"""
from __future__ import annotations

import dataclasses
import threading
from typing import Dict, Optional

import torch

from . import _lib

_DT = {torch.float32: _lib.GNSB_F32, torch.bfloat16: _lib.GNSB_BF16, torch.float64: _lib.GNSB_F64}


def gnsb_dtype(t: torch.dtype) -> int:
    if t not in _DT:
        raise ValueError(f"layers: unsupported dtype {t}")
    return _DT[t]


def stat_dtype(t: torch.dtype) -> torch.dtype:
    return torch.float64 if t == torch.float64 else torch.float32


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else t.data_ptr()


def _stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


@dataclasses.dataclass
class LayerNormLayer:
    """gnstk::LayerNormLayer (layers.hpp:18-22)."""

    gamma: torch.Tensor
    beta: torch.Tensor
    epsilon: float = 1e-5


@dataclasses.dataclass
class LayerNormCache:
    """gnstk::LayerNormCache (layers.hpp:48-51) plus the B200 (x, mean) form."""

    normalized: Optional[torch.Tensor]  # xhat, same shape as the input (may be None)
    inv_std: torch.Tensor               # input shape without the trailing axis
    x: Optional[torch.Tensor] = None    # the input itself (B200 cache)
    mean: Optional[torch.Tensor] = None


@dataclasses.dataclass
class LayerNormForwardResult:
    output: torch.Tensor
    cache: LayerNormCache


@dataclasses.dataclass
class LayerGradOutput:
    """gnstk::LayerGradOutput (layers.hpp:36-41).

    per_example_sqnorms holds 0-dim fp64 device tensors (call float() to read);
    sums4 is the raw device record {sum raw_gamma, sum raw_beta, ||dgamma||^2,
    ||dbeta||^2} consumed by the device GNS accumulator.
    """

    weight_grads: Dict[str, torch.Tensor]
    per_example_sqnorms: Dict[str, torch.Tensor]
    per_example_sqnorms_raw: Dict[str, torch.Tensor]
    batch_size: int
    sums4: Optional[torch.Tensor] = None


@dataclasses.dataclass
class LayerNormBackwardResult:
    grads: LayerGradOutput
    input_grad: Optional[torch.Tensor]


class _Workspace:
    """Zero-initialised device workspace per (device, stream), grown on demand.

    The kernel leaves its counters zeroed after every call, so a workspace is
    reused without re-initialisation; distinct streams get distinct buffers.
    """

    def __init__(self):
        self._bufs = {}
        self._lock = threading.Lock()

    def get(self, device: torch.device, nbytes: int, op: str = "ln") -> torch.Tensor:
        # one buffer per (op, device, stream): the ops lay out their counters
        # differently, so a buffer is never shared between them
        key = (op, device.index, torch.cuda.current_stream(device).cuda_stream)
        with self._lock:
            buf = self._bufs.get(key)
            if buf is None or buf.numel() < nbytes:
                buf = torch.zeros(max(nbytes, 1 << 16), dtype=torch.uint8, device=device)
                self._bufs[key] = buf
            return buf


_WS = _Workspace()


def _bmk(shape) -> tuple:
    """(B, M, D) view of a rank >= 2 shape (proj/src/layers.cpp:19-28)."""
    if len(shape) < 2:
        raise ValueError("layers: expected rank >= 2")
    m = 1
    for e in shape[1:-1]:
        m *= int(e)
    return int(shape[0]), m, int(shape[-1])


def layernorm_forward(layer: LayerNormLayer, x: torch.Tensor, keep_normalized: bool = False) -> LayerNormForwardResult:
    """gnstk::layernorm_forward (proj/src/layers.cpp:189-229) on the GPU."""
    k = layer.gamma.numel()
    if layer.beta.shape != (k,):
        raise ValueError("layers: gamma/beta extent mismatch")
    if not layer.epsilon > 0.0:
        raise ValueError("layers: epsilon must be positive")
    if x.dim() < 1 or x.shape[-1] != k:
        raise ValueError("layers: input trailing extent does not match gamma")
    if k < 2:
        raise ValueError("layers: layernorm needs trailing extent >= 2")
    x = x.contiguous()
    sd = stat_dtype(x.dtype)
    gamma = layer.gamma.to(device=x.device, dtype=sd).contiguous()
    beta = layer.beta.to(device=x.device, dtype=sd).contiguous()
    rows = x.numel() // k
    y = torch.empty_like(x)
    mean = torch.empty(x.shape[:-1], dtype=sd, device=x.device)
    rstd = torch.empty(x.shape[:-1], dtype=sd, device=x.device)
    xhat = torch.empty_like(x) if keep_normalized else None
    _lib.check(
        _lib.lib().gnsb_ln_fwd(
            _ptr(x), _ptr(gamma), _ptr(beta), _ptr(y), _ptr(mean), _ptr(rstd), _ptr(xhat), rows, k,
            float(layer.epsilon), gnsb_dtype(x.dtype), _stream_ptr(x.device),
        )
    )
    return LayerNormForwardResult(y, LayerNormCache(normalized=xhat, inv_std=rstd, x=x, mean=mean))


def layernorm_backward_simultaneous(
    layer: LayerNormLayer,
    cache: LayerNormCache,
    g: torch.Tensor,
    with_norms: bool = True,
    need_input_grad: bool = True,
) -> LayerNormBackwardResult:
    """gnstk::layernorm_backward_simultaneous (proj/src/layers.cpp:231-298) on the GPU.

    One fused kernel: dx, dgamma, dbeta and the per-example ||dgamma_b||^2,
    ||dbeta_b||^2 (raw) plus corrected means.  with_norms=False runs the
    otherwise-identical plain LayerNorm backward.
    """
    k = layer.gamma.numel()
    src = cache.x if (cache.x is not None and cache.mean is not None) else cache.normalized
    if src is None:
        raise ValueError("layers: cache holds neither (x, mean) nor normalized")
    if tuple(src.shape) != tuple(g.shape):
        raise ValueError("layers: cache/gradient shape mismatch")
    if g.dim() < 2:
        raise ValueError("layers: backward expects a leading batch axis")
    B, M, D = _bmk(g.shape)
    if D != k:
        raise ValueError("layers: gradient trailing extent does not match gamma")
    if B == 0:
        raise ValueError("layers: empty batch")
    if g.dtype != src.dtype:
        raise ValueError("layers: gradient dtype must match the cached activations")
    dev = g.device
    sd = stat_dtype(g.dtype)
    g = g.contiguous()
    src = src.contiguous()
    mean = cache.mean.to(sd).contiguous() if src is cache.x else None
    rstd = cache.inv_std.to(sd).contiguous()
    gamma = layer.gamma.to(device=dev, dtype=sd).contiguous()
    dx = torch.empty_like(g) if need_input_grad else None
    dgamma = torch.empty(D, dtype=sd, device=dev)
    dbeta = torch.empty(D, dtype=sd, device=dev)
    raw_g = torch.zeros(B, dtype=torch.float64, device=dev) if with_norms else None
    raw_b = torch.zeros(B, dtype=torch.float64, device=dev) if with_norms else None
    sums = torch.zeros(4, dtype=torch.float64, device=dev) if with_norms else None
    dt = gnsb_dtype(g.dtype)
    nbytes = ctypes_size(B, M, D, dt)
    ws = _WS.get(dev, nbytes)
    _lib.check(
        _lib.lib().gnsb_ln_bwd(
            _ptr(src), _ptr(mean), _ptr(rstd), _ptr(g), _ptr(gamma), _ptr(dx), _ptr(dgamma), _ptr(dbeta),
            _ptr(raw_g), _ptr(raw_b), _ptr(sums), 1 if with_norms else 0, B, M, D, dt, _ptr(ws), ws.numel(),
            _stream_ptr(dev),
        )
    )
    per_ex, raw = {}, {}
    if with_norms:
        bd = float(B)
        # corrected_mean_sqnorm (layers.cpp:39-42): sum / B * B^2
        per_ex = {"gamma": sums[0] / bd * (bd * bd), "beta": sums[1] / bd * (bd * bd)}
        raw = {"gamma": raw_g, "beta": raw_b}
    grads = LayerGradOutput({"gamma": dgamma, "beta": dbeta}, per_ex, raw, B, sums)
    return LayerNormBackwardResult(grads, dx)


def ctypes_size(B: int, M: int, D: int, dt: int) -> int:
    import ctypes

    out = ctypes.c_size_t(0)
    _lib.check(_lib.lib().gnsb_ln_bwd_workspace_size(B, M, D, dt, ctypes.byref(out)))
    return int(out.value)


def ln_bwd_geometry(B: int, M: int, D: int, dtype: torch.dtype) -> dict:
    import ctypes

    g, t, s = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    _lib.check(_lib.lib().gnsb_ln_bwd_geometry(B, M, D, gnsb_dtype(dtype), ctypes.byref(g), ctypes.byref(t),
                                               ctypes.byref(s)))
    return {"grid": g.value, "threads": t.value, "stages": s.value}


def synth_ln(B: int, T: int, D: int, dtype: torch.dtype, device, b_offset: int = 0, B_div: Optional[int] = None,
             sigma: float = 0.3, stream0: int = 0):
    """Materialise the SURVEY §8(d) LayerNorm recipe on the device (bit-identical
    with the oracle's orc_synth_ln).  Returns (x, dy, gamma, beta)."""
    dev = torch.device(device)
    sd = stat_dtype(dtype)
    x = torch.empty(B, T, D, dtype=dtype, device=dev)
    dy = torch.empty(B, T, D, dtype=dtype, device=dev)
    gamma = torch.empty(D, dtype=sd, device=dev)
    beta = torch.empty(D, dtype=sd, device=dev)
    _lib.check(
        _lib.lib().gnsb_synth_ln(
            _ptr(x), _ptr(dy), _ptr(gamma), _ptr(beta), B, T, D, b_offset, B_div or B, float(sigma), stream0,
            gnsb_dtype(dtype), _stream_ptr(dev),
        )
    )
    return x, dy, gamma, beta


def synth_linear(B: int, T: int, K: int, L: int, dtype: torch.dtype, device, b_offset: int = 0,
                 B_div: Optional[int] = None, stream0: int = 10):
    dev = torch.device(device)
    x = torch.empty(B, T, K, dtype=dtype, device=dev)
    dy = torch.empty(B, T, L, dtype=dtype, device=dev)
    _lib.check(
        _lib.lib().gnsb_synth_linear(
            _ptr(x), _ptr(dy), B, T, K, L, b_offset, B_div or B, stream0, gnsb_dtype(dtype), _stream_ptr(dev)
        )
    )
    return x, dy


def sqnorm(v: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Deterministic fp64 ||v||^2 on the device (fp32/fp64 input)."""
    if out is None:
        out = torch.empty((), dtype=torch.float64, device=v.device)
    v = v.contiguous()
    _lib.check(_lib.lib().gnsb_sqnorm(_ptr(v), v.numel(), gnsb_dtype(v.dtype), _ptr(out), _stream_ptr(v.device)))
    return out


class PendingLayerNorm:
    """A LayerNorm whose row pass ran (dx is final) and whose stage 2 is
    deferred to `layernorm_backward_reduce` (gnsb_ln_bwd_rows / gnsb_ln_bwd_reduce).
    Holds its own workspace and the output tensors the reduce will fill."""

    def __init__(self, B, M, D, dt, ws, dgamma, dbeta, raw_g, raw_b, sums):
        self.B, self.M, self.D, self.dt = B, M, D, dt
        self.ws, self.dgamma, self.dbeta, self.raw_g, self.raw_b, self.sums = ws, dgamma, dbeta, raw_g, raw_b, sums

    def _c(self):
        return _lib.LnBwdPending(self.ws.data_ptr(), self.ws.numel(), self.B, self.M, self.D, self.dt,
                                 self.dgamma.data_ptr(), self.dbeta.data_ptr(), self.raw_g.data_ptr(),
                                 self.raw_b.data_ptr(), self.sums.data_ptr())

    def result(self, with_norms: bool = True) -> LayerGradOutput:
        per_ex, raw = {}, {}
        if with_norms:
            bd = float(self.B)
            per_ex = {"gamma": self.sums[0] / bd * (bd * bd), "beta": self.sums[1] / bd * (bd * bd)}
            raw = {"gamma": self.raw_g, "beta": self.raw_b}
        return LayerGradOutput({"gamma": self.dgamma, "beta": self.dbeta}, per_ex, raw, self.B, self.sums)


def layernorm_backward_rows(layer: LayerNormLayer, cache: LayerNormCache, g: torch.Tensor,
                            need_input_grad: bool = True, ws: Optional[torch.Tensor] = None):
    """Row pass of the fused backward: returns (dx, PendingLayerNorm).  The
    per-example combine, squares and dgamma/dbeta of any number of pending
    layers then run in one `layernorm_backward_reduce` launch."""
    k = layer.gamma.numel()
    src = cache.x if (cache.x is not None and cache.mean is not None) else cache.normalized
    if src is None:
        raise ValueError("layers: cache holds neither (x, mean) nor normalized")
    if tuple(src.shape) != tuple(g.shape):
        raise ValueError("layers: cache/gradient shape mismatch")
    B, M, D = _bmk(g.shape)
    if D != k:
        raise ValueError("layers: gradient trailing extent does not match gamma")
    if B == 0:
        raise ValueError("layers: empty batch")
    dev = g.device
    sd = stat_dtype(g.dtype)
    g = g.contiguous()
    src = src.contiguous()
    mean = cache.mean.to(sd).contiguous() if src is cache.x else None
    rstd = cache.inv_std.to(sd).contiguous()
    gamma = layer.gamma.to(device=dev, dtype=sd).contiguous()
    dx = torch.empty_like(g) if need_input_grad else None
    dt = gnsb_dtype(g.dtype)
    nbytes = ctypes_size(B, M, D, dt)
    if ws is None or ws.numel() < nbytes:
        # owned by the pending layer; a caller may pass one back for the next
        # step (the reduce leaves it zeroed, ready for reuse)
        ws = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
    _lib.check(_lib.lib().gnsb_ln_bwd_rows(_ptr(src), _ptr(mean), _ptr(rstd), _ptr(g), _ptr(gamma), _ptr(dx), B, M,
                                           D, dt, _ptr(ws), ws.numel(), _stream_ptr(dev)))
    pend = PendingLayerNorm(B, M, D, dt, ws, torch.empty(D, dtype=sd, device=dev), torch.empty(D, dtype=sd, device=dev),
                            torch.zeros(B, dtype=torch.float64, device=dev),
                            torch.zeros(B, dtype=torch.float64, device=dev),
                            torch.zeros(4, dtype=torch.float64, device=dev))
    return dx, pend


def layernorm_backward_reduce(pending, with_norms: bool = True):
    """Stage 2 of every pending layer in one launch; returns their LayerGradOutputs."""
    pending = list(pending)
    if not pending:
        return []
    arr = (_lib.LnBwdPending * len(pending))(*[p._c() for p in pending])
    dev = pending[0].ws.device
    _lib.check(_lib.lib().gnsb_ln_bwd_reduce(arr, len(pending), 1 if with_norms else 0, _stream_ptr(dev)))
    return [p.result(with_norms) for p in pending]
