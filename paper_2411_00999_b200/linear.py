"""Linear-layer per-example gradient norms on B200, mirroring the reference API.

Mirrors gnstk::linear_backward_simultaneous (proj/include/gnstk/layers.hpp:69,
proj/src/layers.cpp:80-157) and gnstk::linear_perexample_sqnorm_frobenius
(layers.hpp:74, layers.cpp:159-187): same names, map keys ("weight", "bias"),
correction convention and "layers: ..." errors.  Everything runs in libgnsb.so:
the tcgen05 tensor-core kernel for bf16 rows with tile-aligned shapes, a
generic fp64-accumulating CUDA kernel otherwise.
"""
from __future__ import annotations

import ctypes
import dataclasses
from typing import Optional

import torch

from . import _lib
from .layers import LayerGradOutput, _WS, _ptr, _stream_ptr, gnsb_dtype, stat_dtype

FORMS = {"auto": 0, "weight_grad": 1, "simultaneous": 1, "gram": 2, "frobenius": 2}


@dataclasses.dataclass
class LinearLayer:
    """gnstk::LinearLayer (layers.hpp:13-16): weight [K, L], optional bias [L]."""

    weight: torch.Tensor
    bias: Optional[torch.Tensor] = None


@dataclasses.dataclass
class LinearBackwardResult:
    grads: LayerGradOutput
    input_grad: Optional[torch.Tensor]


def _workspace_bytes(B, T, K, L, dt) -> int:
    out = ctypes.c_size_t(0)
    _lib.check(_lib.lib().gnsb_linear_pe_workspace_size(B, T, K, L, dt, ctypes.byref(out)))
    return int(out.value)


def _bmk(t: torch.Tensor):
    if t.dim() < 2:
        raise ValueError("layers: expected rank >= 2")
    m = 1
    for e in t.shape[1:-1]:
        m *= int(e)
    return int(t.shape[0]), m, int(t.shape[-1])


def linear_backward_simultaneous(layer: LinearLayer, x: torch.Tensor, g: torch.Tensor, form: str = "auto",
                                 need_input_grad: bool = True) -> LinearBackwardResult:
    """Weight (and bias) gradients plus corrected per-example squared norms.

    g must be the gradient of a mean-reduced loss over the B leading-axis
    examples (layers.hpp:66-69).  Middle axes are collapsed (layers.cpp:19-28).
    form: "auto" (default: the weight-gradient form, or for short sequences the
    Gram form for the norms plus one plain dW pass -- the same outputs,
    DESIGN §4) or "weight_grad" / "simultaneous" (always the weight-gradient
    kernel).  The norms-only Gram form is linear_perexample_sqnorm_frobenius.
    """
    K, L = int(layer.weight.shape[0]), int(layer.weight.shape[1])
    if x.dim() != g.dim():
        raise ValueError("layers: x and g rank mismatch")
    if tuple(x.shape[:-1]) != tuple(g.shape[:-1]):
        raise ValueError("layers: x and g leading shape mismatch")
    B, M, kx = _bmk(x)
    _, _, lg = _bmk(g)
    if kx != K:
        raise ValueError("layers: input trailing extent does not match weight rows")
    if lg != L:
        raise ValueError("layers: gradient trailing extent does not match weight columns")
    if B == 0:
        raise ValueError("layers: empty batch")
    if layer.bias is not None and tuple(layer.bias.shape) != (L,):
        raise ValueError("layers: bias extent does not match weight columns")
    dev = x.device
    dt = gnsb_dtype(x.dtype)
    sd = stat_dtype(x.dtype)
    x = x.contiguous()
    g = g.contiguous()
    dW = torch.empty(K, L, dtype=sd, device=dev)
    raw_w = torch.empty(B, dtype=torch.float64, device=dev)
    sums = torch.zeros(4, dtype=torch.float64, device=dev)
    nbytes = _workspace_bytes(B, M, K, L, dt)
    ws = _WS.get(dev, nbytes, "linear")
    h = _lib.lib()
    sp = _stream_ptr(dev)
    _lib.check(h.gnsb_linear_pe_norms(_ptr(x), _ptr(g), _ptr(dW), _ptr(raw_w), _ptr(sums), B, M, K, L, FORMS[form],
                                      dt, _ptr(ws), ws.numel(), sp))
    bd = float(B)
    weight_grads = {"weight": dW}
    per_ex = {"weight": sums[0] / bd * (bd * bd)}  # corrected_mean_sqnorm (layers.cpp:39-42)
    raw = {"weight": raw_w}
    if layer.bias is not None:
        db = torch.empty(L, dtype=sd, device=dev)
        raw_b = torch.empty(B, dtype=torch.float64, device=dev)
        ws2 = _WS.get(dev, _workspace_bytes(B, M, 1, L, dt), "linear_bias")
        _lib.check(h.gnsb_linear_bias_pe(_ptr(g), _ptr(db), _ptr(raw_b), _ptr(sums), B, M, L, dt, _ptr(ws2),
                                         ws2.numel(), sp))
        weight_grads["bias"] = db
        per_ex["bias"] = sums[1] / bd * (bd * bd)
        raw["bias"] = raw_b
    dx = None
    if need_input_grad:
        dx = torch.empty_like(x)
        linear_gemm("dx", g, layer.weight, None, dx, B * M, K, L)
    return LinearBackwardResult(LayerGradOutput(weight_grads, per_ex, raw, B, sums), dx)


def _weight_operand(W: torch.Tensor, rows_dtype: torch.dtype, dev) -> torch.Tensor:
    """W as the GEMM's weight operand: bf16 rows take bf16 or fp32 (master)
    weights as they are; fp32 / fp64 rows take weights of their own dtype."""
    W = W.to(device=dev)
    if rows_dtype == torch.bfloat16 and W.dtype in (torch.bfloat16, torch.float32):
        return W.contiguous()
    return W.to(rows_dtype).contiguous()


EPILOGUES = {"none": 0, "tanh": 1, "residual": 2, "dtanh": 3}


def linear_gemm(kind: str, a: torch.Tensor, W: torch.Tensor, bias: Optional[torch.Tensor], out: torch.Tensor,
                rows: int, K: int, L: int, epilogue: str = "none", aux: Optional[torch.Tensor] = None) -> torch.Tensor:
    """kind "fwd": out = a W (+ bias) (gnsb_linear_fwd); "dx": out = a W^T
    (gnsb_linear_dx).  bf16 rows run the tcgen05 GEMM (linear_gemm.cu).
    epilogue (gnsb_linear_gemm): "tanh" / "residual" (out = aux + v) on the
    forward, "dtanh" (out = v * (1 - aux^2)) on the input grad."""
    dev = a.device
    dt = gnsb_dtype(a.dtype)
    Wop = _weight_operand(W, a.dtype, dev)
    wdt = gnsb_dtype(Wop.dtype)
    n = ctypes.c_size_t()
    h = _lib.lib()
    _lib.check(h.gnsb_linear_gemm_workspace_size(K, L, dt, wdt, ctypes.byref(n)))
    ws = _WS.get(dev, n.value, "gemm") if n.value else None
    sp = _stream_ptr(dev)
    if epilogue != "none":
        b = None if (bias is None or kind != "fwd") else bias.to(device=dev, dtype=stat_dtype(a.dtype)).contiguous()
        _lib.check(h.gnsb_linear_gemm(0 if kind == "fwd" else 1, EPILOGUES[epilogue], _ptr(a), _ptr(Wop),
                                      None if b is None else _ptr(b), None if aux is None else _ptr(aux.contiguous()),
                                      _ptr(out), rows, K, L, dt, wdt, None if ws is None else _ptr(ws),
                                      0 if ws is None else ws.numel(), sp))
    elif kind == "fwd":
        b = None if bias is None else bias.to(device=dev, dtype=stat_dtype(a.dtype)).contiguous()
        _lib.check(h.gnsb_linear_fwd(_ptr(a), _ptr(Wop), None if b is None else _ptr(b), _ptr(out), rows, K, L, dt,
                                     wdt, None if ws is None else _ptr(ws), 0 if ws is None else ws.numel(), sp))
    else:
        _lib.check(h.gnsb_linear_dx(_ptr(a), _ptr(Wop), _ptr(out), rows, K, L, dt, wdt,
                                    None if ws is None else _ptr(ws), 0 if ws is None else ws.numel(), sp))
    return out


def linear_forward(layer: LinearLayer, x: torch.Tensor) -> torch.Tensor:
    """y = x W (+ bias), x [B, ..., K] -> [B, ..., L] (layers.hpp:64, layers.cpp:52-78)."""
    K, L = int(layer.weight.shape[0]), int(layer.weight.shape[1])
    if x.dim() < 2:
        raise ValueError("layers: expected rank >= 2")
    if int(x.shape[-1]) != K:
        raise ValueError("layers: input trailing extent does not match weight rows")
    if layer.bias is not None and tuple(layer.bias.shape) != (L,):
        raise ValueError("layers: bias extent does not match weight columns")
    if not x.is_cuda:
        raise RuntimeError("layers: the B200 path has no CPU fallback (input is on the CPU)")
    x = x.contiguous()
    rows = x.numel() // K if K else 0
    y = torch.empty(*x.shape[:-1], L, dtype=x.dtype, device=x.device)
    return linear_gemm("fwd", x, layer.weight, layer.bias, y, rows, K, L)


def linear_perexample_sqnorm_frobenius(x: torch.Tensor, g: torch.Tensor) -> torch.Tensor:
    """Per-example ||dW_b||_F^2 via <X_b X_b^T, G_b G_b^T>_F (layers.cpp:159-187).
    Strictly 3-axis inputs; returns B uncorrected fp64 values."""
    if x.dim() != 3 or g.dim() != 3:
        raise ValueError("layers: frobenius path expects strictly 3-axis inputs")
    if x.shape[0] != g.shape[0] or x.shape[1] != g.shape[1]:
        raise ValueError("layers: x and g leading shape mismatch")
    B, T, K = (int(v) for v in x.shape)
    L = int(g.shape[2])
    out = torch.empty(B, dtype=torch.float64, device=x.device)
    if B == 0:
        return out
    dt = gnsb_dtype(x.dtype)
    ws = _WS.get(x.device, _workspace_bytes(B, T, K, L, dt), "linear")
    _lib.check(_lib.lib().gnsb_linear_pe_norms(_ptr(x.contiguous()), _ptr(g.contiguous()), None, _ptr(out), None, B, T,
                                               K, L, 2, dt, _ptr(ws), ws.numel(), _stream_ptr(x.device)))
    return out
