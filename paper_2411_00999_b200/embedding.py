"""Embedding-table gradient with per-example squared norms (paper Alg. 3).

Mirrors gnstk::embedding_forward (proj/include/gnstk/layers.hpp:83,
proj/src/layers.cpp:300-313) over `gnsb_embedding_fwd` and
gnstk::embedding_backward_simultaneous (layers.hpp:85-88, layers.cpp:315-368)
over `gnsb_embedding_pe`.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from .layers import _WS, LayerGradOutput, _ptr, _stream_ptr, gnsb_dtype, stat_dtype


def embedding_backward_simultaneous(ids: torch.Tensor, g: torch.Tensor, vocab: int,
                                    validate: bool = True) -> LayerGradOutput:
    """ids [B, T] int32 (device), g [B, T, D] gradient of a mean-reduced loss.
    Returns weight grad [V, D] (fp32, fp64 for fp64 rows), the corrected
    per-example norm (B * sum_b raw) and the raw per-example norms [B]."""
    if g.dim() != 3:
        raise ValueError("layers: gradient shape mismatch")
    B, T, D = (int(v) for v in g.shape)
    if ids.numel() != B * T:
        raise ValueError("layers: id count does not match batch * t_len")
    if B == 0:
        raise ValueError("layers: empty batch")
    # layers.cpp:333 (a host round trip; validate=False skips it for ids valid
    # by construction -- out-of-range ids then only raise the kernel's bad flag)
    if validate and ids.numel() and (int(ids.min()) < 0 or int(ids.max()) >= vocab):
        raise ValueError("layers: id out of range")
    dev = g.device
    ids = ids.to(device=dev, dtype=torch.int32).contiguous()
    g = g.contiguous()
    dt = gnsb_dtype(g.dtype)
    sd = stat_dtype(g.dtype)
    n = ctypes.c_size_t()
    _lib.check(_lib.lib().gnsb_embedding_pe_workspace_size(B, T, vocab, D, dt, ctypes.byref(n)))
    ws = _WS.get(dev, n.value, "embedding")
    dW = torch.empty(vocab, D, dtype=sd, device=dev)
    raw = torch.empty(B, dtype=torch.float64, device=dev)
    sums = torch.zeros(4, dtype=torch.float64, device=dev)
    _lib.check(_lib.lib().gnsb_embedding_pe(_ptr(ids), _ptr(g), _ptr(dW), _ptr(raw), _ptr(sums), B, T, vocab, D, dt,
                                            _ptr(ws), ws.numel(), None, _stream_ptr(dev)))
    bd = float(B)
    return LayerGradOutput({"weight": dW}, {"weight": sums[0] / bd * (bd * bd)}, {"weight": raw}, B, sums)


def embedding_forward(weight: torch.Tensor, ids: torch.Tensor, batch: int, t_len: int,
                      validate: bool = True) -> torch.Tensor:
    """out[b, t, :] = weight[ids[b * t_len + t], :] (layers.cpp:300-313); [batch, t_len, D]."""
    if ids.numel() != batch * t_len:
        raise ValueError("layers: id count does not match batch * t_len")
    V, D = int(weight.shape[0]), int(weight.shape[1])
    if validate and ids.numel() and (int(ids.min()) < 0 or int(ids.max()) >= V):
        raise ValueError("layers: id out of range")
    if not weight.is_cuda:
        raise RuntimeError("layers: the B200 path has no CPU fallback (weights are on the CPU)")
    dev = weight.device
    ids = ids.to(device=dev, dtype=torch.int32).contiguous()
    w = weight.contiguous()
    out = torch.empty(batch, t_len, D, dtype=w.dtype, device=dev)
    _lib.check(_lib.lib().gnsb_embedding_fwd(_ptr(ids), _ptr(w), _ptr(out), batch * t_len, V, D, gnsb_dtype(w.dtype),
                                             None, _stream_ptr(dev)))
    return out
