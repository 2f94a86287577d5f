"""PyTorch integration: a LayerNorm module whose backward is the fused B200
kernel and which stashes the per-example gradient norms for the GNS estimator.

This is how the paper deploys the kernel (nanoGPT with the custom LayerNorm,
PAPER.md:489-496, :618-623). The caller side it replaces is the reference's
`model_backward` loop (proj/src/model.cpp:144-188): every LayerNorm backward
also yields its parameters' per-example squared norms, and `Trainer::step`
(proj/src/trainer.cpp:363-418) turns them into GNS statistics.

    ln = LayerNormPE(768).cuda()
    y = ln(x)                      # x [B, T, 768] bf16/fp32, B = the batch (examples)
    loss.backward()                # loss must be a MEAN over the B examples
    rec = ln.norm_record           # fp64 [4]: {sum_b raw_gamma, sum_b raw_beta,
                                   #            ||dgamma||^2, ||dbeta||^2}
    GnsTracker([ln, ...]).step()   # device GNS estimate over every tracked layer

The forward is `gnsb_ln_fwd` (writes y, mean, rstd), the backward one
`gnsb_ln_bwd` call (row kernel + reduce kernel). There is no eager fallback:
without the CUDA extension the module raises.
"""
from __future__ import annotations

from typing import Iterable, Optional

import torch

from . import _lib
from .gns import DeviceGnsAccumulator
from .layers import _WS, _bmk, _ptr, _stream_ptr, ctypes_size, gnsb_dtype, stat_dtype


class _LayerNormPEFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, gamma, beta, eps, module):
        if not x.is_cuda:
            raise RuntimeError("LayerNormPE: the B200 path has no CPU fallback (input is on the CPU)")
        D = gamma.numel()
        x = x.contiguous()
        sd = stat_dtype(x.dtype)
        if gamma.dtype != sd or beta.dtype != sd:
            raise TypeError(f"LayerNormPE: gamma/beta must be {sd} for {x.dtype} rows")
        rows = x.numel() // D
        y = torch.empty_like(x)
        mean = torch.empty(x.shape[:-1], dtype=sd, device=x.device)
        rstd = torch.empty(x.shape[:-1], dtype=sd, device=x.device)
        _lib.check(_lib.lib().gnsb_ln_fwd(_ptr(x), _ptr(gamma), _ptr(beta), _ptr(y), _ptr(mean), _ptr(rstd), None,
                                          rows, D, float(eps), gnsb_dtype(x.dtype), _stream_ptr(x.device)))
        ctx.save_for_backward(x, mean, rstd, gamma)
        ctx.module = module
        return y

    @staticmethod
    def backward(ctx, dy):
        x, mean, rstd, gamma = ctx.saved_tensors
        module = ctx.module
        dy = dy.contiguous()
        if dy.dtype != x.dtype:
            dy = dy.to(x.dtype)
        B, M, D = _bmk(x.shape)
        dev = x.device
        sd = stat_dtype(x.dtype)
        need_dx = ctx.needs_input_grad[0]
        dx = torch.empty_like(x) if need_dx else None
        dgamma = torch.empty(D, dtype=sd, device=dev)
        dbeta = torch.empty(D, dtype=sd, device=dev)
        norms = module.track_norms
        raw = torch.empty(2, B, dtype=torch.float64, device=dev) if norms else None
        rec = torch.empty(4, dtype=torch.float64, device=dev) if norms else None
        dt = gnsb_dtype(x.dtype)
        ws = _WS.get(dev, ctypes_size(B, M, D, dt))
        _lib.check(_lib.lib().gnsb_ln_bwd(
            _ptr(x), _ptr(mean), _ptr(rstd), _ptr(dy), _ptr(gamma), _ptr(dx), _ptr(dgamma), _ptr(dbeta),
            _ptr(raw[0]) if norms else None, _ptr(raw[1]) if norms else None, _ptr(rec), 1 if norms else 0, B, M, D,
            dt, _ptr(ws), ws.numel(), _stream_ptr(dev)))
        if norms:
            module.norm_record = rec
            module.per_example_raw = {"gamma": raw[0], "beta": raw[1]}
            module.batch_size = B
        return dx, dgamma, dbeta, None, None


class LayerNormPE(torch.nn.Module):
    """LayerNorm over the last axis with per-example gradient norms.

    Inputs are [B, ..., D] with the leading axis the examples (the reference's
    bmk view, proj/src/layers.cpp:19-28). bf16 or fp32 rows; gamma/beta fp32.
    After each backward:
      norm_record      fp64 [4] device tensor: sum_b ||dgamma_b||^2,
                       sum_b ||dbeta_b||^2, ||dgamma||^2, ||dbeta||^2
                       (the `sums` record of gnsb_ln_bwd; corrected per-example
                       norm = record[i] * B, proj/src/layers.cpp:39-42)
      per_example_raw  {"gamma": [B], "beta": [B]} fp64 device tensors
    The per-example values are exact only for a loss that is a MEAN over the
    B examples.  dtype=torch.float64 gives fp64 gamma/beta for
    fp64 rows (the reference's own precision).
    """

    layer_type = "layernorm"

    def __init__(self, normalized_shape: int, eps: float = 1e-5, device=None, track_norms: bool = True,
                 dtype=torch.float32):
        super().__init__()
        if not eps > 0.0:
            raise ValueError("layers: epsilon must be positive")
        if normalized_shape < 2:
            raise ValueError("layers: layernorm needs trailing extent >= 2")
        self.normalized_shape = int(normalized_shape)
        self.eps = float(eps)
        if dtype not in (torch.float32, torch.float64):
            raise TypeError("LayerNormPE: gamma/beta are fp32 (bf16/fp32 rows) or fp64 (fp64 rows)")
        self.weight = torch.nn.Parameter(torch.ones(self.normalized_shape, dtype=dtype, device=device))
        self.bias = torch.nn.Parameter(torch.zeros(self.normalized_shape, dtype=dtype, device=device))
        self.track_norms = track_norms
        self.norm_record: Optional[torch.Tensor] = None
        self.per_example_raw: Optional[dict] = None
        self.batch_size: Optional[int] = None

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if x.shape[-1] != self.normalized_shape:
            raise ValueError("layers: input trailing extent does not match gamma")
        if x.dim() < 2:
            raise ValueError("layers: expected rank >= 2")
        return _LayerNormPEFunction.apply(x, self.weight, self.bias, self.eps, self)

    def extra_repr(self) -> str:
        return f"{self.normalized_shape}, eps={self.eps}, track_norms={self.track_norms}"


class GnsTracker:
    """Collects the norm records of tracked modules (LayerNormPE, and LinearPE /
    EmbeddingPE from model.py) after a backward and runs the device GNS step:
    the PerExample packaging of Trainer::step (proj/src/trainer.cpp:363-418):
    per layer g_big = ||grad p1||^2 + ||grad p0||^2, g_small = corrected(p1) +
    corrected(p0); groups {total, embedding, linear, layernorm} by each
    module's `layer_type`; EMA with `alpha`."""

    def __init__(self, modules: Iterable[torch.nn.Module], alpha: float = 1.0):
        self.modules = list(modules)
        if not self.modules:
            raise ValueError("gns: no layers to track")
        dev = next(self.modules[0].parameters()).device
        self.records = torch.zeros(len(self.modules), 4, dtype=torch.float64, device=dev)
        self.acc = DeviceGnsAccumulator([m.layer_type for m in self.modules], alpha, dev)

    def step(self):
        """Returns device tensors (groups [4, 4] {g2, s, gns_ema, defined}, layers [n, 2])."""
        B = None
        for m in self.modules:
            if m.norm_record is None:
                raise RuntimeError("gns: a tracked layer has no norm record (run backward first)")
            B = m.batch_size if B is None else B
            if m.batch_size != B:
                raise ValueError("gns: layers disagree on the batch size")
        torch.stack([m.norm_record for m in self.modules], out=self.records)  # one gather, not one copy per layer
        for m in self.modules:  # consumed: a layer without a backward next step must not reuse it
            m.norm_record = None
        return self.acc.step(self.records, B)
