"""GPU toy model over the three instrumented layer types.

The reference's residual MLP language model (proj/include/gnstk/model.hpp:14-31,
proj/src/model.cpp): embedding -> n_blocks x [LayerNorm -> linear -> tanh ->
linear + residual] -> LayerNorm -> linear head, next-token cross-entropy
(mean over tokens, mean over examples).  Here every layer's backward is the
B200 kernel that also yields its per-example squared gradient norms, exactly
what `model_backward` (proj/src/model.cpp:144-188) collects:

    LayerNormPE  -> gnsb_ln_fwd / gnsb_ln_bwd            (fused LN backward)
    LinearPE     -> gnsb_linear_fwd / gnsb_linear_dx for y and dx (tcgen05
                    GEMMs for bf16 rows), gnsb_linear_pe_norms for dW +
                    per-example norms (tcgen05 when bf16 and aligned),
                    gnsb_linear_bias_pe for the bias
    EmbeddingPE  -> gnsb_embedding_fwd / gnsb_embedding_pe

`ToyModelPE.forward_backward` runs the reference's run_forward +
model_backward sequence (proj/src/model.cpp:87-188) without autograd, every
step on the library's kernels: the tanh of fc1 and the residual add of fc2 are
fused into the forward GEMM epilogues, the tanh derivative into fc2's
input-grad GEMM, the softmax cross-entropy forward+backward is one kernel
(gnsb_xent), and every LayerNorm's stage 2 is deferred to one grouped reduce
at the end of the backward (gnsb_ln_bwd_rows / gnsb_ln_bwd_reduce).

After `loss.backward()` every layer holds a 4-double norm record
{sum_b raw(p0), sum_b raw(p1), ||grad p0||^2, ||grad p1||^2} (p0 = weight or
gamma, p1 = bias or beta); `GnsTracker` turns them into the PerExample GNS of
Trainer::step (proj/src/trainer.cpp:363-418) on the device.
"""
from __future__ import annotations

import ctypes
import math
from typing import List, Optional, Tuple

import torch

from . import _lib
from .layers import _WS, _ptr, _stream_ptr, gnsb_dtype, stat_dtype
from .nn import LayerNormPE


def _linear_norms(x: torch.Tensor, g: torch.Tensor, K: int, L: int, rec: torch.Tensor, has_bias: bool):
    """dW [K, L] (+ dbias [L]) and the per-example norms of one linear layer."""
    B = x.shape[0]
    M = x.numel() // (B * K)
    dt = gnsb_dtype(x.dtype)
    sd = stat_dtype(x.dtype)
    dev = x.device
    n = ctypes.c_size_t()
    _lib.check(_lib.lib().gnsb_linear_pe_workspace_size(B, M, K, L, dt, ctypes.byref(n)))
    ws = _WS.get(dev, n.value, "linear")
    dW = torch.empty(K, L, dtype=sd, device=dev)
    raw = torch.empty(2, B, dtype=torch.float64, device=dev)
    sp = _stream_ptr(dev)
    # form 0 (auto): the weight-gradient form, or Gram + one plain dW pass for short sequences
    _lib.check(_lib.lib().gnsb_linear_pe_norms(_ptr(x), _ptr(g), _ptr(dW), _ptr(raw[0]), _ptr(rec), B, M, K, L, 0, dt,
                                               _ptr(ws), ws.numel(), sp))
    db = None
    if has_bias:
        db = torch.empty(L, dtype=sd, device=dev)
        _lib.check(_lib.lib().gnsb_linear_pe_workspace_size(B, M, 1, L, dt, ctypes.byref(n)))
        ws2 = _WS.get(dev, n.value, "linear_bias")
        _lib.check(_lib.lib().gnsb_linear_bias_pe(_ptr(g), _ptr(db), _ptr(raw[1]), _ptr(rec), B, M, L, dt, _ptr(ws2),
                                                  ws2.numel(), sp))
    return dW, db, raw


class _LinearPEFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, weight, bias, module):
        if not x.is_cuda:
            raise RuntimeError("LinearPE: the B200 path has no CPU fallback (input is on the CPU)")
        from .linear import LinearLayer, linear_forward

        y = linear_forward(LinearLayer(weight.detach(), None if bias is None else bias.detach()), x)
        ctx.save_for_backward(x, weight)
        ctx.has_bias = bias is not None
        ctx.module = module
        return y

    @staticmethod
    def backward(ctx, g):
        x, weight = ctx.saved_tensors
        module = ctx.module
        g = g.contiguous().to(x.dtype)
        x = x.contiguous()
        K, L = weight.shape
        rec = torch.zeros(4, dtype=torch.float64, device=x.device)
        dW, db, raw = _linear_norms(x, g, K, L, rec, ctx.has_bias)
        dx = None
        if ctx.needs_input_grad[0]:
            from .linear import linear_gemm

            dx = torch.empty_like(x)
            linear_gemm("dx", g, weight.detach(), None, dx, x.numel() // K, K, L)
        module.norm_record = rec
        module.per_example_raw = {"weight": raw[0], "bias": raw[1]} if ctx.has_bias else {"weight": raw[0]}
        module.batch_size = x.shape[0]
        return dx, dW.to(weight.dtype), (db.to(weight.dtype) if db is not None else None), None


class LinearPE(torch.nn.Module):
    """y = x W + b with W [K, L] (the reference's layout, layers.hpp:13-16);
    the backward also yields per-example ||dW_b||^2, ||db_b||^2 (raw) in
    `per_example_raw` and the 4-double `norm_record`."""

    layer_type = "linear"

    def __init__(self, K: int, L: int, bias: bool = True, device=None, dtype=torch.float32):
        super().__init__()
        self.weight = torch.nn.Parameter(torch.zeros(K, L, device=device, dtype=dtype))
        self.bias = torch.nn.Parameter(torch.zeros(L, device=device, dtype=dtype)) if bias else None
        self.norm_record: Optional[torch.Tensor] = None
        self.per_example_raw = None
        self.batch_size = None

    def forward(self, x):
        return _LinearPEFunction.apply(x, self.weight, self.bias, self)


class _EmbeddingPEFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, ids, weight, module):
        if not ids.is_cuda:
            raise RuntimeError("EmbeddingPE: the B200 path has no CPU fallback (ids are on the CPU)")
        ctx.save_for_backward(ids)
        ctx.V = weight.shape[0]
        ctx.module = module
        from .embedding import embedding_forward

        return embedding_forward(weight.detach(), ids.reshape(-1), int(ids.shape[0]), int(ids.shape[1]))

    @staticmethod
    def backward(ctx, g):
        (ids,) = ctx.saved_tensors
        module = ctx.module
        from .embedding import embedding_backward_simultaneous

        r = embedding_backward_simultaneous(ids, g.contiguous(), ctx.V)
        module.norm_record = r.sums4
        module.per_example_raw = {"weight": r.per_example_sqnorms_raw["weight"]}
        module.batch_size = ids.shape[0]
        return None, r.weight_grads["weight"], None


class EmbeddingPE(torch.nn.Module):
    """Token embedding [V, D]; the backward yields per-example ||dE_b||^2."""

    layer_type = "embedding"

    def __init__(self, V: int, D: int, device=None, dtype=torch.float32):
        super().__init__()
        self.weight = torch.nn.Parameter(torch.zeros(V, D, device=device, dtype=dtype))
        self.norm_record = None
        self.per_example_raw = None
        self.batch_size = None

    def forward(self, ids):
        return _EmbeddingPEFunction.apply(ids, self.weight, self)


class ToyModelPE(torch.nn.Module):
    """proj/include/gnstk/model.hpp:14-31 on the GPU, initialised as
    make_toy_model (proj/src/model.cpp:30-55): Gaussian weights with std 1
    (embedding), 1/sqrt(D) (fc1, head), 1/sqrt(H) (fc2); zero biases; LN gamma 1,
    beta 0.  init="reference" draws them from the reference's own stream
    (GaussianStream(mix_seed(seed, "init")), same order), so the weights equal
    make_toy_model's bit for bit; init="torch" uses torch's generator.
    dtype: fp32 (default) or fp64 parameters and activations."""

    _INIT_TAG = 0x696E6974  # model.cpp:16

    def __init__(self, vocab: int, dim: int, hidden_multiplier: int, n_blocks: int, seed: int = 0, device=None,
                 dtype=torch.float32, init: str = "torch"):
        super().__init__()
        if vocab < 2 or dim < 2 or hidden_multiplier < 1 or n_blocks < 1:
            raise ValueError("model: invalid model dims")
        if init not in ("torch", "reference"):
            raise ValueError("model: init must be 'torch' or 'reference'")
        H = dim * hidden_multiplier
        self.embed = EmbeddingPE(vocab, dim, device=device, dtype=dtype)
        self.lns = torch.nn.ModuleList([LayerNormPE(dim, device=device, dtype=dtype) for _ in range(n_blocks)])
        self.fc1 = torch.nn.ModuleList([LinearPE(dim, H, device=device, dtype=dtype) for _ in range(n_blocks)])
        self.fc2 = torch.nn.ModuleList([LinearPE(H, dim, device=device, dtype=dtype) for _ in range(n_blocks)])
        self.final_ln = LayerNormPE(dim, device=device, dtype=dtype)
        self.head = LinearPE(dim, vocab, device=device, dtype=dtype)
        if init == "reference":
            from .data import GaussianStream, mix_seed

            g = GaussianStream(mix_seed(seed, self._INIT_TAG))

            def draw(shape, std):
                n = shape[0] * shape[1]
                return torch.from_numpy(std * g.draw(n)).reshape(shape)
        else:
            gen = torch.Generator(device="cpu").manual_seed(seed)

            def draw(shape, std):
                return torch.randn(*shape, generator=gen, dtype=torch.float64) * std
        with torch.no_grad():
            self.embed.weight.copy_(draw((vocab, dim), 1.0))
            for f1, f2 in zip(self.fc1, self.fc2):
                f1.weight.copy_(draw((dim, H), 1.0 / math.sqrt(dim)))
                f2.weight.copy_(draw((H, dim), 1.0 / math.sqrt(H)))
            self.head.weight.copy_(draw((dim, vocab), 1.0 / math.sqrt(dim)))

    def forward(self, ids: torch.Tensor) -> torch.Tensor:
        x = self.embed(ids)
        for ln, f1, f2 in zip(self.lns, self.fc1, self.fc2):
            x = x + f2(torch.tanh(f1(ln(x))))
        return self.head(self.final_ln(x))

    def loss(self, ids: torch.Tensor, targets: torch.Tensor) -> torch.Tensor:
        """Mean over examples of the per-example mean-token cross-entropy
        (proj/src/model.cpp:150-156: dlogits scaled by 1/(T*B))."""
        logits = self.forward(ids)
        B, T, V = logits.shape
        lg = logits.reshape(B * T, V)
        if lg.dtype != torch.float64:
            lg = lg.float()
        ce = torch.nn.functional.cross_entropy(lg, targets.reshape(-1).long(), reduction="none")
        return ce.reshape(B, T).mean(1).mean(0)

    @torch.no_grad()
    def forward_backward(self, ids: torch.Tensor, targets: torch.Tensor, loss_scale: float = 1.0,
                         rows_dtype: Optional[torch.dtype] = None, validate: bool = True) -> torch.Tensor:
        """The reference's model_backward (proj/src/model.cpp:144-188) on the
        library's kernels, no autograd: returns the loss (device fp64 scalar,
        mean over examples of the per-example mean-token cross-entropy times
        loss_scale), sets every parameter's .grad and every instrumented
        layer's norm record (the GnsTracker input).  rows_dtype: activation
        dtype (default: the parameter dtype; bf16 with fp32 parameters runs
        the tcgen05 GEMMs).  validate=False skips the host-side id range
        checks (no host synchronisation: the step can be graph-captured)."""
        from .embedding import embedding_backward_simultaneous, embedding_forward
        from .layers import (LayerNormCache, LayerNormLayer, layernorm_backward_reduce, layernorm_backward_rows,
                             layernorm_forward)
        from .linear import linear_gemm

        pdt = self.embed.weight.dtype
        adt = rows_dtype or pdt
        B, T = (int(v) for v in ids.shape)
        N = B * T
        D = self.embed.weight.shape[1]
        V = self.head.weight.shape[1]
        ids = ids.contiguous()
        targets = targets.to(torch.int32).contiguous()

        def lnl(ln):
            return LayerNormLayer(ln.weight, ln.bias, ln.eps)

        # bf16 rows with fp32 parameters: one bf16 operand copy of each weight
        # per step, shared by its forward and input-grad GEMMs
        wop = {}

        def wt(mod):
            if adt == torch.bfloat16 and mod.weight.dtype != torch.bfloat16:
                if mod not in wop:
                    wop[mod] = mod.weight.to(torch.bfloat16)
                return wop[mod]
            return mod.weight

        # ---- forward (model.cpp:87-109)
        x = embedding_forward(self.embed.weight.to(adt), ids.reshape(-1), B, T, validate=validate)
        saved = []
        for ln, f1, f2 in zip(self.lns, self.fc1, self.fc2):
            fr = layernorm_forward(lnl(ln), x)
            H = f1.weight.shape[1]
            a = torch.empty(B, T, H, dtype=adt, device=x.device)
            linear_gemm("fwd", fr.output, wt(f1), f1.bias, a, N, D, H, epilogue="tanh")
            xn = torch.empty_like(x)
            linear_gemm("fwd", a, wt(f2), f2.bias, xn, N, H, D, epilogue="residual", aux=x)
            saved.append((fr, a))
            x = xn
        ffr = layernorm_forward(lnl(self.final_ln), x)
        logits = torch.empty(B, T, V, dtype=adt, device=x.device)
        linear_gemm("fwd", ffr.output, wt(self.head), self.head.bias, logits, N, D, V)
        # ---- loss + dlogits (model.cpp:113-141, 150-156)
        upstream = loss_scale * (1.0 / T) / B
        dlogits = torch.empty_like(logits)
        loss_rows = torch.empty(N, dtype=torch.float64, device=x.device)
        _lib.check(_lib.lib().gnsb_xent(_ptr(logits), _ptr(targets), _ptr(dlogits), _ptr(loss_rows), N, V,
                                        float(upstream), gnsb_dtype(adt), None, _stream_ptr(x.device)))
        loss = (loss_rows.view(B, T).sum(1) / T * loss_scale).sum() / B
        # ---- backward (model.cpp:158-188)
        pend = []

        def linear_bw(mod, xin, g, epi_aux=None):
            K, L = mod.weight.shape
            rec = torch.zeros(4, dtype=torch.float64, device=g.device)
            dW, db, raw = _linear_norms(xin, g, K, L, rec, mod.bias is not None)
            mod.weight.grad = dW.to(mod.weight.dtype)
            if mod.bias is not None:
                mod.bias.grad = db.to(mod.bias.dtype)
            mod.norm_record, mod.batch_size = rec, B
            mod.per_example_raw = {"weight": raw[0], "bias": raw[1]} if mod.bias is not None else {"weight": raw[0]}
            dx = torch.empty(*g.shape[:-1], K, dtype=g.dtype, device=g.device)
            if epi_aux is None:
                linear_gemm("dx", g, wt(mod), None, dx, N, K, L)
            else:
                linear_gemm("dx", g, wt(mod), None, dx, N, K, L, epilogue="dtanh", aux=epi_aux)
            return dx

        def ln_bw(mod, fr, g):
            # the workspace of the layer's previous step is reused (the grouped
            # reduce leaves it zeroed)
            dx, p = layernorm_backward_rows(lnl(mod), fr.cache, g, ws=getattr(mod, "_rows_ws", None))
            mod._rows_ws = p.ws
            pend.append((mod, p))
            return dx

        dx = ln_bw(self.final_ln, ffr, linear_bw(self.head, ffr.output, dlogits))
        for i in reversed(range(len(self.lns))):
            fr, a = saved[i]
            da = linear_bw(self.fc2[i], a, dx, epi_aux=a)  # fc2 input grad times (1 - tanh^2), fused
            dh = linear_bw(self.fc1[i], fr.output, da)
            dx = dx + ln_bw(self.lns[i], fr, dh)
        r = embedding_backward_simultaneous(ids, dx, int(self.embed.weight.shape[0]), validate=validate)
        self.embed.weight.grad = r.weight_grads["weight"].to(pdt)
        self.embed.norm_record, self.embed.batch_size = r.sums4, B
        self.embed.per_example_raw = {"weight": r.per_example_sqnorms_raw["weight"]}
        outs = layernorm_backward_reduce([p for _, p in pend])  # every LayerNorm's stage 2, one launch
        for (mod, p), o in zip(pend, outs):
            mod.weight.grad = o.weight_grads["gamma"].to(mod.weight.dtype)
            mod.bias.grad = o.weight_grads["beta"].to(mod.bias.dtype)
            mod.norm_record, mod.batch_size = p.sums, B
            mod.per_example_raw = {"gamma": p.raw_g, "beta": p.raw_b}
        return loss

    def instrumented_layers(self) -> List[Tuple[str, torch.nn.Module]]:
        """Layers in the reference's LayerKey order of model_backward's output
        (proj/src/model.cpp:183-187): embed, then per block ln, fc1, fc2, then
        final_ln, head."""
        out = [("embed", self.embed)]
        for i, (ln, f1, f2) in enumerate(zip(self.lns, self.fc1, self.fc2)):
            out += [(f"block{i}.ln", ln), (f"block{i}.fc1", f1), (f"block{i}.fc2", f2)]
        out += [("final_ln", self.final_ln), ("head", self.head)]
        return out
