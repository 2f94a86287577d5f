"""GPU parity of the linear-layer GEMMs (linear_gemm.cu).

gnsb_linear_fwd (y = x W + bias, proj/src/layers.cpp:52-78) and gnsb_linear_dx
(dx = g W^T, layers.cpp:142-155) on the tcgen05 kernel, bf16 rows, against an
fp64 contraction of the same bf16 operands.  Tolerance: the output is rounded
to bf16, so rel 2^-8 with the close() atol rule 1e-5 * ||ref||_inf (fp32
accumulation order).  fp64 rows run the generic kernel and match the
reference order exactly (the golden dx vectors in test_linear_gpu.py).
Shapes cover tile tails in every axis (rows, K, L not multiples of the
128 x 256 x 64 tile) and the cfg3 size (B=16 T=2048 K=L=4096, sampled rows).
"""
import numpy as np
import pytest
import torch

from conftest import close

pytestmark = pytest.mark.gpu

RT = 2.0 ** -8


def _ref(kind, a, W, bias):
    a64, W64 = a.double(), W.double()
    y = a64 @ W64 if kind == "fwd" else a64 @ W64.t()
    if bias is not None:
        y = y + bias.double()
    return y


def _check(out, ref):
    o = out.double().cpu().numpy()
    r = ref.cpu().numpy()
    atol = 1e-5 * float(np.max(np.abs(r))) if r.size else 0.0
    assert close(o, r, RT, atol), float(np.max(np.abs(o - r)))


SHAPES = [(7, 8, 8), (128, 256, 256), (300, 136, 264), (1000, 520, 72), (257, 64, 1032), (2048, 1024, 4096),
          # split-K (few tiles, long reduction): dx of N = 264 over L = 8200, forward of N = 520 over K = 6000
          (1000, 264, 8200), (900, 6000, 520)]


@pytest.mark.parametrize("rows,K,L", SHAPES)
@pytest.mark.parametrize("wdt", [torch.float32, torch.bfloat16])
def test_forward_and_dx(cuda, rows, K, L, wdt):
    from paper_2411_00999_b200 import linear

    gen = torch.Generator(device="cpu").manual_seed(rows * 7 + K + L)
    x = torch.randn(rows, K, generator=gen).to(cuda, torch.bfloat16)
    g = torch.randn(rows, L, generator=gen).to(cuda, torch.bfloat16)
    W = (torch.randn(K, L, generator=gen) / K ** 0.5).to(cuda, wdt)
    bias = torch.randn(L, generator=gen).to(cuda)
    Wb = W.to(torch.bfloat16)  # the operand the tensor cores see
    for b in (None, bias):
        y = torch.empty(rows, L, dtype=torch.bfloat16, device=cuda)
        linear.linear_gemm("fwd", x, W, b, y, rows, K, L)
        torch.cuda.synchronize()
        _check(y, _ref("fwd", x, Wb, b))
    dx = torch.empty(rows, K, dtype=torch.bfloat16, device=cuda)
    linear.linear_gemm("dx", g, W, None, dx, rows, K, L)
    torch.cuda.synchronize()
    _check(dx, _ref("dx", g, Wb, None))


def test_linear_forward_api_rank3(cuda):
    from paper_2411_00999_b200 import linear

    gen = torch.Generator(device="cpu").manual_seed(5)
    x = torch.randn(3, 50, 96, generator=gen).to(cuda, torch.bfloat16)
    layer = linear.LinearLayer(torch.randn(96, 40, generator=gen).to(cuda), torch.randn(40, generator=gen).to(cuda))
    y = linear.linear_forward(layer, x)
    torch.cuda.synchronize()
    assert y.shape == (3, 50, 40)
    _check(y.reshape(150, 40), _ref("fwd", x.reshape(150, 96), layer.weight.to(torch.bfloat16), layer.bias))
    with pytest.raises(Exception, match="layers: input trailing extent does not match weight rows"):
        linear.linear_forward(layer, torch.zeros(2, 3, 95, device=cuda, dtype=torch.bfloat16))


def test_fp64_forward_is_reference_order(cuda):
    # proj/tests/test_layers.cpp:33-47 (exact values)
    from paper_2411_00999_b200 import linear

    t = lambda v, s: torch.tensor(v, dtype=torch.float64, device=cuda).reshape(s)
    assert linear.linear_forward(linear.LinearLayer(t([1, 1], (2, 1))), t([2, 3], (1, 2))).tolist() == [[5.0]]
    assert linear.linear_forward(linear.LinearLayer(t([1, 1], (2, 1)), t([7], (1,))), t([0, 0], (1, 2))).tolist() == [[7.0]]
    assert linear.linear_forward(linear.LinearLayer(t([1, 0, 0, 1], (2, 2))), t([3.5, -2.0], (1, 2))).tolist() == [[3.5, -2.0]]


def test_cfg3_input_grad(cuda):
    """cfg3 (B=16 T=2048 K=L=4096 bf16) through linear_backward_simultaneous with
    need_input_grad=True: dx of sampled rows against fp64, plus dW / norms
    unchanged by the dx launch."""
    import paper_2411_00999_b200 as m
    from paper_2411_00999_b200 import linear

    B, T, K, L = 16, 2048, 4096, 4096
    x, g = m.synth_linear(B, T, K, L, torch.bfloat16, cuda)
    gen = torch.Generator(device="cpu").manual_seed(3)
    W = (torch.randn(K, L, generator=gen) / K ** 0.5).to(cuda)
    r = linear.linear_backward_simultaneous(linear.LinearLayer(W), x, g, need_input_grad=True)
    torch.cuda.synchronize()
    rows = torch.tensor([0, 1, 2047, 2048, 13 * 2048 + 777, B * T - 1], device=cuda)
    g2 = g.reshape(B * T, L)[rows]
    ref = _ref("dx", g2, W.to(torch.bfloat16), None)
    _check(r.input_grad.reshape(B * T, K)[rows], ref)
    # and a full-tensor sanity check: no tile left unwritten (all finite, nonzero energy per row block)
    dxf = r.input_grad.reshape(B * T // 128, 128 * K).float()
    assert bool(torch.isfinite(dxf).all())
    assert bool((dxf.abs().sum(1) > 0).all())


def test_embedding_forward(cuda):
    import paper_2411_00999_b200 as m

    for dt in (torch.float32, torch.bfloat16, torch.float64):
        gen = torch.Generator(device="cpu").manual_seed(2)
        W = torch.randn(50, 24, generator=gen).to(cuda, dt)
        ids = torch.randint(0, 50, (3, 7), generator=gen, dtype=torch.int32).to(cuda)
        out = m.embedding_forward(W, ids.reshape(-1), 3, 7)
        torch.cuda.synchronize()
        assert torch.equal(out, W[ids.long()])
    with pytest.raises(ValueError, match="layers: id out of range"):
        m.embedding_forward(W, torch.tensor([0, 50], dtype=torch.int32, device=cuda), 1, 2)


F32_SHAPES = [(7, 4, 4), (128, 256, 256), (300, 132, 260), (1000, 516, 68), (4096, 1024, 2048)]


@pytest.mark.parametrize("rows,K,L", F32_SHAPES)
def test_fp32_rows_3xtf32(cuda, rows, K, L):
    """fp32 rows on the 3xTF32 tensor-core kernel (operands split into tf32
    hi + lo, lo*hi + hi*lo + hi*hi) against fp64 (forward with bias and the
    fused epilogues, and dx).  Tolerance rel 1e-5 with atol 5e-5 * ||ref||_inf:
    the split itself is good to ~2^-22, but the tensor core's fp32
    accumulation over the K-long reduction loses ~1e-5 of the largest partial
    sums at K ~ 500 (measured 1.3e-5), as any tensor-core fp32-accumulate GEMM
    does."""
    from paper_2411_00999_b200 import linear

    gen = torch.Generator(device="cpu").manual_seed(rows + 3 * K + 7 * L)
    x = torch.randn(rows, K, generator=gen).to(cuda)
    g = torch.randn(rows, L, generator=gen).to(cuda)
    W = (torch.randn(K, L, generator=gen) / K ** 0.5).to(cuda)
    bias = torch.randn(L, generator=gen).to(cuda)
    res = torch.randn(rows, L, generator=gen).to(cuda)

    def chk(out, ref, what):
        o, r = out.double().cpu().numpy(), ref.cpu().numpy()
        atol = 5e-5 * float(np.max(np.abs(r)))
        assert close(o, r, 1e-5, atol), (what, float(np.max(np.abs(o - r)) / max(float(np.max(np.abs(r))), 1e-300)))

    y = torch.empty(rows, L, device=cuda)
    linear.linear_gemm("fwd", x, W, bias, y, rows, K, L)
    torch.cuda.synchronize()
    chk(y, x.double() @ W.double() + bias.double(), "fwd+bias")
    linear.linear_gemm("fwd", x, W, bias, y, rows, K, L, epilogue="tanh")
    torch.cuda.synchronize()
    chk(y, torch.tanh(x.double() @ W.double() + bias.double()), "fwd tanh")
    linear.linear_gemm("fwd", x, W, None, y, rows, K, L, epilogue="residual", aux=res)
    torch.cuda.synchronize()
    chk(y, res.double() + x.double() @ W.double(), "fwd residual")
    dx = torch.empty(rows, K, device=cuda)
    linear.linear_gemm("dx", g, W, None, dx, rows, K, L)
    torch.cuda.synchronize()
    chk(dx, g.double() @ W.double().t(), "dx")
    z = torch.tanh(torch.randn(rows, K, generator=gen)).to(cuda)
    linear.linear_gemm("dx", g, W, None, dx, rows, K, L, epilogue="dtanh", aux=z)
    torch.cuda.synchronize()
    chk(dx, (g.double() @ W.double().t()) * (1 - z.double() ** 2), "dx dtanh")
