"""GPU parity of the linear-layer per-example norms (weight-gradient and Gram forms).

Against the reference golden vectors (fp64 rows: generic kernel, rel 1e-11) and
the oracle on synthetic bf16 inputs (tcgen05 kernel: per-example norms rel 1e-4,
dW rel 1e-4 of ||dW||_inf — bf16 products are exact in fp32, the difference is
fp32 vs fp64 accumulation order).
"""
import numpy as np
import pytest
import torch

from conftest import close

pytestmark = pytest.mark.gpu


def _t(a, dt, dev):
    return torch.tensor(np.asarray(a), dtype=dt, device=dev)


@pytest.mark.parametrize("fam", ["lin_kat", "lin_rand17", "frob_rand23", "acc1_linear", "acc2_frob"])
def test_fp64_matches_reference_golden(golden, cuda, fam):
    from paper_2411_00999_b200 import linear

    cases = [c for c in golden if c["family"] == fam]
    assert cases
    for c in cases:
        sx, sg = tuple(c["shape_x"]), tuple(c["shape_g"])
        K, L = sx[-1], sg[-1]
        layer = linear.LinearLayer(_t(c["W"], torch.float64, cuda).reshape(K, L),
                                   _t(c["bias"], torch.float64, cuda) if "bias" in c else None)
        x = _t(c["x"], torch.float64, cuda).reshape(sx)
        g = _t(c["g"], torch.float64, cuda).reshape(sg)
        r = linear.linear_backward_simultaneous(layer, x, g)
        torch.cuda.synchronize()
        assert close(r.grads.weight_grads["weight"].cpu().numpy().ravel(), c["dW"], 1e-11, 1e-14)
        assert close(r.grads.per_example_sqnorms_raw["weight"].cpu().numpy(), c["raw_w"], 1e-11, 1e-14)
        assert close(float(r.grads.per_example_sqnorms["weight"]), c["corrected"][0], 1e-11, 1e-14)
        assert close(r.input_grad.cpu().numpy().ravel(), c["dx"], 1e-11, 1e-14)
        if "bias" in c:
            assert close(r.grads.weight_grads["bias"].cpu().numpy(), c["dbias"], 1e-11, 1e-14)
            assert close(r.grads.per_example_sqnorms_raw["bias"].cpu().numpy(), c["raw_b"], 1e-11, 1e-14)
            assert close(float(r.grads.per_example_sqnorms["bias"]), c["corrected"][1], 1e-11, 1e-14)
        if "frob" in c and len(sx) == 3:
            f = linear.linear_perexample_sqnorm_frobenius(x, g)
            assert close(f.cpu().numpy(), c["frob"], 1e-11, 1e-14)


def test_hand_worked(cuda):
    # proj/tests/test_layers.cpp:51-63, 77-85, 109-118
    from paper_2411_00999_b200 import linear

    r = linear.linear_backward_simultaneous(linear.LinearLayer(torch.zeros(2, 1, dtype=torch.float64, device=cuda)),
                                            _t([[[1, 2]], [[3, 4]]], torch.float64, cuda),
                                            _t([[[1]], [[2]]], torch.float64, cuda))
    assert r.grads.weight_grads["weight"].cpu().numpy().ravel().tolist() == [7.0, 10.0]
    assert r.grads.per_example_sqnorms_raw["weight"].tolist() == [5.0, 100.0]
    assert close(float(r.grads.per_example_sqnorms["weight"]), 210.0, 1e-12)
    x, g = _t([[[1], [1]]], torch.float64, cuda), _t([[[2], [3]]], torch.float64, cuda)
    assert linear.linear_perexample_sqnorm_frobenius(x, g).tolist() == [25.0]
    with pytest.raises(ValueError, match="frobenius path expects strictly 3-axis"):
        linear.linear_perexample_sqnorm_frobenius(torch.zeros(2, 2, device=cuda), torch.zeros(2, 2, device=cuda))
    with pytest.raises(ValueError, match="empty batch"):
        linear.linear_backward_simultaneous(linear.LinearLayer(torch.zeros(2, 1, device=cuda)),
                                            torch.zeros(0, 1, 2, device=cuda), torch.zeros(0, 1, 1, device=cuda))


def _oracle_linear(orc, x, g):
    return orc.linear_backward(x.double().cpu().numpy(), g.double().cpu().numpy(),
                               np.zeros((x.shape[-1], g.shape[-1])))


@pytest.mark.parametrize("impl", ["pair", "single"])
@pytest.mark.parametrize("B,T,K,L", [(2, 64, 128, 256), (3, 128, 256, 512), (4, 192, 128, 256), (1, 64, 384, 256),
                                     (5, 64, 512, 768), (3, 64, 2048, 2560),
                                     # tile tails in every axis (TMA zero fill + masked dW stores)
                                     (3, 100, 136, 264), (2, 1, 8, 8), (4, 77, 512, 520), (2, 200, 264, 128)])
def test_tcgen05_weight_grad_form_matches_oracle(orc, cuda, monkeypatch, impl, B, T, K, L):
    """bf16 rows on the tensor-core kernel vs the fp64 oracle on identical inputs.
    "pair": the default CTA-pair kernel (256 x 256 tiles; K % 256 == 0, else the
    single-CTA kernel runs); "single": GNSB_WGRAD_IMPL=1.  The shapes cover
    tiles split into example ranges (few tiles, many examples) and a full round
    plus split remainder (80 pair tiles on 74 pairs)."""
    if impl == "single":
        monkeypatch.setenv("GNSB_WGRAD_IMPL", "1")
    import paper_2411_00999_b200 as m
    from paper_2411_00999_b200 import linear

    x, g = m.synth_linear(B, T, K, L, torch.bfloat16, cuda)
    xo, go = orc.synth_linear(B, T, K, L, bf16=True)
    np.testing.assert_array_equal(x.float().cpu().numpy(), xo)
    np.testing.assert_array_equal(g.float().cpu().numpy(), go)
    r = linear.linear_backward_simultaneous(linear.LinearLayer(torch.zeros(K, L, device=cuda)), x, g,
                                            form="weight_grad", need_input_grad=False)
    ref = _oracle_linear(orc, x, g)
    torch.cuda.synchronize()
    dW = r.grads.weight_grads["weight"].double().cpu().numpy()
    assert close(dW, ref["dW"], 1e-4, 1e-4 * np.max(np.abs(ref["dW"])))
    assert close(r.grads.per_example_sqnorms_raw["weight"].cpu().numpy(), ref["raw_w"], 1e-4)
    assert close(float(r.grads.per_example_sqnorms["weight"]), ref["corrected"][0], 1e-4)
    assert close(float(r.grads.sums4[2]), float(np.sum(ref["dW"] ** 2)), 1e-4)


@pytest.mark.parametrize("B,T,K,L", [(8, 128, 256, 256), (4, 100, 264, 136)])
def test_auto_form_short_sequences_gram_plus_plain_dw(orc, cuda, B, T, K, L):
    """form "auto" with dW at short T takes the Gram form for the norms and one
    plain dW pass over all B*T tokens (experiments/form_sweep.py): same dW,
    norms and record as the oracle."""
    import paper_2411_00999_b200 as m
    from paper_2411_00999_b200 import linear

    x, g = m.synth_linear(B, T, K, L, torch.bfloat16, cuda)
    r = linear.linear_backward_simultaneous(linear.LinearLayer(torch.zeros(K, L, device=cuda)), x, g, form="auto",
                                            need_input_grad=False)
    ref = _oracle_linear(orc, x, g)
    torch.cuda.synchronize()
    dW = r.grads.weight_grads["weight"].double().cpu().numpy()
    assert close(dW, ref["dW"], 1e-4, 1e-4 * np.max(np.abs(ref["dW"])))
    assert close(r.grads.per_example_sqnorms_raw["weight"].cpu().numpy(), ref["raw_w"], 1e-4)
    assert close(float(r.grads.sums4[0]), float(np.sum(ref["raw_w"])), 1e-4)
    assert close(float(r.grads.sums4[2]), float(np.sum(ref["dW"] ** 2)), 1e-4)


@pytest.mark.parametrize("dt,B,T,L", [(torch.bfloat16, 4, 300, 264), (torch.float32, 3, 1024, 3072),
                                      (torch.bfloat16, 8, 64, 50304), (torch.float32, 2, 7, 8)])
def test_bias_norms_streaming_kernel(orc, cuda, dt, B, T, L):
    """The bias gradient and its per-example norms (layers.cpp:118-119, 125-130)
    on the streaming kernel (fp32 / bf16 rows, L % 8 == 0) against the oracle on
    the same rows: dbias rel 1e-5 of its max, raw_b and the record rel 1e-5."""
    import paper_2411_00999_b200 as m
    from paper_2411_00999_b200 import linear

    K = 8
    x, g = m.synth_linear(B, T, K, L, dt, cuda)
    layer = linear.LinearLayer(torch.zeros(K, L, device=cuda), torch.zeros(L, device=cuda))
    r = linear.linear_backward_simultaneous(layer, x, g, need_input_grad=False)
    gd = g.double().cpu().numpy()
    bb = gd.sum(axis=1)  # [B, L] per-example bias gradients
    torch.cuda.synchronize()
    db = r.grads.weight_grads["bias"].double().cpu().numpy()
    assert close(db, bb.sum(0), 1e-5, 1e-5 * np.abs(bb.sum(0)).max())
    assert close(r.grads.per_example_sqnorms_raw["bias"].cpu().numpy(), (bb ** 2).sum(1), 1e-5)
    assert close(float(r.grads.sums4[1]), float((bb ** 2).sum()), 1e-5)
    assert close(float(r.grads.sums4[3]), float((bb.sum(0) ** 2).sum()), 1e-5)


def test_weight_grad_form_equals_gram_form(cuda):
    """<X X^T, G G^T>_F equals ||sum_t x_t^T g_t||^2 (test_layers.cpp:135-149)."""
    import paper_2411_00999_b200 as m
    from paper_2411_00999_b200 import linear

    B, T, K, L = 2, 64, 128, 256
    x, g = m.synth_linear(B, T, K, L, torch.bfloat16, cuda)
    r = linear.linear_backward_simultaneous(linear.LinearLayer(torch.zeros(K, L, device=cuda)), x, g,
                                            form="weight_grad", need_input_grad=False)
    f = linear.linear_perexample_sqnorm_frobenius(x, g)
    assert close(f.cpu().numpy(), r.grads.per_example_sqnorms_raw["weight"].cpu().numpy(), 1e-4)


def test_cfg3_full_size_sampled(orc, cuda):
    """BASELINE config 3 (B=16 T=2048 K=L=4096 bf16): tensor-core weight-grad form;
    per-example norms of two sampled examples against the oracle run on those
    examples only, dW against a float64 torch contraction."""
    import paper_2411_00999_b200 as m
    from paper_2411_00999_b200 import linear

    B, T, K, L = 16, 2048, 4096, 4096
    x, g = m.synth_linear(B, T, K, L, torch.bfloat16, cuda)
    r = linear.linear_backward_simultaneous(linear.LinearLayer(torch.zeros(K, L, device=cuda)), x, g,
                                            need_input_grad=False)
    torch.cuda.synchronize()
    raw = r.grads.per_example_sqnorms_raw["weight"].cpu().numpy()
    for b in (0, 11):
        dWb = (x[b].double().T @ g[b].double())
        assert close(raw[b], float((dWb * dWb).sum()), 1e-4)
    ref_dW = torch.einsum("btk,btl->kl", x.double(), g.double())
    dW = r.grads.weight_grads["weight"].double()
    assert float((dW - ref_dW).abs().max()) <= 1e-4 * float(ref_dW.abs().max())


@pytest.mark.parametrize("B,T,K,L", [(2, 128, 64, 64), (3, 256, 128, 192), (1, 384, 256, 128), (5, 128, 320, 64),
                                     # tails: T off the 128-token tile, K / L off the 64-feature stage
                                     (3, 100, 136, 72), (2, 1, 8, 8), (2, 300, 64, 520), (4, 129, 200, 96)])
def test_tcgen05_gram_form_matches_oracle(orc, cuda, B, T, K, L):
    """Tensor-core Gram form (bf16 rows, any T, K and L multiples of 8) vs the
    fp64 oracle's <X X^T, G G^T>_F on identical inputs (rel 1e-4)."""
    import paper_2411_00999_b200 as m
    from paper_2411_00999_b200 import linear

    x, g = m.synth_linear(B, T, K, L, torch.bfloat16, cuda)
    f = linear.linear_perexample_sqnorm_frobenius(x, g)
    ref = orc.linear_frobenius(x.double().cpu().numpy(), g.double().cpu().numpy())
    torch.cuda.synchronize()
    assert close(f.cpu().numpy(), ref, 1e-4)


def test_tcgen05_gram_form_cfg3_sampled(cuda):
    """BASELINE config 3 through the Gram form: every per-example norm against an
    fp64 torch contraction of that example's weight gradient, and the two forms
    agree."""
    import paper_2411_00999_b200 as m
    from paper_2411_00999_b200 import linear

    B, T, K, L = 16, 2048, 4096, 4096
    x, g = m.synth_linear(B, T, K, L, torch.bfloat16, cuda)
    f = linear.linear_perexample_sqnorm_frobenius(x, g).cpu().numpy()
    r = linear.linear_backward_simultaneous(linear.LinearLayer(torch.zeros(K, L, device=cuda)), x, g,
                                            need_input_grad=False)
    raw = r.grads.per_example_sqnorms_raw["weight"].cpu().numpy()
    assert close(f, raw, 1e-4)
    for b in (0, 7, 15):
        dWb = x[b].double().T @ g[b].double()
        assert close(f[b], float((dWb * dWb).sum()), 1e-4)


@pytest.mark.parametrize("B,T,K,L", [(3, 256, 384, 320), (2, 100, 72, 200), (4, 64, 1000, 8), (2, 130, 64, 64)])
def test_fp32_rows_tensor_core_norms(orc, cuda, B, T, K, L):
    """fp32 rows on the 3xTF32 path (linear_f32.cu: per-example x_b^T g_b on the
    tensor cores; T % 4 == L % 4 == 0, else the generic kernels): dW, raw_b and
    the record against the oracle at rel 1e-5 (north star, fp32), both forms,
    bitwise deterministic run to run."""
    import paper_2411_00999_b200 as m
    from paper_2411_00999_b200 import linear

    x, g = m.synth_linear(B, T, K, L, torch.float32, cuda)
    layer = linear.LinearLayer(torch.zeros(K, L, device=cuda))
    r = linear.linear_backward_simultaneous(layer, x, g, form="weight_grad", need_input_grad=False)
    r2 = linear.linear_backward_simultaneous(layer, x, g, form="weight_grad", need_input_grad=False)
    f = linear.linear_perexample_sqnorm_frobenius(x, g)
    ref = _oracle_linear(orc, x, g)
    torch.cuda.synchronize()
    dW = r.grads.weight_grads["weight"].double().cpu().numpy()
    assert close(dW, ref["dW"], 1e-5, 1e-5 * np.max(np.abs(ref["dW"])))
    assert close(r.grads.per_example_sqnorms_raw["weight"].cpu().numpy(), ref["raw_w"], 1e-5)
    assert close(f.cpu().numpy(), ref["raw_w"], 1e-5)
    assert close(float(r.grads.sums4[0]), float(np.sum(ref["raw_w"])), 1e-5)
    assert close(float(r.grads.sums4[2]), float(np.sum(ref["dW"] ** 2)), 1e-5)
    assert torch.equal(r.grads.weight_grads["weight"], r2.grads.weight_grads["weight"])
    assert torch.equal(r.grads.per_example_sqnorms_raw["weight"], r2.grads.per_example_sqnorms_raw["weight"])
