"""GPU parity of the fused LayerNorm backward (+ per-example norms) and forward.

Every check compares the CUDA path (libgnsb.so through the C ABI) with the
reference: the golden vectors produced by the unmodified reference library
(tests/golden) and the oracle restatement (oracle/) on identical inputs.

Tolerances (BASELINE.json north_star / SURVEY §8(d)):
  fp64 rows : rtol 1e-11 (summation order differs from the sequential reference)
  fp32 rows : dx/dgamma/dbeta rtol 1e-5 with atol = 1e-5*||ref||_inf (test_helpers.hpp close());
              per-example norms and corrected values rtol 1e-4
  bf16 rows : the oracle consumes the same bf16 values; dx (bf16 output) rtol 2^-8 + atol 2^-8*||ref||_inf;
              dgamma/dbeta rtol 1e-4 (+1e-4*||ref||_inf); norms rtol 1e-4
"""
import numpy as np
import pytest
import torch

from conftest import close

pytestmark = pytest.mark.gpu

F32_TOL = 1e-5
NORM_TOL = 1e-4
BF16_DX = 2.0 ** -8


def _mod():
    import paper_2411_00999_b200 as m

    return m


def _t(a, dt, dev):
    return torch.tensor(np.asarray(a), dtype=dt, device=dev)


def _close_inf(got, ref, rtol, scale=None):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    s = np.max(np.abs(ref)) if scale is None else scale
    return close(got, ref, rtol, rtol * s)


# --------------------------------------------------------------------------- fp64 vs golden
@pytest.mark.parametrize("fam", ["ln_rand31", "acc1_ln", "ln_zero", "ln_fwd_kat"])
def test_fp64_backward_matches_reference_golden(golden, cuda, fam):
    m = _mod()
    cases = [c for c in golden if c["family"] == fam]
    assert cases
    for c in cases:
        shape = tuple(c["shape"])
        layer = m.LayerNormLayer(_t(c["gamma"], torch.float64, cuda), _t(c["beta"], torch.float64, cuda), c["eps"])
        cache = m.LayerNormCache(normalized=_t(c["xhat"], torch.float64, cuda).reshape(shape),
                                 inv_std=_t(c["inv_std"], torch.float64, cuda).reshape(shape[:-1]))
        r = m.layernorm_backward_simultaneous(layer, cache, _t(c["g"], torch.float64, cuda).reshape(shape))
        torch.cuda.synchronize()
        assert close(r.input_grad.cpu().numpy().ravel(), c["dx"], 1e-11, 1e-14), fam
        assert close(r.grads.weight_grads["gamma"].cpu().numpy(), c["dgamma"], 1e-11, 1e-14)
        assert close(r.grads.weight_grads["beta"].cpu().numpy(), c["dbeta"], 1e-11, 1e-14)
        assert close(r.grads.per_example_sqnorms_raw["gamma"].cpu().numpy(), c["raw_gamma"], 1e-11, 1e-14)
        assert close(r.grads.per_example_sqnorms_raw["beta"].cpu().numpy(), c["raw_beta"], 1e-11, 1e-14)
        assert close(float(r.grads.per_example_sqnorms["gamma"]), c["corrected"][0], 1e-11, 1e-14)
        assert close(float(r.grads.per_example_sqnorms["beta"]), c["corrected"][1], 1e-11, 1e-14)
        assert r.grads.batch_size == shape[0]


def test_fp64_hand_worked(cuda):
    # proj/tests/test_layers.cpp:167-176 — exact
    m = _mod()
    layer = m.LayerNormLayer(_t([1, 1], torch.float64, cuda), _t([0, 0], torch.float64, cuda), 1e-5)
    cache = m.LayerNormCache(normalized=_t([[[1, -1]]], torch.float64, cuda), inv_std=_t([[1.0]], torch.float64, cuda))
    r = m.layernorm_backward_simultaneous(layer, cache, _t([[[2, 3]]], torch.float64, cuda))
    assert r.grads.weight_grads["gamma"].tolist() == [2.0, -3.0]
    assert r.grads.weight_grads["beta"].tolist() == [2.0, 3.0]
    assert float(r.grads.per_example_sqnorms["gamma"]) == 13.0
    assert float(r.grads.per_example_sqnorms["beta"]) == 13.0


@pytest.mark.parametrize("fam", ["ln_rand31", "acc1_ln", "ln_fwd_kat"])
def test_fp64_forward_matches_reference_golden(golden, cuda, fam):
    m = _mod()
    for c in [c for c in golden if c["family"] == fam]:
        shape = tuple(c["shape"])
        layer = m.LayerNormLayer(_t(c["gamma"], torch.float64, cuda), _t(c["beta"], torch.float64, cuda), c["eps"])
        f = m.layernorm_forward(layer, _t(c["x"], torch.float64, cuda).reshape(shape), keep_normalized=True)
        assert close(f.output.cpu().numpy().ravel(), c["y"], 1e-11, 1e-13)
        assert close(f.cache.normalized.cpu().numpy().ravel(), c["xhat"], 1e-11, 1e-13)
        assert close(f.cache.inv_std.cpu().numpy().ravel(), c["inv_std"], 1e-11)


# --------------------------------------------------------------------------- fp32 cfg1 vs golden
def test_cfg1_fp32_matches_reference(golden, orc, cuda):
    """BASELINE config 1: B=8 T=128 D=768 fp32, synthetic recipe, vs the reference run."""
    m = _mod()
    c = [c for c in golden if c["family"] == "ln_cfg1"][0]
    B, T, D = c["shape"]
    x, dy, gamma, beta = m.synth_ln(B, T, D, torch.float32, cuda, sigma=c["sigma"], stream0=c["stream0"])
    xo, dyo, go, bo = orc.synth_ln(B, T, D, sigma=c["sigma"], stream0=c["stream0"])
    # the device generator is bit-identical with the oracle's
    np.testing.assert_array_equal(x.cpu().numpy(), xo)
    np.testing.assert_array_equal(dy.cpu().numpy(), dyo)
    np.testing.assert_array_equal(gamma.cpu().numpy(), go)
    np.testing.assert_array_equal(beta.cpu().numpy(), bo)

    layer = m.LayerNormLayer(gamma, beta, 1e-5)
    f = m.layernorm_forward(layer, x)
    assert _close_inf(f.cache.inv_std.cpu().numpy().ravel(), c["inv_std"], F32_TOL)
    idx = np.array(c["dx_sample_idx"], dtype=np.int64)
    assert _close_inf(f.output.cpu().numpy().ravel()[idx], c["y_sample"], F32_TOL)
    r = m.layernorm_backward_simultaneous(layer, f.cache, dy)
    torch.cuda.synchronize()
    assert _close_inf(r.grads.weight_grads["gamma"].cpu().numpy(), c["dgamma"], F32_TOL)
    assert _close_inf(r.grads.weight_grads["beta"].cpu().numpy(), c["dbeta"], F32_TOL)
    assert close(r.grads.per_example_sqnorms_raw["gamma"].cpu().numpy(), c["raw_gamma"], NORM_TOL)
    assert close(r.grads.per_example_sqnorms_raw["beta"].cpu().numpy(), c["raw_beta"], NORM_TOL)
    assert close(float(r.grads.per_example_sqnorms["gamma"]), c["corrected"][0], NORM_TOL)
    assert close(float(r.grads.per_example_sqnorms["beta"]), c["corrected"][1], NORM_TOL)
    dx = r.input_grad.cpu().numpy().ravel()
    scale = np.max(np.abs(c["dx_sample"]))
    assert close(dx[idx], c["dx_sample"], F32_TOL, F32_TOL * scale)
    assert close(dx.reshape(B * T, D).astype(np.float64).sum(1), c["dx_row_sum"], F32_TOL, F32_TOL * scale * 10)


def _oracle_on_device_stats(orc, x, dy, gamma, mean, rstd):
    """Reference backward on the same (x, mean, rstd) the kernel consumed."""
    return orc.ln_backward(x.cpu().double().numpy(), rstd.cpu().double().numpy(), dy.cpu().double().numpy(),
                           gamma.cpu().double().numpy(), mean=mean.cpu().double().numpy())


@pytest.mark.parametrize(
    "dt,B,T,D",
    [
        (torch.float32, 8, 128, 768),
        (torch.float32, 3, 5, 6),
        (torch.float32, 4, 7, 5),      # unaligned rows: non-TMA producer
        (torch.float32, 2, 33, 1024),
        (torch.float32, 5, 9, 4096),
        (torch.float32, 2, 4, 8192),
        (torch.bfloat16, 4, 64, 768),
        (torch.bfloat16, 4, 64, 1024),
        (torch.bfloat16, 3, 50, 2048),
        (torch.bfloat16, 2, 40, 4096),
        (torch.bfloat16, 2, 20, 8192),
        (torch.bfloat16, 2, 9, 16384),
        (torch.bfloat16, 3, 5, 13),    # unaligned
        (torch.float64, 3, 17, 2048),
        (torch.float64, 2, 5, 7),      # unaligned
        (torch.float32, 300, 1, 64),   # many examples per CTA
        (torch.float32, 1, 1000, 256), # one example spread over every CTA
        (torch.bfloat16, 1, 3, 8),     # fewer rows than SMs
    ],
)
def test_backward_matches_oracle(orc, cuda, dt, B, T, D):
    m = _mod()
    bf = dt == torch.bfloat16
    x, dy, gamma, beta = m.synth_ln(B, T, D, dt, cuda, stream0=7)
    xo, dyo, _, _ = orc.synth_ln(B, T, D, stream0=7, bf16=bf)
    np.testing.assert_array_equal(x.float().cpu().numpy(), xo)
    np.testing.assert_array_equal(dy.float().cpu().numpy(), dyo)
    layer = m.LayerNormLayer(gamma, beta, 1e-5)
    f = m.layernorm_forward(layer, x)
    r = m.layernorm_backward_simultaneous(layer, f.cache, dy)
    ref = _oracle_on_device_stats(orc, x, dy, gamma, f.cache.mean, f.cache.inv_std)
    torch.cuda.synchronize()
    dxt = {torch.float64: 1e-11, torch.float32: F32_TOL, torch.bfloat16: BF16_DX}[dt]
    gt = {torch.float64: 1e-11, torch.float32: F32_TOL, torch.bfloat16: NORM_TOL}[dt]
    nt = {torch.float64: 1e-11, torch.float32: NORM_TOL, torch.bfloat16: NORM_TOL}[dt]
    assert _close_inf(r.input_grad.double().cpu().numpy(), ref["dx"], dxt)
    assert _close_inf(r.grads.weight_grads["gamma"].double().cpu().numpy(), ref["dgamma"], gt)
    assert _close_inf(r.grads.weight_grads["beta"].double().cpu().numpy(), ref["dbeta"], gt)
    assert close(r.grads.per_example_sqnorms_raw["gamma"].cpu().numpy(), ref["raw_gamma"], nt)
    assert close(r.grads.per_example_sqnorms_raw["beta"].cpu().numpy(), ref["raw_beta"], nt)
    assert close(float(r.grads.per_example_sqnorms["gamma"]), ref["corrected"][0], nt)
    assert close(float(r.grads.per_example_sqnorms["beta"]), ref["corrected"][1], nt)
    # ||dgamma||^2, ||dbeta||^2 records (used by the GNS accumulator)
    s = r.grads.sums4.cpu().numpy()
    dg = r.grads.weight_grads["gamma"].double().cpu().numpy()
    db = r.grads.weight_grads["beta"].double().cpu().numpy()
    assert close(s[2], np.dot(dg, dg), 1e-12) and close(s[3], np.dot(db, db), 1e-12)


@pytest.mark.parametrize("dt,D", [(torch.bfloat16, 4096), (torch.float32, 768), (torch.float64, 6), (torch.bfloat16, 5)])
def test_plain_equals_fused(cuda, dt, D):
    """The plain LN backward runs the same kernels over one example of B*M rows:
    identical dx (same row math), dgamma/dbeta equal up to the summation order
    over examples (fp32 accumulation: 1e-5 relative; fp64: 1e-12)."""
    m = _mod()
    x, dy, gamma, beta = m.synth_ln(4, 100, D, dt, cuda, stream0=3)
    layer = m.LayerNormLayer(gamma, beta)
    f = m.layernorm_forward(layer, x)
    a = m.layernorm_backward_simultaneous(layer, f.cache, dy, with_norms=True)
    b = m.layernorm_backward_simultaneous(layer, f.cache, dy, with_norms=False)
    assert torch.equal(a.input_grad, b.input_grad)
    tol = 1e-12 if dt == torch.float64 else 1e-5
    for k in ("gamma", "beta"):
        ga, gb = a.grads.weight_grads[k].double().cpu().numpy(), b.grads.weight_grads[k].double().cpu().numpy()
        assert close(gb, ga, tol), k
    assert b.grads.per_example_sqnorms == {}


@pytest.mark.parametrize("B,T,D", [(1, 32768, 8192), (2, 8192, 4096), (1, 4096, 768)])
def test_grouped_reduce_one_example_many_ctas(cuda, B, T, D):
    """Stage 2 when one example spans more row CTAs than fit its shared-memory
    stage (B = 1 over many rows, several layers sharing the reduce grid): the
    example's slots are staged in chunks, summed in the same fixed order."""
    m = _mod()
    from paper_2411_00999_b200 import _lib
    x, dy, gamma, beta = m.synth_ln(B, T, D, torch.bfloat16, cuda, stream0=9)
    layer = m.LayerNormLayer(gamma, beta)
    f = m.layernorm_forward(layer, x)
    ref = m.layernorm_backward_simultaneous(layer, f.cache, dy, with_norms=True)
    NL = 6
    nb = m.layers.ctypes_size(B, T, D, 1)
    ws = [torch.zeros(nb, dtype=torch.uint8, device=cuda) for _ in range(NL)]
    outs = [(torch.empty(D, device=cuda), torch.empty(D, device=cuda), torch.zeros(B, dtype=torch.float64, device=cuda),
             torch.zeros(B, dtype=torch.float64, device=cuda), torch.zeros(4, dtype=torch.float64, device=cuda))
            for _ in range(NL)]
    dx = torch.empty_like(x)
    lib = _lib.lib()
    sp = torch.cuda.current_stream(cuda).cuda_stream
    for l in range(NL):
        _lib.check(lib.gnsb_ln_bwd_rows(x.data_ptr(), f.cache.mean.data_ptr(), f.cache.inv_std.data_ptr(),
                                        dy.data_ptr(), gamma.data_ptr(), dx.data_ptr(), B, T, D, 1,
                                        ws[l].data_ptr(), nb, sp))
    pend = (_lib.LnBwdPending * NL)(*[_lib.LnBwdPending(ws[l].data_ptr(), nb, B, T, D, 1, *[o.data_ptr() for o in outs[l]])
                                       for l in range(NL)])
    _lib.check(lib.gnsb_ln_bwd_reduce(pend, NL, 1, sp))
    torch.cuda.synchronize()
    for dg, db, rg, rb, sums in outs:
        assert close(dg.double().cpu().numpy(), ref.grads.weight_grads["gamma"].double().cpu().numpy(), 1e-6)
        assert close(db.double().cpu().numpy(), ref.grads.weight_grads["beta"].double().cpu().numpy(), 1e-6)
        assert close(rg.cpu().numpy(), ref.grads.per_example_sqnorms_raw["gamma"].cpu().numpy(), 1e-9)
        assert close(rb.cpu().numpy(), ref.grads.per_example_sqnorms_raw["beta"].cpu().numpy(), 1e-9)


@pytest.mark.parametrize("dt,B,T,D", [(torch.bfloat16, 32, 256, 4096), (torch.float32, 7, 33, 768)])
def test_deterministic_run_to_run(cuda, dt, B, T, D):
    m = _mod()
    x, dy, gamma, beta = m.synth_ln(B, T, D, dt, cuda, stream0=5)
    layer = m.LayerNormLayer(gamma, beta)
    f = m.layernorm_forward(layer, x)
    outs = [m.layernorm_backward_simultaneous(layer, f.cache, dy) for _ in range(3)]
    for o in outs[1:]:
        assert torch.equal(o.input_grad, outs[0].input_grad)
        assert torch.equal(o.grads.weight_grads["gamma"], outs[0].grads.weight_grads["gamma"])
        assert torch.equal(o.grads.per_example_sqnorms_raw["gamma"], outs[0].grads.per_example_sqnorms_raw["gamma"])
        assert torch.equal(o.grads.sums4, outs[0].grads.sums4)


def test_rank2_and_rank4_views(orc, cuda):
    """(B, M, D) view: rank-2 input has M = 1; rank-4 collapses middle axes (layers.cpp:19-28)."""
    m = _mod()
    for shape in [(6, 32), (2, 3, 4, 16)]:
        B, D = shape[0], shape[-1]
        M = int(np.prod(shape[1:-1])) if len(shape) > 2 else 1
        x, dy, gamma, beta = m.synth_ln(B, M, D, torch.float32, cuda, stream0=11)
        x = x.reshape(shape)
        dy = dy.reshape(shape)
        layer = m.LayerNormLayer(gamma, beta)
        f = m.layernorm_forward(layer, x)
        r = m.layernorm_backward_simultaneous(layer, f.cache, dy)
        ref = _oracle_on_device_stats(orc, x.reshape(B, M, D), dy.reshape(B, M, D), gamma, f.cache.mean.reshape(B, M),
                                      f.cache.inv_std.reshape(B, M))
        assert r.input_grad.shape == shape
        assert close(r.grads.per_example_sqnorms_raw["gamma"].cpu().numpy(), ref["raw_gamma"], NORM_TOL)
        assert _close_inf(r.input_grad.reshape(B, M, D).double().cpu().numpy(), ref["dx"], F32_TOL)


def test_empty_middle_axis_and_errors(cuda):
    m = _mod()
    layer = m.LayerNormLayer(torch.ones(8, device=cuda), torch.zeros(8, device=cuda))
    cache = m.LayerNormCache(normalized=torch.empty(3, 0, 8, device=cuda), inv_std=torch.empty(3, 0, device=cuda))
    r = m.layernorm_backward_simultaneous(layer, cache, torch.empty(3, 0, 8, device=cuda))
    assert r.grads.weight_grads["gamma"].abs().sum().item() == 0
    assert r.grads.per_example_sqnorms_raw["gamma"].tolist() == [0.0, 0.0, 0.0]
    assert float(r.grads.per_example_sqnorms["beta"]) == 0.0
    with pytest.raises(ValueError, match="layers: empty batch"):
        m.layernorm_backward_simultaneous(
            layer, m.LayerNormCache(torch.empty(0, 2, 8, device=cuda), torch.empty(0, 2, device=cuda)),
            torch.empty(0, 2, 8, device=cuda))
    with pytest.raises(ValueError, match="layers: cache/gradient shape mismatch"):
        m.layernorm_backward_simultaneous(
            layer, m.LayerNormCache(torch.zeros(2, 3, 8, device=cuda), torch.ones(2, 3, device=cuda)),
            torch.zeros(2, 3, 9, device=cuda))
    with pytest.raises(ValueError, match="layers: epsilon must be positive"):
        m.layernorm_forward(m.LayerNormLayer(torch.ones(8, device=cuda), torch.zeros(8, device=cuda), 0.0),
                            torch.zeros(2, 8, device=cuda))
    # zero upstream gradient -> zero norms and zero dx (test_layers.cpp:178-188)
    x = torch.randn(2, 3, 8, device=cuda)
    f = m.layernorm_forward(layer, x)
    r = m.layernorm_backward_simultaneous(layer, f.cache, torch.zeros_like(x))
    assert float(r.grads.per_example_sqnorms["gamma"]) == 0.0 and r.input_grad.abs().sum().item() == 0.0


def test_scaling_gradient_scales_norms_quadratically(cuda):
    # proj/tests/test_layers.cpp:349-362 analogue for LN: g*2 -> norms*4 exactly (fp64 rows)
    m = _mod()
    x, dy, gamma, beta = m.synth_ln(3, 10, 64, torch.float64, cuda, stream0=2)
    layer = m.LayerNormLayer(gamma, beta)
    f = m.layernorm_forward(layer, x)
    a = m.layernorm_backward_simultaneous(layer, f.cache, dy)
    b = m.layernorm_backward_simultaneous(layer, f.cache, dy * 2)
    assert float(b.grads.per_example_sqnorms["gamma"]) == 4 * float(a.grads.per_example_sqnorms["gamma"])
    assert float(b.grads.per_example_sqnorms["beta"]) == 4 * float(a.grads.per_example_sqnorms["beta"])


def test_cfg2_full_size_properties(orc, cuda):
    """BASELINE config 2 at full size (B=32 T=1024 D=4096 bf16): sampled examples
    against the oracle (per-example quantities depend on that example only),
    and dgamma/dbeta against an fp64 per-example sum of all examples."""
    m = _mod()
    B, T, D = 32, 1024, 4096
    x, dy, gamma, beta = m.synth_ln(B, T, D, torch.bfloat16, cuda)
    layer = m.LayerNormLayer(gamma, beta)
    f = m.layernorm_forward(layer, x)
    r = m.layernorm_backward_simultaneous(layer, f.cache, dy)
    torch.cuda.synchronize()
    rg = r.grads.per_example_sqnorms_raw["gamma"].cpu().numpy()
    rb = r.grads.per_example_sqnorms_raw["beta"].cpu().numpy()
    for b in (0, 13, 31):
        ref = _oracle_on_device_stats(orc, x[b:b + 1], dy[b:b + 1], gamma, f.cache.mean[b:b + 1],
                                      f.cache.inv_std[b:b + 1])
        assert close(rg[b], ref["raw_gamma"][0], NORM_TOL)
        assert close(rb[b], ref["raw_beta"][0], NORM_TOL)
        assert _close_inf(r.input_grad[b].double().cpu().numpy(), ref["dx"][0], BF16_DX)
    # batch sums: dgamma = sum_b gamma'_b, computed in fp64 on the GPU by torch as an independent check
    xh = (x.double() - f.cache.mean.double()[..., None]) * f.cache.inv_std.double()[..., None]
    ref_dg = (xh * dy.double()).sum((0, 1)).cpu().numpy()
    ref_db = dy.double().sum((0, 1)).cpu().numpy()
    pg = (xh * dy.double()).sum(1)
    ref_raw = (pg * pg).sum(1).cpu().numpy()
    assert _close_inf(r.grads.weight_grads["gamma"].double().cpu().numpy(), ref_dg, NORM_TOL)
    assert _close_inf(r.grads.weight_grads["beta"].double().cpu().numpy(), ref_db, NORM_TOL)
    assert close(rg, ref_raw, NORM_TOL)
    assert close(float(r.grads.per_example_sqnorms["gamma"]), B * ref_raw.sum(), NORM_TOL)


def test_two_streams_distinct_workspaces(cuda):
    m = _mod()
    x, dy, gamma, beta = m.synth_ln(8, 256, 1024, torch.bfloat16, cuda, stream0=9)
    layer = m.LayerNormLayer(gamma, beta)
    f = m.layernorm_forward(layer, x)
    base = m.layernorm_backward_simultaneous(layer, f.cache, dy)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    outs = []
    for s in (s1, s2, s1, s2):
        with torch.cuda.stream(s):
            outs.append(m.layernorm_backward_simultaneous(layer, f.cache, dy))
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o.input_grad, base.input_grad)
        assert torch.equal(o.grads.sums4, base.grads.sums4)


def test_deferred_grouped_reduce_matches_per_layer(cuda):
    """gnsb_ln_bwd_rows for several LayerNorms + one gnsb_ln_bwd_reduce equals
    per-layer gnsb_ln_bwd: dx and dgamma/dbeta bitwise (same kernels, same
    per-column order), norm records to 1e-12 (the per-example squares are
    summed over different column ranges)."""
    m = _mod()
    from paper_2411_00999_b200 import layers

    shapes = [(torch.bfloat16, 4, 96, 768), (torch.bfloat16, 3, 70, 4096), (torch.float32, 5, 33, 1024),
              (torch.bfloat16, 2, 8, 13)]
    pend, ref, dxs = [], [], []
    for i, (dt, B, T, D) in enumerate(shapes):
        x, dy, gamma, beta = m.synth_ln(B, T, D, dt, cuda, stream0=40 + 8 * i)
        layer = m.LayerNormLayer(gamma, beta)
        f = m.layernorm_forward(layer, x)
        ref.append(m.layernorm_backward_simultaneous(layer, f.cache, dy))
        dx, p = layers.layernorm_backward_rows(layer, f.cache, dy)
        dxs.append(dx)
        pend.append(p)
    out = layers.layernorm_backward_reduce(pend)
    torch.cuda.synchronize()
    for r, o, dx in zip(ref, out, dxs):
        assert torch.equal(r.input_grad, dx)
        assert torch.equal(r.grads.weight_grads["gamma"], o.weight_grads["gamma"])
        assert torch.equal(r.grads.weight_grads["beta"], o.weight_grads["beta"])
        assert close(r.grads.per_example_sqnorms_raw["gamma"].cpu().numpy(),
                     o.per_example_sqnorms_raw["gamma"].cpu().numpy(), 1e-12)
        assert close(r.grads.per_example_sqnorms_raw["beta"].cpu().numpy(),
                     o.per_example_sqnorms_raw["beta"].cpu().numpy(), 1e-12)
        assert close(r.grads.sums4.cpu().numpy(), o.sums4.cpu().numpy(), 1e-12)
    # the plain twin through the same path
    pend2 = []
    for i, (dt, B, T, D) in enumerate(shapes[:2]):
        x, dy, gamma, beta = m.synth_ln(B, T, D, dt, cuda, stream0=40 + 8 * i)
        layer = m.LayerNormLayer(gamma, beta)
        f = m.layernorm_forward(layer, x)
        pend2.append(layers.layernorm_backward_rows(layer, f.cache, dy)[1])
    out2 = layers.layernorm_backward_reduce(pend2, with_norms=False)
    torch.cuda.synchronize()
    for r, o in zip(ref[:2], out2):
        assert torch.equal(r.grads.weight_grads["gamma"], o.weight_grads["gamma"])
        assert o.per_example_sqnorms == {}


@pytest.mark.parametrize("dt,B,T,D", [(torch.bfloat16, 2048, 4, 768), (torch.float32, 1100, 3, 96)])
def test_many_examples_blocked_stage2(orc, cuda, dt, B, T, D):
    """B beyond one shared-memory block of the reduce (512 examples) and beyond
    the final fold's on-chip buffer: still the oracle's norms."""
    m = _mod()
    x, dy, gamma, beta = m.synth_ln(B, T, D, dt, cuda, stream0=9)
    layer = m.LayerNormLayer(gamma, beta)
    f = m.layernorm_forward(layer, x)
    r = m.layernorm_backward_simultaneous(layer, f.cache, dy)
    ref = _oracle_on_device_stats(orc, x, dy, gamma, f.cache.mean, f.cache.inv_std)
    torch.cuda.synchronize()
    assert close(r.grads.per_example_sqnorms_raw["gamma"].cpu().numpy(), ref["raw_gamma"], NORM_TOL)
    assert close(r.grads.per_example_sqnorms_raw["beta"].cpu().numpy(), ref["raw_beta"], NORM_TOL)
    assert close(float(r.grads.per_example_sqnorms["gamma"]), ref["corrected"][0], NORM_TOL)
    gt = F32_TOL if dt == torch.float32 else NORM_TOL
    assert _close_inf(r.grads.weight_grads["gamma"].double().cpu().numpy(), ref["dgamma"], gt)


def test_deferred_reduce_limits(cuda):
    """64 pending LayerNorms in one launch; more, or mixed fp32/fp64
    statistics, are rejected with the reference-style error."""
    m = _mod()
    from paper_2411_00999_b200 import layers

    pend = []
    for i in range(64):
        x, dy, gamma, beta = m.synth_ln(2, 3, 32, torch.bfloat16, cuda, stream0=100 + i)
        layer = m.LayerNormLayer(gamma, beta)
        f = m.layernorm_forward(layer, x)
        pend.append(layers.layernorm_backward_rows(layer, f.cache, dy)[1])
        if i == 63:
            ref = m.layernorm_backward_simultaneous(layer, f.cache, dy)
    out = layers.layernorm_backward_reduce(pend)
    torch.cuda.synchronize()
    assert torch.equal(out[-1].weight_grads["gamma"], ref.grads.weight_grads["gamma"])
    assert close(out[-1].sums4.cpu().numpy(), ref.grads.sums4.cpu().numpy(), 1e-12)
    with pytest.raises(ValueError, match="too many pending"):
        layers.layernorm_backward_reduce(pend + pend[:1])
    x, dy, gamma, beta = m.synth_ln(2, 3, 8, torch.float64, cuda)
    f = m.layernorm_forward(m.LayerNormLayer(gamma, beta), x)
    p64 = layers.layernorm_backward_rows(m.LayerNormLayer(gamma, beta), f.cache, dy)[1]
    with pytest.raises(ValueError, match="mix fp64 and fp32"):
        layers.layernorm_backward_reduce([pend[0], p64])


@pytest.mark.parametrize(
    "dt,B,T,D,offset,use_xhat",
    [
        (torch.bfloat16, 5, 13, 256, 0, False),
        (torch.bfloat16, 7, 8, 512, 0, False),
        (torch.bfloat16, 4, 9, 768, 0, False),
        (torch.bfloat16, 37, 11, 1024, 0, False), # many examples per CTA
        (torch.float32, 3, 50, 384, 0, False),
        (torch.float32, 2, 64, 512, 0, True),     # x-hat cache (no mean)
        (torch.bfloat16, 3, 20, 768, 3, False),   # rows not 16-byte aligned: element-wise path
        (torch.float32, 3, 20, 256, 1, True),
        (torch.float64, 3, 16, 96, 0, False),
        (torch.bfloat16, 2, 7, 768, 0, False),
        (torch.bfloat16, 300, 2, 768, 0, False),  # CTAs spanning 3+ examples (parked first example + L2 middle)
        (torch.bfloat16, 5, 700, 768, 0, False),  # CTAs inside one example and across one boundary
    ],
)
def test_row_pass_edge_cases_match_oracle(orc, cuda, dt, B, T, D, offset, use_xhat):
    """Row pass against the oracle at example boundaries in every position of
    a row stage, with the x-hat cache (no mean), with row pointers that are not
    16-byte aligned (storage offset: the non-TMA producer) and through the
    deferred grouped reduce."""
    m = _mod()
    bf = dt == torch.bfloat16
    x, dy, gamma, beta = m.synth_ln(B, T, D, dt, cuda, stream0=11)
    if offset:
        def shift(t):
            buf = torch.empty(t.numel() + offset, dtype=t.dtype, device=cuda)
            v = buf[offset:].view(t.shape)
            v.copy_(t)
            return v
        x, dy = shift(x), shift(dy)
        assert x.data_ptr() % 16 != 0
    layer = m.LayerNormLayer(gamma, beta, 1e-5)
    f = m.layernorm_forward(layer, x)
    cache = f.cache
    if use_xhat:
        xh = ((x.double() - f.cache.mean.double()[..., None]) * f.cache.inv_std.double()[..., None]).to(dt)
        if offset:
            xh = shift(xh)
        cache = m.LayerNormCache(normalized=xh, inv_std=f.cache.inv_std)
        ref = orc.ln_backward(xh.cpu().double().numpy(), f.cache.inv_std.cpu().double().numpy(),
                              dy.cpu().double().numpy(), gamma.cpu().double().numpy())
    else:
        ref = _oracle_on_device_stats(orc, x, dy, gamma, f.cache.mean, f.cache.inv_std)
    from paper_2411_00999_b200 import layers

    r = m.layernorm_backward_simultaneous(layer, cache, dy)
    dxd, pend = layers.layernorm_backward_rows(layer, cache, dy)
    rd = layers.layernorm_backward_reduce([pend])[0]
    torch.cuda.synchronize()
    dxt = {torch.float64: 1e-11, torch.float32: F32_TOL, torch.bfloat16: BF16_DX}[dt]
    gt = {torch.float64: 1e-11, torch.float32: F32_TOL, torch.bfloat16: NORM_TOL}[dt]
    nt = {torch.float64: 1e-11, torch.float32: NORM_TOL, torch.bfloat16: NORM_TOL}[dt]
    for dxv, gr in ((r.input_grad, r.grads), (dxd, rd)):
        assert _close_inf(dxv.double().cpu().numpy(), ref["dx"], dxt)
        assert _close_inf(gr.weight_grads["gamma"].double().cpu().numpy(), ref["dgamma"], gt)
        assert _close_inf(gr.weight_grads["beta"].double().cpu().numpy(), ref["dbeta"], gt)
        assert close(gr.per_example_sqnorms_raw["gamma"].cpu().numpy(), ref["raw_gamma"], nt)
        assert close(gr.per_example_sqnorms_raw["beta"].cpu().numpy(), ref["raw_beta"], nt)
    assert torch.equal(r.input_grad, dxd)
    if dt == torch.float64:
        # fp64 gnsb_ln_bwd forms the per-example parameter gradients, norms and
        # their sums in the reference's order (ln_ref.cu): bit-identical to the
        # reference restatement on the x-hat cache it consumes
        if use_xhat:
            np.testing.assert_array_equal(r.grads.weight_grads["gamma"].cpu().numpy(), ref["dgamma"])
            np.testing.assert_array_equal(r.grads.weight_grads["beta"].cpu().numpy(), ref["dbeta"])
            np.testing.assert_array_equal(r.grads.per_example_sqnorms_raw["gamma"].cpu().numpy(), ref["raw_gamma"])
            np.testing.assert_array_equal(r.grads.per_example_sqnorms_raw["beta"].cpu().numpy(), ref["raw_beta"])
    else:
        assert torch.equal(r.grads.weight_grads["gamma"], rd.weight_grads["gamma"])


def test_fp64_per_example_values_are_batch_invariant(cuda):
    """fp64 rows: example b's share of a batched call equals a B = 1 call on
    its rows bit for bit (what the reference's PerExample-vs-Microbatch trainer
    identity needs, proj/tests/test_trainer.cpp:123-130), for the LayerNorm and
    the linear layer."""
    from paper_2411_00999_b200 import linear

    m = _mod()
    B, T, D = 4, 24, 40
    x, dy, gamma, beta = m.synth_ln(B, T, D, torch.float64, cuda, stream0=5)
    layer = m.LayerNormLayer(gamma, beta, 1e-5)
    xh = m.layernorm_forward(layer, x, keep_normalized=True).cache
    cache = m.LayerNormCache(normalized=xh.normalized, inv_std=xh.inv_std)
    full = m.layernorm_backward_simultaneous(layer, cache, dy)
    W = torch.randn(D, 24, dtype=torch.float64, device=cuda)
    g2 = torch.randn(B, T, 24, dtype=torch.float64, device=cuda)
    lfull = linear.linear_backward_simultaneous(linear.LinearLayer(W, torch.zeros(24, dtype=torch.float64, device=cuda)),
                                                x, g2, need_input_grad=False)
    for b in range(B):
        one = m.layernorm_backward_simultaneous(
            layer, m.LayerNormCache(normalized=cache.normalized[b:b + 1], inv_std=cache.inv_std[b:b + 1]), dy[b:b + 1])
        assert float(one.grads.per_example_sqnorms_raw["gamma"][0]) == float(full.grads.per_example_sqnorms_raw["gamma"][b])
        assert float(one.grads.per_example_sqnorms_raw["beta"][0]) == float(full.grads.per_example_sqnorms_raw["beta"][b])
        lo = linear.linear_backward_simultaneous(
            linear.LinearLayer(W, torch.zeros(24, dtype=torch.float64, device=cuda)), x[b:b + 1], g2[b:b + 1],
            need_input_grad=False)
        assert float(lo.grads.per_example_sqnorms_raw["weight"][0]) == float(lfull.grads.per_example_sqnorms_raw["weight"][b])
        assert float(lo.grads.per_example_sqnorms_raw["bias"][0]) == float(lfull.grads.per_example_sqnorms_raw["bias"][b])
        # and the squared norm of the B = 1 gradient, summed in order, is that raw value
        dg = one.grads.weight_grads["gamma"].cpu().numpy()
        s = 0.0
        for v in dg:
            s += v * v
        assert s == float(full.grads.per_example_sqnorms_raw["gamma"][b])


@pytest.mark.parametrize("dt,D", [(torch.bfloat16, 1024), (torch.float32, 768)])
def test_gamma_view_at_unaligned_offset(orc, cuda, dt, D):
    """gamma as a view into a flat parameter buffer at a 4-byte (not 16-byte)
    offset: the kernel stages it element-wise instead of faulting on a uint4 load
    (ln_bwd.cuh gamma staging)."""
    m = _mod()
    x, dy, gamma, beta = m.synth_ln(4, 64, D, dt, cuda, stream0=21)
    flat = torch.empty(D + 1, dtype=torch.float32, device=cuda)
    gv = flat[1:]
    gv.copy_(gamma)
    assert gv.data_ptr() % 16 != 0
    layer = m.LayerNormLayer(gv, beta)
    f = m.layernorm_forward(layer, x)
    r = m.layernorm_backward_simultaneous(layer, f.cache, dy)
    ref = _oracle_on_device_stats(orc, x, dy, gamma, f.cache.mean, f.cache.inv_std)
    torch.cuda.synchronize()
    dxt = BF16_DX if dt == torch.bfloat16 else F32_TOL
    assert _close_inf(r.input_grad.double().cpu().numpy(), ref["dx"], dxt)
    assert close(r.grads.per_example_sqnorms_raw["gamma"].cpu().numpy(), ref["raw_gamma"], NORM_TOL)
    base = m.layernorm_backward_simultaneous(m.LayerNormLayer(gamma, beta), f.cache, dy)
    assert torch.equal(base.input_grad, r.input_grad)
