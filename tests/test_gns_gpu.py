"""Device GNS accumulator (gnsb_gns_step) and the BASELINE config-4 pipeline.

The reference path is Trainer::step's PerExample packaging + fill_group
(proj/src/trainer.cpp:324-325, 363-415) over gns.cpp's estimators.  The
checks restate that arithmetic on the host (the reference functions exposed by
the C ABI's host side, themselves pinned by tests/test_capi_host.py) and
compare the device results.  Tolerance: rel 1e-12 (fp64 on both sides, only
FMA contraction differs); pipeline parity vs the oracle: rel 1e-4 (north star).
"""
import math

import numpy as np
import pytest
import torch

from conftest import close

pytestmark = pytest.mark.gpu


def _host_step(records, types, B, states, alpha):
    """Host restatement of one Trainer::step GNS update (trainer.cpp:363-415)."""
    from paper_2411_00999_b200 import gns

    def corr(v):
        b = float(B)
        return v / b * (b * b)  # layers.cpp:39-42

    stats = {}
    per_layer = []
    for i, (r, t) in enumerate(zip(records, types)):
        big = 0.0 + r[3] + r[2]
        small = 0.0 + corr(r[1]) + corr(r[0])
        st = gns.GradStats(big, small, B, 1, B)
        stats[(f"l{i:03d}", t)] = st
        per_layer.append((gns.estimate_g2(st), gns.estimate_s(st)))
    out = []
    for gi, grp in enumerate([None, "embedding", "linear", "layernorm"]):
        try:
            agg = gns.aggregate(stats, grp)
        except ValueError:
            out.append(None)
            continue
        g2, s = gns.estimate_g2(agg), gns.estimate_s(agg)
        states[gi][0] = gns.ema_update(states[gi][0], g2)
        states[gi][1] = gns.ema_update(states[gi][1], s)
        e = gns.smoothed_gns(states[gi][0], states[gi][1])
        out.append((g2, s, e.b_simple if e.b_simple_defined else 0.0, 1.0 if e.b_simple_defined else 0.0))
    return out, per_layer


def test_device_gns_step_matches_host(cuda):
    from paper_2411_00999_b200 import gns

    rng = np.random.default_rng(7)
    types = ["layernorm", "linear", "layernorm", "embedding", "linear", "layernorm"]
    B, alpha = 16, 0.3
    acc = gns.DeviceGnsAccumulator(types, alpha, cuda)
    states = [[gns.EmaState(alpha), gns.EmaState(alpha)] for _ in range(4)]
    for step in range(5):
        recs = rng.uniform(0.1, 2.0, size=(len(types), 4))
        dev = torch.tensor(recs, dtype=torch.float64, device=cuda)
        groups, layers = acc.step(dev, B)
        ref, ref_layers = _host_step(recs, types, B, states, alpha)
        g = groups.cpu().numpy()
        for gi in range(4):
            assert close(g[gi, :2], ref[gi][:2], 1e-12), (step, gi)
            assert g[gi, 3] == ref[gi][3]
            assert close(g[gi, 2], ref[gi][2], 1e-12)
        assert close(layers.cpu().numpy(), np.array(ref_layers), 1e-12)


def test_device_gns_empty_group_and_errors(cuda):
    from paper_2411_00999_b200 import _lib, gns

    acc = gns.DeviceGnsAccumulator(["layernorm", "layernorm"], 1.0, cuda)
    groups, _ = acc.step(torch.ones(2, 4, dtype=torch.float64, device=cuda), 4)
    g = groups.cpu().numpy()
    assert np.isfinite(g[0]).all() and np.isfinite(g[3]).all()
    assert np.isnan(g[1, :3]).all() and np.isnan(g[2, :3]).all()  # no embedding / linear layers
    assert g[1, 3] == 0.0 and g[2, 3] == 0.0  # ... and so no defined estimate
    with pytest.raises(ValueError, match="batch >= 2"):
        acc.step(torch.ones(2, 4, dtype=torch.float64, device=cuda), 1)
    with pytest.raises(ValueError, match="alpha"):
        gns.DeviceGnsAccumulator(["layernorm"], 1.5, cuda).step(torch.ones(1, 4, dtype=torch.float64, device=cuda), 4)


@pytest.mark.parametrize("sigma", [0.3, 3.0, 30.0])
def test_cfg4_gns_over_25_layernorms(orc, cuda, sigma):
    """BASELINE config 4 (reduced T for the fp64 oracle): 25 LayerNorms of a
    12-layer D=768 transformer, B=64, synthetic activations/grads with layer
    streams offset by 16*l; one fused backward per layer -> device GNS step.
    Compared with the reference arithmetic (oracle backward + host GNS)."""
    from paper_2411_00999_b200 import gns
    import paper_2411_00999_b200 as m

    L, B, T, D = 25, 64, 128, 768
    recs = []
    ref_recs = []
    for l in range(L):
        x, dy, gamma, beta = m.synth_ln(B, T, D, torch.bfloat16, cuda, sigma=sigma, stream0=16 * l)
        gamma.fill_(1.0)  # gamma=1, beta=0 as the toy model initialises (model.cpp:39-40)
        beta.zero_()
        layer = m.LayerNormLayer(gamma, beta)
        f = m.layernorm_forward(layer, x)
        r = m.layernorm_backward_simultaneous(layer, f.cache, dy, need_input_grad=False)
        recs.append(r.grads.sums4)
        ref = orc.ln_backward(x.double().cpu().numpy(), f.cache.inv_std.double().cpu().numpy(),
                              dy.double().cpu().numpy(), np.ones(D), mean=f.cache.mean.double().cpu().numpy())
        ref_recs.append([ref["raw_gamma"].sum(), ref["raw_beta"].sum(), float(np.dot(ref["dgamma"], ref["dgamma"])),
                         float(np.dot(ref["dbeta"], ref["dbeta"]))])
    records = torch.stack(recs).contiguous()
    acc = gns.DeviceGnsAccumulator(["layernorm"] * L, 1.0, cuda)
    groups, layers = acc.step(records, B)
    torch.cuda.synchronize()
    assert close(records.cpu().numpy(), np.array(ref_recs), 1e-4)
    states = [[gns.EmaState(1.0), gns.EmaState(1.0)] for _ in range(4)]
    ref_groups, ref_layers = _host_step(np.array(ref_recs), ["layernorm"] * L, B, states, 1.0)
    g = groups.cpu().numpy()
    # plain rel 1e-4 (north star) on G^2, S and B_simple, no scale-aware loosening
    assert close(g[0, 0], ref_groups[0][0], 1e-4)
    assert close(g[0, 1], ref_groups[0][1], 1e-4)
    assert close(g[3, :2], g[0, :2], 0.0)  # every layer is a LayerNorm
    assert ref_groups[0][3] == 1.0 and g[0, 3] == 1.0
    assert close(g[0, 2], ref_groups[0][2], 1e-4)
