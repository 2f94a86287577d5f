"""Batch-sharded host logic at world size 2 over gloo, on CPU.

Each rank runs the oracle's LayerNorm backward on its contiguous example block
(the oracle stands in for the device kernel, which needs a GPU), fills the
product's exchange buckets exactly as `gnsb_ln_bwd` would, and calls
`GradBuckets.reduce`. The reduced gradients, the re-formed ||G_big||^2 and
the B_global-corrected per-example norms must equal the unsharded
reference's, and so must the GNS estimates built from them.
"""
import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import close

WIDTHS = (8, 6, 5)
B_GLOBAL, T = 5, 4


def _np_sqnorm(v, out):
    a = v.detach().double().numpy()
    out.fill_(float(np.dot(a, a)))


def _layer(orc, l, b0, b1):
    """Oracle backward of examples [b0, b1) of layer l (dy from a mean loss over B_GLOBAL)."""
    D = WIDTHS[l]
    x, dy, gamma, beta = orc.synth_ln(B_GLOBAL, T, D, B_div=B_GLOBAL, stream0=16 * l)
    _, xhat, inv = orc.ln_forward(x[b0:b1], gamma, beta)
    return orc.ln_backward(xhat, inv, dy[b0:b1], gamma)


def _worker(rank, world, init_file, errfile):
    try:
        from oracle.ffi import Oracle

        import paper_2411_00999_b200 as m
        from paper_2411_00999_b200 import sharded

        dist.init_process_group("gloo", init_method=f"file://{init_file}", rank=rank, world_size=world)
        orc = Oracle()
        b0, b1 = sharded.shard_bounds(B_GLOBAL, world, rank)
        bk = sharded.GradBuckets(WIDTHS, "cpu", grad_dtype=torch.float64)
        for l in range(len(WIDTHS)):
            r = _layer(orc, l, b0, b1)
            dg, db = bk.grad(l)
            dg.copy_(torch.from_numpy(r["dgamma"]))
            db.copy_(torch.from_numpy(r["dbeta"]))
            rec = bk.record(l)
            # what gnsb_ln_bwd writes into `sums`: LOCAL sums and squared norms
            rec.copy_(torch.tensor([r["raw_gamma"].sum(), r["raw_beta"].sum(),
                                    float(np.dot(r["dgamma"], r["dgamma"])), float(np.dot(r["dbeta"], r["dbeta"]))]))
        bk.reduce(sqnorm=_np_sqnorm)

        g_big = g_small = 0.0
        for l in range(len(WIDTHS)):
            full = _layer(orc, l, 0, B_GLOBAL)
            dg, db = bk.grad(l)
            assert close(dg.numpy(), full["dgamma"], 1e-12, 1e-14), l
            assert close(db.numpy(), full["dbeta"], 1e-12, 1e-14), l
            st = sharded.layer_grad_stats(bk.record(l).tolist(), B_GLOBAL)
            ref_big = float(np.dot(full["dbeta"], full["dbeta"]) + np.dot(full["dgamma"], full["dgamma"]))
            ref_small = float(full["corrected"][1] + full["corrected"][0])
            assert close(st.g_big_sqnorm, ref_big, 1e-12), (l, st.g_big_sqnorm, ref_big)
            assert close(st.g_small_sqnorm_mean, ref_small, 1e-12), (l, st.g_small_sqnorm_mean, ref_small)
            assert (st.b_big, st.b_small, st.n_small) == (B_GLOBAL, 1, B_GLOBAL)
            g_big += ref_big
            g_small += ref_small
        # group estimate over all layers (aggregate then estimate, gns.cpp:31-89)
        stats = {("ln", i): sharded.layer_grad_stats(bk.record(i).tolist(), B_GLOBAL) for i in range(len(WIDTHS))}
        agg = m.aggregate({(k[1], "layernorm"): v for k, v in stats.items()}, None)
        ref = m.GradStats(g_big, g_small, B_GLOBAL, 1, B_GLOBAL)
        assert close(m.estimate_g2(agg), m.estimate_g2(ref), 1e-10)
        assert close(m.estimate_s(agg), m.estimate_s(ref), 1e-10)
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as exc:  # surface the failure to the parent
        with open(errfile + f".{rank}", "w") as f:
            f.write(repr(exc))
        raise


def test_shard_bounds():
    from paper_2411_00999_b200.sharded import shard_bounds

    for B in (1, 5, 8, 256):
        for world in (1, 2, 3, 8):
            blocks = [shard_bounds(B, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == B
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(world - 1))
            sizes = [b1 - b0 for b0, b1 in blocks]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(0, 2, 0)
    with pytest.raises(ValueError):
        shard_bounds(4, 2, 2)


def test_layer_grad_stats_matches_reference_packaging():
    """trainer.cpp:363-378: g_big = sum ||grad||^2, g_small = sum B*sum raw."""
    from paper_2411_00999_b200.sharded import layer_grad_stats

    st = layer_grad_stats([1.5, 0.5, 2.0, 3.0], 4)
    assert st.g_big_sqnorm == 5.0
    assert st.g_small_sqnorm_mean == 0.5 / 4 * 16 + 1.5 / 4 * 16
    assert (st.b_big, st.b_small, st.n_small) == (4, 1, 4)


def test_sharded_world2_matches_unsharded_reference():
    world = 2
    with tempfile.TemporaryDirectory() as d:
        init_file = os.path.join(d, "pg")
        errfile = os.path.join(d, "err")
        try:
            mp.spawn(_worker, args=(world, init_file, errfile), nprocs=world, join=True)
        except Exception:
            msgs = [open(os.path.join(d, f)).read() for f in os.listdir(d) if f.startswith("err")]
            pytest.fail("; ".join(msgs) or "worker failed")
