"""Batch-sharded fused LN backward on the GPU, world size 2.

The pool has one GPU, so both ranks share cuda:0 and talk over gloo (the
measured path is NCCL with one GPU per rank; the host logic is the same
GradBuckets.reduce). Each rank runs the fused kernel on its contiguous block of
examples of a globally-indexed synthetic batch (synth b_offset = the block
start, dy scaled by 1/B_global). The reduced dgamma/dbeta, the re-formed
||G_big||^2 and the B_global-corrected norms must match one process running
the whole batch: dgamma/dbeta to fp32 summation-order tolerance (1e-5), norm
records to 1e-6.
"""
import json
import os
import socket
import subprocess
import sys
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, close

pytestmark = pytest.mark.gpu

B_GLOBAL, T, WIDTHS = 6, 64, (768, 1024)


def _shard_records(b0, b1, dev):
    import paper_2411_00999_b200 as m
    from paper_2411_00999_b200.sharded import GradBuckets

    bk = GradBuckets(WIDTHS, dev)
    for l, D in enumerate(WIDTHS):
        x, dy, gamma, beta = m.synth_ln(b1 - b0, T, D, torch.bfloat16, dev, b_offset=b0, B_div=B_GLOBAL,
                                        stream0=16 * l)
        layer = m.LayerNormLayer(gamma, beta)
        f = m.layernorm_forward(layer, x)
        r = m.layernorm_backward_simultaneous(layer, f.cache, dy, need_input_grad=False)
        dg, db = bk.grad(l)
        dg.copy_(r.grads.weight_grads["gamma"])
        db.copy_(r.grads.weight_grads["beta"])
        bk.record(l).copy_(r.grads.sums4)
    return bk


def _worker(rank, world, init_file, out):
    from paper_2411_00999_b200.sharded import shard_bounds

    dist.init_process_group("gloo", init_method=f"file://{init_file}", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    b0, b1 = shard_bounds(B_GLOBAL, world, rank)
    bk = _shard_records(b0, b1, dev)
    bk.reduce()
    torch.cuda.synchronize()
    if rank == 0:
        np.savez(out, grads=bk.grads.cpu().numpy(), records=bk.records.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_world2_matches_single_process(cuda):
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "r.npz")
        mp.spawn(_worker, args=(2, os.path.join(d, "pg"), out), nprocs=2, join=True)
        res = np.load(out)
    full = _shard_records(0, B_GLOBAL, cuda)
    torch.cuda.synchronize()
    g = full.grads.cpu().numpy()
    assert close(res["grads"], g, 1e-5, 1e-5 * np.abs(g).max())
    rec = full.records.cpu().numpy()
    assert close(res["records"], rec, 1e-6)
    # corrected per-example norm uses B_global: sum over ranks of local raw sums
    from paper_2411_00999_b200.sharded import layer_grad_stats

    for l in range(len(WIDTHS)):
        a, b = layer_grad_stats(res["records"][l], B_GLOBAL), layer_grad_stats(rec[l], B_GLOBAL)
        assert close(a.g_small_sqnorm_mean, b.g_small_sqnorm_mean, 1e-6)
        assert close(a.g_big_sqnorm, b.g_big_sqnorm, 1e-6)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_multirank_path_runs(cuda):
    """bench.py under torchrun with 2 ranks (gloo, both on cuda:0): the N > 1
    line is the configs[4] strong-scaling step (here at a reduced B_global,T,D):
    one JSON line from rank 0, n_gpus=2, scaling strong, ONE collective per
    step (the packed fp64 bucket) and the C-ABI kernels of the step counted."""
    env = dict(os.environ, GNSB_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-cpu", "--cfg5", "64,256,1024"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["value"] > 0 and rec["scaling"] == "strong"
    assert rec["config"]["global_batch"] == 64 and rec["config"]["B_global"] == 64
    assert rec["collectives_per_step"] == 1 and rec["gpu_launches"] == 5 * 3
    assert rec["e2e"]["h2d_bytes_per_step"] == 32 * 256 * 1024 * 4 + 32 * 256 * 8
    assert rec["roofline"]["achieved"] > 0


@pytest.mark.parametrize("gdt", [torch.float32, torch.float64])
def test_c_abi_allreduce_buckets_single_rank(cuda, gdt):
    """gnsb_allreduce_buckets (the C ABI's exchange step): with no communicator
    and with a one-rank NCCL communicator the gradients are unchanged (an
    fp64 round trip), records[l][0..1] too, and records[l][2..3] are
    re-formed as ||p0||^2, ||p1||^2 of the gradient bucket.  Layers of
    unequal (p0, p1) widths: a LayerNorm (768, 768), a linear layer (K*L, L)
    with K*L spanning several unpack chunks, a bias-less layer (n, 0)."""
    import ctypes

    from paper_2411_00999_b200 import _lib
    from paper_2411_00999_b200.sharded import GradBuckets

    lib = _lib.lib()
    pairs = [(768, 768), (5, 5), (256 * 300, 300), (1024, 0), (40000, 1)]
    n = sum(a + b for a, b in pairs)
    gen = torch.Generator(device="cpu").manual_seed(3)
    bk = GradBuckets(pairs, cuda, grad_dtype=gdt)
    bk.grads.copy_(torch.randn(n, generator=gen, dtype=torch.float64))
    bk.records[:, :2] = torch.arange(2 * len(pairs), dtype=torch.float64).reshape(-1, 2)
    expect = []
    for l in range(len(pairs)):
        a, b = (v.double() for v in bk.grad(l))
        expect.append([float((a * a).sum()), float((b * b).sum())])
    comms = [None]
    if lib.gnsb_nccl_available():
        class _C:
            pass
        uid = ctypes.create_string_buffer(128)
        _lib.check(lib.gnsb_nccl_get_unique_id(uid))
        comm = _C()
        comm.handle = ctypes.c_void_p()
        _lib.check(lib.gnsb_nccl_comm_init_rank(ctypes.byref(comm.handle), 1, uid, 0))
        comms.append(comm)
    for comm in comms:
        for rec in (True, False):
            g0, r0 = bk.grads.clone(), bk.records[:, :2].clone()
            bk.records[:, 2:] = -1.0
            if comm is None:
                bk.reduce(records=rec)
            else:
                bk.allreduce_nccl(comm, records=rec)
            torch.cuda.synchronize()
            assert torch.equal(bk.grads, g0) and torch.equal(bk.records[:, :2], r0)
            if rec:
                assert close(bk.records[:, 2:].cpu().numpy(), np.array(expect), 1e-12)
            else:
                assert (bk.records[:, 2:] == -1.0).all()
    if len(comms) > 1:
        _lib.check(lib.gnsb_nccl_comm_destroy(comms[1].handle))
    w = (ctypes.c_int64 * 2)(4, 4)
    sp = torch.cuda.current_stream().cuda_stream
    with pytest.raises(ValueError, match="bucket"):
        _lib.check(lib.gnsb_allreduce_buckets(bk.grads.data_ptr(), 0, w, 0, bk.records.data_ptr(),
                                              bk._ws.data_ptr(), bk._ws.numel(), None, sp))
    with pytest.raises(ValueError, match="workspace too small"):
        _lib.check(lib.gnsb_allreduce_buckets(bk.grads.data_ptr(), 0, w, 1, bk.records.data_ptr(),
                                              bk._ws.data_ptr(), 8, None, sp))
