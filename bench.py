#!/usr/bin/env python
"""Benchmark: fused LN-backward + per-example-norm HBM GB/s and % overhead vs plain LN-backward.

Workload (BASELINE.json configs[1]): LayerNorm backward + per-example
||dgamma_b||^2, ||dbeta_b||^2 over the sweep D in {768, 1024, 2048, 4096, 8192},
B=32 T=1024 per GPU, bf16 rows / fp32 accumulation.  One "step" = one fused
backward per D of the sweep (plus, for N > 1, the NCCL all-reduce of the
sweep's [dgamma | dbeta] bucket and fp64 norm-record bucket).  Inputs are synthetic
(SURVEY §8(d) recipe, generated on the device; identical to the oracle's).

value      = sum over ranks and D of algorithmic bytes / max-over-ranks device time
             bytes(D) = N*D*(2*s_in + s_out) + 8N + 12D + 16B; s = 2 (bf16)
e2e        = same metric through the C ABI with HOST (pinned) buffers: H2D of x, dy,
             mean, rstd, the kernel, D2H of dx, dgamma, dbeta, raw norms and sums
overhead   = (t_fused - t_plain) / t_plain, same kernel with norms compiled out
L2         = flushed (256 MiB write) before every timed kernel, outside the events

--impl reference times the reference's own CPU implementation (oracle/_ref:
the unmodified gnstk sources compiled from /root/reference, multi-threaded over
example slices) on bounded samples of the same workload.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SWEEP_D = [768, 1024, 2048, 4096, 8192]
B_LOCAL, T = 32, 1024
METRIC = "fused LN-bwd+per-example-norm HBM GB/s & % overhead vs plain LN-bwd"
WORKLOAD = "cfg2: LayerNorm backward + per-example dgamma/dbeta norms, sweep D=768..8192, B=32 T=1024 per GPU, bf16 in / fp32 acc"


def alg_bytes(B, T_, D, s_in=2, s_out=2, norms=True):
    N = B * T_
    return N * D * (2 * s_in + s_out) + 8 * N + 4 * D + 8 * D + (16 * B if norms else 0)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms",
                 "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self._proc = None
        return self

    def _read(self):
        for line in self._proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self._proc is not None:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=2)
            except Exception:
                self._proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ----------------------------------------------------------------------------- reference arm
def ref_layer_sample(ref, orc, D, b_sample, threads):
    """One bounded sample: b_sample examples of the cfg2 workload at width D,
    the reference's layernorm_backward_simultaneous over `threads` example slices."""
    import numpy as np

    x, dy, gamma, beta = orc.synth_ln(b_sample, T, D, B_div=B_LOCAL, bf16=True)
    _, xhat, inv = ref.ln_forward(x.astype(np.float64), gamma.astype(np.float64), beta.astype(np.float64))
    g = dy.astype(np.float64)
    gm = gamma.astype(np.float64)
    t0 = time.perf_counter()
    ref.ln_backward(xhat, inv, g, gm, threads=threads)
    return time.perf_counter() - t0


def run_reference_arm(args):
    import numpy as np  # noqa: F401

    from oracle import ffi

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    if not ffi.reference_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libgnstk_ref.so not built"}))
        return 0
    ref, orc = ffi.reference(), ffi.oracle()
    threads = os.cpu_count() or 1
    b_sample = min(B_LOCAL, threads)
    times = []
    for i in range(args.warmup + args.steps):
        step_t = sum(ref_layer_sample(ref, orc, D, b_sample, threads) for D in SWEEP_D)
        if i >= args.warmup:
            times.append(step_t)
    sample_bytes = sum(alg_bytes(b_sample, T, D) for D in SWEEP_D)
    gbs = sample_bytes / statistics.median(times) / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": statistics.median(times) * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "B": B_LOCAL, "T": T, "D": SWEEP_D},
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": threads, "kind": "reference",
                         "sample": f"{b_sample} of {B_LOCAL} examples x T={T} per D of the sweep per step, "
                                   f"gnstk::layernorm_backward_simultaneous over {threads} example slices, fp64; "
                                   "bytes counted with the bf16 workload formula"},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- our arm
class LnCase:
    """Device buffers + raw C-ABI argument tuples for one D of the sweep.
    dgamma/dbeta/sums are views into the step's exchange buckets (sharded.py)."""

    def __init__(self, m, lib, D, B, rank, dev, torch, buckets, l):
        self.D, self.B = D, B
        bf = torch.bfloat16
        self.x, self.dy, self.gamma, self.beta = m.synth_ln(B, T, D, bf, dev, b_offset=rank * B, B_div=B)
        layer = m.LayerNormLayer(self.gamma, self.beta)
        f = m.layernorm_forward(layer, self.x)
        self.mean, self.rstd = f.cache.mean, f.cache.inv_std
        self.dx = torch.empty_like(self.x)
        self.dgamma, self.dbeta = buckets.grad(l)
        self.sums = buckets.record(l)
        self.raw_g = torch.zeros(B, dtype=torch.float64, device=dev)
        self.raw_b = torch.zeros(B, dtype=torch.float64, device=dev)
        nbytes = m.layers.ctypes_size(B, T, D, 1)
        self.ws = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
        self.lib = lib
        self.bytes = alg_bytes(B, T, D)
        self.bytes_plain = alg_bytes(B, T, D, norms=False)

    def run_rows(self, stream_ptr, norms=True):
        """Row pass.  norms=False: the plain LayerNorm backward's row pass, the
        same rows viewed as ONE example of B*T rows (no per-example
        bookkeeping), as gnsb_ln_bwd(with_norms=0) runs it."""
        p = lambda t: t.data_ptr()
        Bv, Mv = (self.B, T) if norms else (1, self.B * T)
        rc = self.lib.gnsb_ln_bwd_rows(p(self.x), p(self.mean), p(self.rstd), p(self.dy), p(self.gamma), p(self.dx),
                                       Bv, Mv, self.D, 1, p(self.ws), self.ws.numel(), stream_ptr)
        if rc:
            raise RuntimeError(self.lib.gnsb_last_error().decode())

    def pending(self, _lib, norms=True):
        Bv, Mv = (self.B, T) if norms else (1, self.B * T)
        return _lib.LnBwdPending(self.ws.data_ptr(), self.ws.numel(), Bv, Mv, self.D, 1, self.dgamma.data_ptr(),
                                 self.dbeta.data_ptr(), self.raw_g.data_ptr(), self.raw_b.data_ptr(),
                                 self.sums.data_ptr())

    def aten_args(self, torch):
        """PyTorch's own LayerNorm backward on the same bf16 rows (the paper's
        baseline): bf16 weight/bias, fp32 mean/rstd."""
        if not hasattr(self, "_aten"):
            self._aten = (self.dy.view(self.B, T, self.D), self.x.view(self.B, T, self.D), [self.D],
                          self.mean.view(self.B, T, 1), self.rstd.view(self.B, T, 1),
                          self.gamma.to(torch.bfloat16), self.beta.to(torch.bfloat16), [True, True, True])
        return self._aten

    def run_aten(self, torch):
        torch.ops.aten.native_layer_norm_backward(*self.aten_args(torch))

    def run(self, norms, stream_ptr):
        p = lambda t: t.data_ptr()
        rc = self.lib.gnsb_ln_bwd(
            p(self.x), p(self.mean), p(self.rstd), p(self.dy), p(self.gamma), p(self.dx), p(self.dgamma),
            p(self.dbeta), p(self.raw_g), p(self.raw_b), p(self.sums), 1 if norms else 0, self.B, T, self.D, 1,
            p(self.ws), self.ws.numel(), stream_ptr)
        if rc:
            raise RuntimeError(self.lib.gnsb_last_error().decode())


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2411_00999_b200 as m
    from paper_2411_00999_b200 import _lib
    from paper_2411_00999_b200.sharded import GradBuckets

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # GNSB_DIST_BACKEND=gloo with more ranks than GPUs exercises the multi-rank
    # path on one device (tests only; the measured path is NCCL, one GPU per rank)
    backend = os.environ.get("GNSB_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # communicator lines (nranks, NVLS/NVLink transport) in the log
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    lib = _lib.lib()
    if world > 1:
        return run_sharded_main(args, m, lib, dev, torch, np, world, rank, local, backend)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    sweep = args.d_list
    buckets = GradBuckets(sweep, dev)
    cases = [LnCase(m, lib, D, B_LOCAL, rank, dev, torch, buckets, l) for l, D in enumerate(sweep)]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()

    pend = {True: (_lib.LnBwdPending * len(cases))(*[c.pending(_lib) for c in cases]),
            False: (_lib.LnBwdPending * len(cases))(*[c.pending(_lib, False) for c in cases])}

    def run_step(norms):
        """The compute of one step (captured as one CUDA graph): the fused (or
        plain) LN backward for every D of the sweep, as a backward pass runs it:
        the row pass of each layer as it comes, then the deferred stage 2 of all
        of them in one launch (gnsb_ln_bwd_reduce)."""
        sp_now = torch.cuda.current_stream(dev).cuda_stream
        for c in cases:
            c.run_rows(sp_now, norms)
        rc = lib.gnsb_ln_bwd_reduce(pend[norms], len(cases), 1 if norms else 0, sp_now)
        if rc:
            raise RuntimeError(lib.gnsb_last_error().decode())

    def exchange(norms):
        """N > 1: the step's one exchange, issued eagerly after the
        graph: all-reduce of every layer's [dgamma | dbeta] (fp32 bucket) and,
        with norms, of the fp64 norm records, then ||G_big||^2 re-formed from
        the reduced gradients.  The plain twin all-reduces its gradients too."""
        if world > 1:
            buckets.reduce(records=norms)

    def timed(case, norms):
        """Single kernel, cold: L2 flushed (256 MiB write) before, CUDA events around."""
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        case.run(norms, sp)
        e1.record(stream)
        return e0, e1

    # warm-up (also builds every launch plan) and CUDA-graph capture of the step
    side = torch.cuda.Stream(dev)
    side.wait_stream(stream)
    with torch.cuda.stream(side):
        for _ in range(args.warmup):
            run_step(True)
            run_step(False)
    stream.wait_stream(side)
    torch.cuda.synchronize()
    graphs = {}
    for norms in (True, False):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            run_step(norms)
        graphs[norms] = g
    torch.cuda.synchronize()

    def replay(norms):
        graphs[norms].replay()
        exchange(norms)

    for _ in range(args.warmup):
        replay(True)
        replay(False)
    torch.cuda.synchronize()

    # ---- timed region: K steps of the fused sweep (value) ----
    if world > 1:
        dist.barrier()
    clk = ClockSampler(local).__enter__()
    time.sleep(0.3)  # let nvidia-smi attach before the timed region
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        replay(True)
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_local = e0.elapsed_time(e1)
    ms_per_step = t_local / args.steps
    t = torch.tensor([t_local], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max_ms = float(t.item())
    total_bytes = sum(c.bytes for c in cases) * world * args.steps
    value = total_bytes / (t_max_ms * 1e-3) / 1e9

    # ---- step-level fused vs plain vs aten: interleaved graph replays ----
    reps = max(args.steps, 20)
    aten_graph = None
    if world == 1:
        aten_graph = capture_graph(lambda: [c.run_aten(torch) for c in cases], torch, dev)
    variants = {"fused": lambda: replay(True), "plain": lambda: replay(False)}
    if aten_graph is not None:
        variants["aten"] = aten_graph.replay
    st = interleaved(variants, reps, stream, torch, np)
    step_f, step_p = st["fused"]["median"], st["plain"]["median"]

    # ---- per-kernel cold launches (flush + events): per-D breakdown ----
    fk = np.zeros((reps, len(cases)))
    pk = np.zeros((reps, len(cases)))
    for r in range(reps):
        pairs = [(timed(c, True), timed(c, False)) for c in cases]
        torch.cuda.synchronize()
        for i, (a_, b_) in enumerate(pairs):
            fk[r, i] = a_[0].elapsed_time(a_[1])
            pk[r, i] = b_[0].elapsed_time(b_[1])
    peak, peak_kind = load_peaks()
    sweep_rows = []
    for i, c in enumerate(cases):
        tf, tp = float(np.median(fk[:, i])), float(np.median(pk[:, i]))
        geo = m.ln_bwd_geometry(c.B, T, c.D, torch.bfloat16)
        sweep_rows.append({
            "D": c.D, "fused_us": tf * 1e3, "plain_us": tp * 1e3, "fused_GBps": c.bytes / tf / 1e6,
            "plain_GBps": c.bytes_plain / tp / 1e6, "frac_of_measured_peak": c.bytes / tf / 1e6 / peak,
            "frac_of_8TBps": c.bytes / tf / 1e6 / 8000.0, "overhead_pct": 100.0 * (tf - tp) / tp,
            "grid": geo["grid"], "threads": geo["threads"], "stages": geo["stages"],
            "timing": "single cold launch: L2 flushed before, CUDA events around (includes launch latency)",
        })
    # ---- per D in a model-like step: NL LayerNorms of that width back to back
    # (distinct buffers, row pass each) + one grouped reduce, graph-replayed;
    # the sustained rate of each width as a backward pass runs it
    NL = 8
    for i, c in enumerate(cases):
        if args.no_extra:
            break
        extra_cases = [c] + [LnCase(m, lib, c.D, B_LOCAL, rank, dev, torch, GradBuckets([c.D], dev), 0)
                             for _ in range(NL - 1)]
        pend_d = {nm: (_lib.LnBwdPending * NL)(*[e.pending(_lib, nm) for e in extra_cases]) for nm in (True, False)}

        def layer_step(norms, extra_cases=extra_cases, pend_d=pend_d):
            spn = torch.cuda.current_stream(dev).cuda_stream
            for e in extra_cases:
                e.run_rows(spn, norms)
            if lib.gnsb_ln_bwd_reduce(pend_d[norms], NL, 1 if norms else 0, spn):
                raise RuntimeError(lib.gnsb_last_error().decode())

        gr = {"fused": capture_graph(lambda: layer_step(True), torch, dev),
              "plain": capture_graph(lambda: layer_step(False), torch, dev),
              "aten": capture_graph(lambda: [e.run_aten(torch) for e in extra_cases], torch, dev)}
        sd = interleaved({k: g.replay for k, g in gr.items()}, max(args.steps, 15), stream, torch, np)
        ms_f, ms_p, ms_a = sd["fused"]["median"], sd["plain"]["median"], sd["aten"]["median"]
        gbs = NL * c.bytes / (ms_f * 1e-3) / 1e9
        sweep_rows[i].update({
            "steady_layers": NL, "steady_fused_GBps": gbs, "steady_frac_of_measured_peak": gbs / peak,
            "steady_fused_us_per_layer": ms_f * 1e3 / NL, "steady_fused_iqr_us": [v * 1e3 / NL for v in sd["fused"]["iqr"]],
            "steady_plain_GBps": NL * c.bytes_plain / (ms_p * 1e-3) / 1e9,
            "steady_plain_us_per_layer": ms_p * 1e3 / NL, "steady_plain_iqr_us": [v * 1e3 / NL for v in sd["plain"]["iqr"]],
            "steady_overhead_pct": 100.0 * (ms_f - ms_p) / ms_p,
            "steady_overhead_pct_iqr": sd["fused"]["paired_overhead_iqr"]["plain"],
            "steady_aten_us_per_layer": ms_a * 1e3 / NL, "steady_aten_GBps": NL * c.bytes_plain / (ms_a * 1e-3) / 1e9,
            "overhead_vs_aten_pct": 100.0 * (ms_f - ms_a) / ms_a,
            "overhead_vs_aten_pct_iqr": sd["fused"]["paired_overhead_iqr"]["aten"],
            "steady_timing": f"{NL} layers of this width (distinct buffers) + one grouped reduce per CUDA graph; "
                             "fused / plain / aten graphs replayed interleaved, median and interquartile range",
            "plain_def": "same kernels over one example of B*T rows (no per-example bookkeeping, no squares)",
            "aten_def": "torch.ops.aten.native_layer_norm_backward, bf16 rows/weight, fp32 mean/rstd, same buffers",
        })
        del extra_cases, gr
        torch.cuda.empty_cache()
    big = [r for r in sweep_rows if r["D"] >= 1024]
    overhead_ge1024 = 100.0 * (sum(r["fused_us"] for r in big) - sum(r["plain_us"] for r in big)) / max(
        sum(r["plain_us"] for r in big), 1e-9)
    step_bytes = sum(c.bytes for c in cases)
    achieved = step_bytes / (step_f * 1e-3) / 1e9

    clk.__exit__()
    # ---- e2e through the C ABI with host buffers ----
    e2e = run_e2e(args, m, lib, cases, dev, stream, torch, np)

    # ---- CPU baseline (rank 0, bounded sample) ----
    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = cpu_baseline(args)

    # ---- the dominant kernel alone: the row pass at the widest D of the sweep
    # (largest share of the step), back-to-back launches, events on its stream
    dom = max(cases, key=lambda c: c.D)
    for _ in range(3):
        dom.run_rows(sp)
    nrep = max(args.steps, 10)
    d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d0.record(stream)
    for _ in range(nrep):
        dom.run_rows(sp)
    d1.record(stream)
    torch.cuda.synchronize()
    dom_us = d0.elapsed_time(d1) * 1e3 / nrep
    dom_bytes = dom.bytes - 8 * dom.D - 16 * dom.B  # the row pass: all but the dgamma/dbeta and norm outputs
    dom_achieved = dom_bytes / (dom_us * 1e-6) / 1e9

    extra = {}
    if rank == 0 and not (args.no_extra or args.no_side):
        extra["ln_forward"] = run_ln_fwd(m, lib, cases, dev, torch, np)
        extra["cfg3_linear"] = run_cfg3(m, lib, dev, torch, np)
        extra["cfg4_gns"] = run_cfg4(m, lib, dev, torch, np)
        extra["cfg5_g1"] = run_cfg5(m, lib, dev, torch, np)
        # the G=1 point of the configs[4] strong-scaling curve, measured the way
        # `bench.py --gpus N` measures N > 1 (same step, exchange without a peer)
        extra["cfg5_strong_g1"] = Cfg5Strong(args, m, lib, dev, torch, np, 1, 0, "none").measure(args.steps,
                                                                                                args.warmup)
        extra["embedding"] = run_embedding(m, lib, dev, torch, np)
        extra["toy_model_step"] = run_toy_step(m, dev, torch, np)

    traffic = load_traffic()
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (SURVEY §8(d) recipe, generated on device)",
        "config": {"workload": WORKLOAD, "B": B_LOCAL, "T": T, "D": sweep, "global_batch": B_LOCAL * world,
                   "parallelism": f"dp{world}", "backend": backend if world > 1 else None,
                   "l2": "inputs larger than L2: a step streams %.2f GB (>> 126 MB L2) between reuses of any buffer"
                         % (step_bytes / 1e9),
                   "launch": "one CUDA graph per step (compute); N > 1: the bucket all-reduce eagerly after it",
                   "stage2": "deferred: row pass per layer, one grouped reduce launch per step (gnsb_ln_bwd_reduce)"},
        "overhead_pct": 100.0 * (step_f - step_p) / step_p, "overhead_pct_D_ge_1024": overhead_ge1024,
        "overhead_pct_iqr": st["fused"]["paired_overhead_iqr"]["plain"],
        "step_ms_fused": step_f, "step_ms_plain": step_p,
        "step_ms_fused_iqr": st["fused"]["iqr"], "step_ms_plain_iqr": st["plain"]["iqr"],
        "step_ms_aten": st["aten"]["median"] if "aten" in st else None,
        "overhead_vs_aten_pct": 100.0 * (step_f - st["aten"]["median"]) / st["aten"]["median"] if "aten" in st else None,
        "overhead_def": "fused step vs the plain LayerNorm backward step (same kernels over one example of B*T rows: "
                        "no per-example bookkeeping, no squares), interleaved graph replays, median; iqr of the "
                        "per-replay-pair overhead",
        "roofline": {"bound": "hbm", "achieved": dom_achieved, "peak": peak, "unit": "GB/s",
                     "frac": dom_achieved / peak, "peak_kind": peak_kind, "frac_of_8TBps": dom_achieved / 8000.0,
                     "traffic": traffic, "alg_bytes_per_launch": dom_bytes, "us_per_launch": dom_us,
                     "kernel": f"ln_bwd_kernel<bf16, D={dom.D}> row pass (largest share of the step)",
                     "achieved_def": "algorithmic bytes per launch / CUDA-event duration, back-to-back launches"},
        "roofline_step": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                          "frac_of_8TBps": achieved / 8000.0,
                          "kernels": "5 row passes (one per D) + one ln_bwd_reduce_group_kernel<float,NORMS=1>",
                          "achieved_def": "algorithmic bytes of the step / median graph-replayed step time"},
        "sweep": sweep_rows, "e2e": e2e, "cpu_baseline": cpu, **extra,
        "gpu_launches": (len(cases) + 1 + (2 * len(cases) if world > 1 else 0)) * args.steps, "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def time_graph(fn, torch, np, dev, reps=10, warm=3):
    """Median device time (ms) of fn() replayed as one CUDA graph (events on the
    capturing stream)."""
    side = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(side):
        for _ in range(warm):
            fn()
    torch.cuda.current_stream(dev).wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(warm):
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def capture_graph(fn, torch, dev, warm=3):
    """fn() captured as one CUDA graph (after warm-up on a side stream)."""
    side = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(side):
        for _ in range(warm):
            fn()
    torch.cuda.current_stream(dev).wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(warm):
        g.replay()
    torch.cuda.synchronize()
    return g


def interleaved(variants, reps, stream, torch, np):
    """Replay the variants round-robin (v1 v2 v3, v2 v3 v1, ...), each bracketed by
    CUDA events on `stream`, so slow drifts (clocks, temperature) hit all of
    them alike.  Per variant: median and interquartile range (ms), and per
    other variant the interquartile range of the paired overhead (%)."""
    ev = {k: [] for k in variants}
    names = list(variants)
    for r in range(reps):
        # rotate the order every replay round: each variant follows each other
        # one equally often (what the previous graph left in L2 -- dirty lines,
        # resident inputs -- biases whoever runs next)
        for k in names[r % len(names):] + names[:r % len(names)]:
            fn = variants[k]
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            ev[k].append((a, b))
    torch.cuda.synchronize()
    ts = {k: np.array([a.elapsed_time(b) for a, b in v]) for k, v in ev.items()}
    out = {}
    for k, t in ts.items():
        pair = {o: [float(x) for x in np.percentile(100.0 * (t - ts[o]) / ts[o], [25, 75])] for o in ts if o != k}
        out[k] = {"median": float(np.median(t)), "iqr": [float(x) for x in np.percentile(t, [25, 75])],
                  "paired_overhead_iqr": pair}
    return out


def run_ln_fwd(m, lib, cases, dev, torch, np):
    """LayerNorm forward (gnsb_ln_fwd: y, mean, rstd) at every D of the sweep:
    bytes = N*D*(s_in + s_out) + 8N + 8D.  Four back-to-back calls on distinct
    buffer sets per graph replay (steady state; > 400 MB moved per replay, so
    no call finds its input in L2), time per call."""
    out = []
    NS = 4
    for c in cases:
        N = c.B * T
        xs = [c.x] + [c.x.clone() for _ in range(NS - 1)]
        ys = [torch.empty_like(c.x) for _ in range(NS)]
        means = [torch.empty_like(c.mean) for _ in range(NS)]
        rstds = [torch.empty_like(c.rstd) for _ in range(NS)]

        def fn(c=c, xs=xs, ys=ys, means=means, rstds=rstds):
            sp = torch.cuda.current_stream(dev).cuda_stream
            for i in range(NS):
                rc = lib.gnsb_ln_fwd(xs[i].data_ptr(), c.gamma.data_ptr(), c.beta.data_ptr(), ys[i].data_ptr(),
                                     means[i].data_ptr(), rstds[i].data_ptr(), None, N, c.D, 1e-5, 1, sp)
                if rc:
                    raise RuntimeError(lib.gnsb_last_error().decode())

        ms = time_graph(fn, torch, np, dev, reps=10) / NS
        nbytes = N * c.D * 4 + 8 * N + 8 * c.D
        out.append({"D": c.D, "us": ms * 1e3, "GBps": nbytes / (ms * 1e-3) / 1e9,
                    "timing": f"{NS} calls on distinct buffers per CUDA graph replay, per call"})
        del xs, ys, means, rstds
        torch.cuda.empty_cache()
    return out


def run_cfg3(m, lib, dev, torch, np):
    """BASELINE config 3: per-example linear-layer norms, B=16 T=2048 K=L=4096 bf16,
    both forms on tcgen05 (weight-grad form also writes dW)."""
    import ctypes

    B, T_, K, L = 16, 2048, 4096, 4096
    x, g = m.synth_linear(B, T_, K, L, torch.bfloat16, dev)
    dW = torch.empty(K, L, device=dev)
    raw = torch.empty(B, dtype=torch.float64, device=dev)
    sums = torch.zeros(4, dtype=torch.float64, device=dev)
    n = ctypes.c_size_t()
    lib.gnsb_linear_pe_workspace_size(B, T_, K, L, 1, ctypes.byref(n))
    ws = torch.zeros(n.value, dtype=torch.uint8, device=dev)
    out = {"workload": "cfg3: per-example linear norms B=16 T=2048 K=L=4096 bf16 (fp32 accumulate)"}
    peak = 1695.1
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak = float(json.load(f)["bf16_tflops"])
    except Exception:
        pass
    for form, name in ((1, "weight_grad"), (2, "gram")):
        def fn(form=form):
            sp = torch.cuda.current_stream(dev).cuda_stream
            rc = lib.gnsb_linear_pe_norms(x.data_ptr(), g.data_ptr(), dW.data_ptr() if form == 1 else None,
                                          raw.data_ptr(), sums.data_ptr(), B, T_, K, L, form, 1, ws.data_ptr(),
                                          ws.numel(), sp)
            if rc:
                raise RuntimeError(lib.gnsb_last_error().decode())
        ms = time_graph(fn, torch, np, dev)
        # algorithmic FLOPs: weight-grad form 2BTKL; Gram form with symmetry
        # B*T^2*(K+L) (half of 2BT^2(K+L); the kernel executes ~12% more: 128x256 blocks on the diagonal)
        fl = 2.0 * B * T_ * K * L if form == 1 else 1.0 * B * T_ * T_ * (K + L)
        out[name] = {"us": ms * 1e3, "TFLOPs": fl / (ms * 1e-3) / 1e12, "frac_of_bf16_peak": fl / (ms * 1e-3) / 1e12 / peak,
                     "flops": fl}
    out["faster_form"] = min(("weight_grad", "gram"), key=lambda k: out[k]["us"])
    # the other half of linear_backward_simultaneous: dx = g W^T (gnsb_linear_dx,
    # tcgen05), and the forward y = x W (gnsb_linear_fwd); bf16 W operand
    Wb = (torch.randn(K, L, device=dev) / K ** 0.5).to(torch.bfloat16)
    ybuf = torch.empty(B * T_, K, dtype=torch.bfloat16, device=dev)
    for name, fnname, src in (("input_grad", "gnsb_linear_dx", g), ("forward", "gnsb_linear_fwd", x)):
        def fn(fnname=fnname, src=src):
            sp = torch.cuda.current_stream(dev).cuda_stream
            if fnname == "gnsb_linear_dx":
                rc = lib.gnsb_linear_dx(src.data_ptr(), Wb.data_ptr(), ybuf.data_ptr(), B * T_, K, L, 1, 1, None, 0, sp)
            else:
                rc = lib.gnsb_linear_fwd(src.data_ptr(), Wb.data_ptr(), None, ybuf.data_ptr(), B * T_, K, L, 1, 1,
                                         None, 0, sp)
            if rc:
                raise RuntimeError(lib.gnsb_last_error().decode())
        ms = time_graph(fn, torch, np, dev)
        fl = 2.0 * B * T_ * K * L
        out[name] = {"us": ms * 1e3, "TFLOPs": fl / (ms * 1e-3) / 1e12, "frac_of_bf16_peak": fl / (ms * 1e-3) / 1e12 / peak,
                     "flops": fl, "kernel": "gemm_kernel (tcgen05, 128x256 tiles, TMA ring)"}
    del x, g, dW, ws, Wb, ybuf
    torch.cuda.empty_cache()
    return out


def run_cfg4(m, lib, dev, torch, np):
    """BASELINE config 4: full GNS estimate over all 25 LayerNorms of a 12-layer
    D=768 transformer backward, B=64 T=1024 bf16: 25 fused LN backwards writing
    their records, then the device GNS step, one CUDA graph."""
    from paper_2411_00999_b200.gns import DeviceGnsAccumulator
    from paper_2411_00999_b200.sharded import GradBuckets

    NL, B, T_, D = 25, 64, 1024, 768
    bk = GradBuckets([D] * NL, dev)
    cases = []
    for l in range(NL):
        x, dy, gamma, beta = m.synth_ln(B, T_, D, torch.bfloat16, dev, sigma=3.0, stream0=16 * l)
        gamma.fill_(1.0)
        beta.zero_()
        f = m.layernorm_forward(m.LayerNormLayer(gamma, beta), x)
        dx = torch.empty_like(x)
        ws = torch.zeros(m.layers.ctypes_size(B, T_, D, 1), dtype=torch.uint8, device=dev)
        raw = torch.zeros(2, B, dtype=torch.float64, device=dev)
        cases.append((x, f.cache.mean, f.cache.inv_std, dy, gamma, dx, ws, raw))
    acc = DeviceGnsAccumulator(["layernorm"] * NL, 0.5, dev)

    from paper_2411_00999_b200 import _lib as L

    pend = (L.LnBwdPending * NL)(*[
        L.LnBwdPending(ws.data_ptr(), ws.numel(), B, T_, D, 1, bk.grad(l)[0].data_ptr(), bk.grad(l)[1].data_ptr(),
                       raw[0].data_ptr(), raw[1].data_ptr(), bk.record(l).data_ptr())
        for l, (x, mean, rstd, dy, gamma, dx, ws, raw) in enumerate(cases)])

    def fn():
        sp = torch.cuda.current_stream(dev).cuda_stream
        for l, (x, mean, rstd, dy, gamma, dx, ws, raw) in enumerate(cases):
            rc = lib.gnsb_ln_bwd_rows(x.data_ptr(), mean.data_ptr(), rstd.data_ptr(), dy.data_ptr(), gamma.data_ptr(),
                                      dx.data_ptr(), B, T_, D, 1, ws.data_ptr(), ws.numel(), sp)
            if rc:
                raise RuntimeError(lib.gnsb_last_error().decode())
        if lib.gnsb_ln_bwd_reduce(pend, NL, 1, sp):
            raise RuntimeError(lib.gnsb_last_error().decode())
        acc.step(bk.records, B)

    ms = time_graph(fn, torch, np, dev)
    nbytes = NL * alg_bytes(B, T_, D)
    groups = acc.groups.cpu().numpy()
    out = {"workload": "cfg4: GNS over 25 LayerNorms, B=64 T=1024 D=768 bf16, sigma=3 (synthetic)",
           "ms_per_step": ms, "GBps": nbytes / (ms * 1e-3) / 1e9, "alg_bytes": nbytes,
           "gns_total": {"g2": float(groups[0, 0]), "s": float(groups[0, 1]), "b_simple_ema": float(groups[0, 2])},
           "launches_per_step": NL + 2, "stage2": "deferred: one grouped reduce for the 25 layers"}
    del cases
    torch.cuda.empty_cache()
    return out


def run_toy_step(m, dev, torch, np):
    """SURVEY §8(f) rank 4 at GPT-2-small width: one training step (forward +
    backward) of the reference toy model (proj/src/model.cpp) with EVERY
    layer's per-example gradient norms and the device GNS step, all on the
    library's kernels (ToyModelPE.forward_backward, bf16 activations, fp32
    parameters), against the same architecture as an uninstrumented PyTorch
    step (cuBLAS, autograd, bf16 autocast, no per-example norms) -- the
    paper's deployment comparison.  Both graph-replayed."""
    from paper_2411_00999_b200.model import ToyModelPE
    from paper_2411_00999_b200.nn import GnsTracker

    V, D, HM, NB, B, T_ = 50304, 768, 4, 12, 8, 1024
    gen = torch.Generator(device="cpu").manual_seed(0)
    ids = torch.randint(0, V, (B, T_), generator=gen, dtype=torch.int32).to(dev)
    tg = torch.randint(0, V, (B, T_), generator=gen, dtype=torch.int32).to(dev)
    model = ToyModelPE(V, D, HM, NB, seed=1, device=dev)
    inst = model.instrumented_layers()
    tracker = GnsTracker([mod for _, mod in inst], alpha=0.9)
    nparam = sum(p.numel() for p in model.parameters())

    def ours():
        model.forward_backward(ids, tg, rows_dtype=torch.bfloat16, validate=False)
        tracker.step()

    ms_ours = time_graph(ours, torch, np, dev, reps=10)
    H = D * HM
    tm = torch.nn.ModuleDict({
        "emb": torch.nn.Embedding(V, D), "lnf": torch.nn.LayerNorm(D), "head": torch.nn.Linear(D, V),
        "lns": torch.nn.ModuleList([torch.nn.LayerNorm(D) for _ in range(NB)]),
        "fc1": torch.nn.ModuleList([torch.nn.Linear(D, H) for _ in range(NB)]),
        "fc2": torch.nn.ModuleList([torch.nn.Linear(H, D) for _ in range(NB)])}).to(dev)

    def plain():
        for p in tm.parameters():
            p.grad = None
        with torch.autocast("cuda", dtype=torch.bfloat16):
            x = tm["emb"](ids.long())
            for ln, f1, f2 in zip(tm["lns"], tm["fc1"], tm["fc2"]):
                x = x + f2(torch.tanh(f1(ln(x))))
            logits = tm["head"](tm["lnf"](x))
            loss = torch.nn.functional.cross_entropy(logits.reshape(-1, V).float(), tg.reshape(-1).long())
        loss.backward()

    ms_torch = time_graph(plain, torch, np, dev, reps=10)
    flops = 6.0 * nparam * B * T_
    peak_tf = 1647.2
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak_tf = float(json.load(f)["bf16_tflops"])
    except Exception:
        pass
    out = {"workload": f"toy model (proj/src/model.cpp) V={V} D={D} H={H} blocks={NB}, B={B} T={T_}: forward + "
                       f"backward + per-example norms of all {len(inst)} instrumented layers + device GNS step",
           "params": nparam, "flops_per_step": flops, "ms_ours": ms_ours, "ms_torch_uninstrumented": ms_torch,
           "ratio_ours_over_torch": ms_ours / ms_torch, "model_TFLOPs_ours": flops / ms_ours / 1e9,
           "mfu_ours": flops / ms_ours / 1e9 / peak_tf,
           "torch_def": "same architecture, cuBLAS + autograd, bf16 autocast, NO per-example norms"}
    del model, tm, tracker
    torch.cuda.empty_cache()
    return out


def run_embedding(m, lib, dev, torch, np):
    """embedding-table gradient + per-example norms at a
    GPT-2 embedding (B=32 T=1024 V=50257 D=768, bf16 gradient rows, fp32 dW).
    Algorithmic bytes: g + ids in, dW out (every table row is written)."""
    import ctypes

    B, T_, V, D = 32, 1024, 50257, 768
    gen = torch.Generator(device="cpu").manual_seed(0)
    ids = torch.randint(0, V, (B, T_), generator=gen, dtype=torch.int32).to(dev)
    g = torch.randn(B, T_, D, generator=gen).to(dev, torch.bfloat16)
    n = ctypes.c_size_t()
    lib.gnsb_embedding_pe_workspace_size(B, T_, V, D, 1, ctypes.byref(n))
    ws = torch.zeros(n.value, dtype=torch.uint8, device=dev)
    dW = torch.empty(V, D, device=dev)
    raw = torch.empty(B, dtype=torch.float64, device=dev)
    sums = torch.zeros(4, dtype=torch.float64, device=dev)

    def fn():
        sp = torch.cuda.current_stream(dev).cuda_stream
        rc = lib.gnsb_embedding_pe(ids.data_ptr(), g.data_ptr(), dW.data_ptr(), raw.data_ptr(), sums.data_ptr(), B,
                                   T_, V, D, 1, ws.data_ptr(), ws.numel(), None, sp)
        if rc:
            raise RuntimeError(lib.gnsb_last_error().decode())

    ms = time_graph(fn, torch, np, dev, reps=10)
    nbytes = B * T_ * D * 2 + B * T_ * 4 + V * D * 4
    peak, _ = load_peaks()
    out = {"workload": "embedding per-example norms B=32 T=1024 V=50257 D=768 bf16 rows, fp32 dW",
           "us": ms * 1e3, "GBps": nbytes / (ms * 1e-3) / 1e9, "frac_of_measured_peak":
           nbytes / (ms * 1e-3) / 1e9 / peak, "alg_bytes": nbytes}
    del ids, g, ws, dW
    torch.cuda.empty_cache()
    return out


def run_cfg5(m, lib, dev, torch, np):
    """BASELINE config 5 at G=1: the whole batch-sharded workload on one GPU,
    B=256 T=2048 D=4096 bf16 (12.9 GB per step), fused LN backward + norms.
    At G GPUs each rank runs B/G of these examples plus the bucket all-reduce."""
    B, T_, D = 256, 2048, 4096
    x, dy, gamma, beta = m.synth_ln(B, T_, D, torch.bfloat16, dev, B_div=B)
    f = m.layernorm_forward(m.LayerNormLayer(gamma, beta), x)
    dx = torch.empty_like(x)
    dg = torch.empty(D, device=dev)
    db = torch.empty(D, device=dev)
    raw = torch.zeros(2, B, dtype=torch.float64, device=dev)
    rec = torch.zeros(4, dtype=torch.float64, device=dev)
    ws = torch.zeros(m.layers.ctypes_size(B, T_, D, 1), dtype=torch.uint8, device=dev)
    mean, rstd = f.cache.mean, f.cache.inv_std

    def fn():
        sp = torch.cuda.current_stream(dev).cuda_stream
        rc = lib.gnsb_ln_bwd(x.data_ptr(), mean.data_ptr(), rstd.data_ptr(), dy.data_ptr(), gamma.data_ptr(),
                             dx.data_ptr(), dg.data_ptr(), db.data_ptr(), raw[0].data_ptr(), raw[1].data_ptr(),
                             rec.data_ptr(), 1, B, T_, D, 1, ws.data_ptr(), ws.numel(), sp)
        if rc:
            raise RuntimeError(lib.gnsb_last_error().decode())

    ms = time_graph(fn, torch, np, dev, reps=5)
    nbytes = alg_bytes(B, T_, D)
    peak, _ = load_peaks()
    out = {"workload": "cfg5 at G=1: LN bwd + per-example norms B=256 T=2048 D=4096 bf16",
           "ms_per_step": ms, "GBps": nbytes / (ms * 1e-3) / 1e9, "frac_of_measured_peak":
           nbytes / (ms * 1e-3) / 1e9 / peak, "alg_bytes": nbytes}
    del x, dy, dx, f, ws
    torch.cuda.empty_cache()
    return out


CFG5_WORKLOAD = ("cfg5: batch-sharded LN bwd + per-example norms + GNS, B_global=256 T=2048 D=4096 bf16, "
                 "strong scaling (B_global/N examples per GPU), one packed fp64 all-reduce per step")


class Cfg5Strong:
    """BASELINE.json configs[4]: the batch-sharded step at N GPUs, strong scaling.

    Rank r owns the contiguous examples [b0, b1) = shard_bounds(B_global, N, r)
    of a globally-indexed synthetic batch (dy scaled by 1/B_global), so every
    value is the same whichever rank holds it.  One step, captured as ONE CUDA
    graph on the NCCL path:
      gnsb_ln_bwd_rows (dx + per-(CTA, example) partials)
      gnsb_ln_bwd_reduce (per-example squares, dgamma/dbeta into the exchange bucket)
      gnsb_allreduce_buckets: pack -> ONE ncclAllReduce of the fp64 bucket
        {record, dgamma, dbeta} -> unpack (||G_big||^2 of the reduced gradients)
      gnsb_gns_step (B = B_global)
    The gloo test mode (several ranks on one device) runs the same kernels with
    the all-reduce of the packed buffer issued eagerly between two graphs.
    N = 1: the same step with no collective (pack -> unpack)."""

    def __init__(self, args, m, lib, dev, torch, np, world, rank, backend):
        import ctypes

        from paper_2411_00999_b200 import _lib
        from paper_2411_00999_b200.gns import DeviceGnsAccumulator
        from paper_2411_00999_b200.sharded import GradBuckets, NcclComm, shard_bounds

        self.torch, self.np, self.lib, self.dev = torch, np, lib, dev
        self.world, self.rank, self.backend = world, rank, backend
        Bg, T5, D5 = args.cfg5
        self.Bg, self.T5, self.D5 = Bg, T5, D5
        b0, b1 = shard_bounds(Bg, world, rank)
        self.b0, self.Bl = b0, b1 - b0
        bf = torch.bfloat16
        self.x, self.dy, self.gamma, self.beta = m.synth_ln(self.Bl, T5, D5, bf, dev, b_offset=b0, B_div=Bg)
        f = m.layernorm_forward(m.LayerNormLayer(self.gamma, self.beta), self.x)
        self.mean, self.rstd = f.cache.mean, f.cache.inv_std
        self.dx = torch.empty_like(self.x)
        self.bk = GradBuckets([D5], dev)
        self.raw = torch.zeros(2, self.Bl, dtype=torch.float64, device=dev)
        self.ws = torch.zeros(m.layers.ctypes_size(self.Bl, T5, D5, 1), dtype=torch.uint8, device=dev)
        dg, db = self.bk.grad(0)
        self.pend = (_lib.LnBwdPending * 1)(_lib.LnBwdPending(
            self.ws.data_ptr(), self.ws.numel(), self.Bl, T5, D5, 1, dg.data_ptr(), db.data_ptr(),
            self.raw[0].data_ptr(), self.raw[1].data_ptr(), self.bk.record(0).data_ptr()))
        self.acc = DeviceGnsAccumulator(["layernorm"], 0.5, dev)
        self.comm = NcclComm() if (world > 1 and backend == "nccl") else None
        self.bytes_local = alg_bytes(self.Bl, T5, D5)
        self.bytes_local_plain = alg_bytes(self.Bl, T5, D5, norms=False)
        self.rows_bytes = self.bytes_local - 8 * D5 - 16 * self.Bl
        self.graph_all = world == 1 or self.comm is not None
        self.packed_bytes = 8 * (4 + 2 * D5)
        self._graphs = {}
        self._ctypes = ctypes

    # ---------------------------------------------------------------- pieces
    def rows(self, sp):
        p = lambda t: t.data_ptr()
        if self.lib.gnsb_ln_bwd_rows(p(self.x), p(self.mean), p(self.rstd), p(self.dy), p(self.gamma), p(self.dx),
                                     self.Bl, self.T5, self.D5, 1, p(self.ws), self.ws.numel(), sp):
            raise RuntimeError(self.lib.gnsb_last_error().decode())

    def compute(self, norms):
        sp = self.torch.cuda.current_stream(self.dev).cuda_stream
        self.rows(sp)
        if self.lib.gnsb_ln_bwd_reduce(self.pend, 1, 1 if norms else 0, sp):
            raise RuntimeError(self.lib.gnsb_last_error().decode())

    def head(self, norms):
        """Graph part 1: compute, then the exchange (NCCL / one rank) or its pack (gloo)."""
        self.compute(norms)
        if self.graph_all:
            self.bk.allreduce_nccl(self.comm, records=norms)
            if norms:
                self.acc.step(self.bk.records, self.Bg)
        else:
            self.bk.pack(records=norms)

    def tail(self, norms):
        """gloo only: the collective on the packed buffer, then unpack + GNS step."""
        import torch.distributed as dist

        dist.all_reduce(self.bk.packed(records=norms))
        self.bk.unpack(records=norms)
        if norms:
            self.acc.step(self.bk.records, self.Bg)

    def launches_per_step(self, norms=True):
        # rows, reduce, pack, unpack (+ gns step); the NCCL kernel is not ours
        return 4 + (1 if norms else 0)

    def capture(self):
        torch = self.torch
        side = torch.cuda.Stream(self.dev)
        side.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(side):
            for norms in (True, False):
                self.head(norms)
                if not self.graph_all:
                    self.tail(norms)
        torch.cuda.current_stream(self.dev).wait_stream(side)
        torch.cuda.synchronize()
        for norms in (True, False):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, capture_error_mode="thread_local"):
                self.head(norms)
            self._graphs[norms] = g
        torch.cuda.synchronize()

    def step(self, norms=True):
        self._graphs[norms].replay()
        if not self.graph_all:
            self.tail(norms)

    def _barrier(self):
        import torch.distributed as dist

        if self.world > 1:
            dist.barrier()

    def _max(self, v):
        import torch.distributed as dist

        t = self.torch.tensor([v], dtype=self.torch.float64, device=self.dev)
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def _sum(self, v):
        import torch.distributed as dist

        t = self.torch.tensor([v], dtype=self.torch.float64, device=self.dev)
        if self.world > 1:
            dist.all_reduce(t)
        return float(t.item())

    def timed_steps(self, k, norms=True):
        """K steps between barrier + synchronize, device time (events on the
        replay stream), max over ranks (ms)."""
        torch = self.torch
        self._barrier()
        torch.cuda.synchronize()
        st = torch.cuda.current_stream(self.dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(k):
            self.step(norms)
        e1.record(st)
        torch.cuda.synchronize()
        self._barrier()
        return self._max(e0.elapsed_time(e1))

    def measure(self, steps, warmup, clocks=None):
        torch, np = self.torch, self.np
        if not self._graphs:
            self.capture()
        for _ in range(warmup):
            self.step(True)
            self.step(False)
        torch.cuda.synchronize()
        if clocks is not None:
            clocks.__enter__()
            time.sleep(0.3)
        t_ms = self.timed_steps(steps, True)
        total_bytes = self._sum(self.bytes_local)
        value = total_bytes * steps / (t_ms * 1e-3) / 1e9
        # fused vs plain twin (plain: no squares, gradients-only exchange, no GNS
        # step), alternating blocks of steps; median + IQR of the per-block ratio
        kb = max(3, min(steps, 10))
        ov, tf, tp = [], [], []
        for _ in range(7):
            a = self.timed_steps(kb, True)
            b = self.timed_steps(kb, False)
            tf.append(a / kb)
            tp.append(b / kb)
            ov.append(100.0 * (a - b) / b)
        # the exchange alone (graph of gnsb_allreduce_buckets), and the row pass
        # alone back to back (the dominant kernel), max over ranks
        ex_us = None
        if self.graph_all:
            from paper_2411_00999_b200 import _lib  # noqa: F401

            ex_ms = time_graph(lambda: self.bk.allreduce_nccl(self.comm, records=True), torch, np, self.dev, reps=20)
            ex_us = self._max(ex_ms * 1e3)
        st = torch.cuda.current_stream(self.dev)
        sp = st.cuda_stream
        for _ in range(3):
            self.rows(sp)
        nrep = max(steps, 10)
        self._barrier()
        torch.cuda.synchronize()
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record(st)
        for _ in range(nrep):
            self.rows(sp)
        d1.record(st)
        torch.cuda.synchronize()
        rows_us = self._max(d0.elapsed_time(d1) * 1e3 / nrep)
        if clocks is not None:
            clocks.__exit__()
        peak, peak_kind = load_peaks()
        per_gpu = value / self.world
        q = lambda v: [float(np.percentile(v, 25)), float(np.percentile(v, 75))]
        return {
            "workload": CFG5_WORKLOAD, "n_gpus": self.world, "value": value, "unit": "GB/s",
            "ms_per_step": t_ms / steps, "steps": steps, "B_global": self.Bg, "B_per_gpu_rank0": self.Bl,
            "T": self.T5, "D": self.D5, "per_gpu_GBps": per_gpu, "frac_of_measured_peak_per_gpu": per_gpu / peak,
            "overhead_pct": float(np.median(ov)), "overhead_pct_iqr": q(ov),
            "step_ms_fused": float(np.median(tf)), "step_ms_plain": float(np.median(tp)),
            "exchange_us": ex_us, "exchange_bytes": self.packed_bytes,
            "exchange": ("gnsb_allreduce_buckets: pack, one ncclAllReduce(fp64, %d B), unpack, in the step graph"
                         % self.packed_bytes) if self.comm is not None else (
                "pack, unpack (one rank: no collective)" if self.world == 1 else
                "pack, torch.distributed all_reduce of the packed fp64 buffer (%s), unpack" % self.backend),
            "rows_us": rows_us, "rows_GBps": self.rows_bytes / (rows_us * 1e-6) / 1e9,
            "rows_frac_of_measured_peak": self.rows_bytes / (rows_us * 1e-6) / 1e9 / peak,
            "rows_alg_bytes": self.rows_bytes, "peak": peak, "peak_kind": peak_kind,
            "gpu_launches_per_step": self.launches_per_step(True),
            "collectives_per_step": 1 if self.world > 1 else 0,
        }

    def e2e(self, steps):
        """The same step through the C ABI with this rank's shard in pinned host
        memory: H2D of x, dy, mean, rstd; the step; D2H of dx, dgamma, dbeta,
        the per-example norms and the record.  Max over ranks."""
        torch = self.torch
        h = {k: getattr(self, k).cpu().pin_memory() for k in ("x", "dy", "mean", "rstd")}
        hdx = torch.empty(self.dx.shape, dtype=self.dx.dtype).pin_memory()
        hg = torch.empty(self.bk.grads.shape, dtype=self.bk.grads.dtype).pin_memory()
        hraw = torch.empty(self.raw.shape, dtype=self.raw.dtype).pin_memory()
        hrec = torch.empty(self.bk.records.shape, dtype=torch.float64).pin_memory()
        h2d = sum(v.numel() * v.element_size() for v in h.values())
        d2h = hdx.numel() * 2 + hg.numel() * 4 + hraw.numel() * 8 + hrec.numel() * 8

        def one():
            for k, v in h.items():
                getattr(self, k).copy_(v, non_blocking=True)
            self.step(True)
            hdx.copy_(self.dx, non_blocking=True)
            hg.copy_(self.bk.grads, non_blocking=True)
            hraw.copy_(self.raw, non_blocking=True)
            hrec.copy_(self.bk.records, non_blocking=True)

        one()
        torch.cuda.synchronize()
        k = max(3, min(steps, 5))
        self._barrier()
        torch.cuda.synchronize()
        st = torch.cuda.current_stream(self.dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(k):
            one()
        e1.record(st)
        torch.cuda.synchronize()
        self._barrier()
        ms = self._max(e0.elapsed_time(e1)) / k
        total = self._sum(self.bytes_local)
        return {"value": total / (ms * 1e-3) / 1e9, "unit": "GB/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": ms, "steps": k,
                "path": "per rank: pinned host shard -> H2D -> step graph (C ABI kernels + exchange) -> D2H, "
                        "one stream, max over ranks"}

    def close(self):
        if self.comm is not None:
            self.comm.close()


def run_sharded_main(args, m, lib, dev, torch, np, world, rank, local, backend):
    """N > 1: BASELINE.json configs[4], strong scaling."""
    import torch.distributed as dist

    c5 = Cfg5Strong(args, m, lib, dev, torch, np, world, rank, backend)
    clk = ClockSampler(local)
    r = c5.measure(args.steps, args.warmup, clocks=clk)
    e2e = c5.e2e(args.steps)
    line = {
        "metric": METRIC, "value": r["value"], "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (SURVEY §8(d) recipe, global example index, on device)",
        "config": {"workload": CFG5_WORKLOAD, "B_global": c5.Bg, "T": c5.T5, "D": c5.D5, "global_batch": c5.Bg,
                   "parallelism": f"dp{world}", "backend": backend,
                   "l2": "inputs larger than L2: %.2f GB per rank per step" % (c5.bytes_local / 1e9),
                   "launch": "one CUDA graph per step incl. the NCCL all-reduce" if c5.graph_all else
                             "two CUDA graphs per step around the eager gloo all-reduce (test mode)"},
        "overhead_pct": r["overhead_pct"], "overhead_pct_iqr": r["overhead_pct_iqr"],
        "step_ms_fused": r["step_ms_fused"], "step_ms_plain": r["step_ms_plain"],
        "per_gpu_GBps": r["per_gpu_GBps"], "frac_of_measured_peak_per_gpu": r["frac_of_measured_peak_per_gpu"],
        "exchange": r["exchange"], "exchange_us": r["exchange_us"], "collectives_per_step": 1,
        "roofline": {"bound": "hbm", "achieved": r["rows_GBps"], "peak": r["peak"], "unit": "GB/s",
                     "frac": r["rows_frac_of_measured_peak"], "peak_kind": r["peak_kind"], "traffic": None,
                     "alg_bytes_per_launch": r["rows_alg_bytes"], "us_per_launch": r["rows_us"],
                     "kernel": f"ln_bwd_kernel<bf16, D={c5.D5}> row pass, {c5.Bl} examples per rank",
                     "achieved_def": "algorithmic bytes per launch / CUDA-event duration, back-to-back, max over ranks"},
        "e2e": e2e, "cpu_baseline": None, "gpu_launches": r["gpu_launches_per_step"] * args.steps,
        "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    c5.close()
    dist.destroy_process_group()
    return 0


def run_e2e(args, m, lib, cases, dev, stream, torch, np):
    """Same metric through the public C ABI with host-resident inputs/outputs."""
    sp = stream.cuda_stream
    host = []
    for c in cases:
        h = {
            "x": c.x.cpu().pin_memory(), "dy": c.dy.cpu().pin_memory(), "mean": c.mean.cpu().pin_memory(),
            "rstd": c.rstd.cpu().pin_memory(), "dx": torch.empty(c.dx.shape, dtype=c.dx.dtype).pin_memory(),
            "dgamma": torch.empty(c.D, dtype=torch.float32).pin_memory(),
            "dbeta": torch.empty(c.D, dtype=torch.float32).pin_memory(),
            "sums": torch.empty(4, dtype=torch.float64).pin_memory(),
            "raw_g": torch.empty(c.B, dtype=torch.float64).pin_memory(),
            "raw_b": torch.empty(c.B, dtype=torch.float64).pin_memory(),
        }
        host.append(h)
    h2d = sum(h["x"].numel() * 2 + h["dy"].numel() * 2 + h["mean"].numel() * 4 + h["rstd"].numel() * 4 for h in host)
    d2h = sum(h["dx"].numel() * 2 + 2 * c.D * 4 + 32 + 16 * c.B for h, c in zip(host, cases))

    # Three streams: host->device copies, the kernels, device->host copies.
    # Layer l's kernel waits for its inputs; its outputs go back while the
    # next layer computes and the one after uploads (PCIe is full duplex).
    # Per-layer device buffers are reused across steps, so a step's upload of
    # layer l waits for the previous step's kernel l, and kernel l waits for
    # the previous step's download of layer l.
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    n = len(cases)
    comp_done = [None] * n
    out_done = [None] * n

    def step():
        for l, (c, h) in enumerate(zip(cases, host)):
            with torch.cuda.stream(s_in):
                if comp_done[l] is not None:
                    s_in.wait_event(comp_done[l])
                c.x.copy_(h["x"], non_blocking=True)
                c.dy.copy_(h["dy"], non_blocking=True)
                c.mean.copy_(h["mean"], non_blocking=True)
                c.rstd.copy_(h["rstd"], non_blocking=True)
                in_done = torch.cuda.Event()
                in_done.record(s_in)
            stream.wait_event(in_done)
            if out_done[l] is not None:
                stream.wait_event(out_done[l])
            c.run(True, sp)
            comp_done[l] = torch.cuda.Event()
            comp_done[l].record(stream)
            with torch.cuda.stream(s_out):
                s_out.wait_event(comp_done[l])
                h["dx"].copy_(c.dx, non_blocking=True)
                h["dgamma"].copy_(c.dgamma, non_blocking=True)
                h["dbeta"].copy_(c.dbeta, non_blocking=True)
                h["sums"].copy_(c.sums, non_blocking=True)
                h["raw_g"].copy_(c.raw_g, non_blocking=True)
                h["raw_b"].copy_(c.raw_b, non_blocking=True)
                out_done[l] = torch.cuda.Event()
                out_done[l].record(s_out)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    k = max(3, min(args.steps, 10))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s_in)
    stream.wait_stream(s_in)
    s_out.wait_stream(s_in)
    for _ in range(k):
        step()
    s_out.wait_stream(stream)
    s_out.wait_stream(s_in)
    e1.record(s_out)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / k
    value = sum(c.bytes for c in cases) / (ms * 1e-3) / 1e9
    return {"value": value, "unit": "GB/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": ms, "steps": k,
            "path": "gnsb_ln_bwd (C ABI) with pinned host buffers; H2D, kernels and D2H on three streams, "
                    "copies inside the timing"}


def cpu_baseline(args):
    from oracle import ffi

    if not ffi.reference_available():
        return None
    ref, orc = ffi.reference(), ffi.oracle()
    threads = os.cpu_count() or 1
    b_sample = min(B_LOCAL, threads)
    t0 = time.perf_counter()
    tsum, nbytes = 0.0, 0
    for D in args.d_list:
        tsum += ref_layer_sample(ref, orc, D, b_sample, threads)
        nbytes += alg_bytes(b_sample, T, D)
        if time.perf_counter() - t0 > 60:
            break
    # the reference is single-threaded by design: one example per
    # width on one core as well
    t1, n1 = 0.0, 0
    for D in args.d_list:
        t1 += ref_layer_sample(ref, orc, D, 1, 1)
        n1 += alg_bytes(1, T, D)
    return {"value": nbytes / tsum / 1e9, "unit": "GB/s", "cores": threads, "kind": "reference",
            "value_1core": n1 / t1 / 1e9,
            "sample": f"{b_sample} examples x T={T} per D (one pass of the sweep), reference gnstk fp64 "
                      f"layernorm_backward_simultaneous over {threads} threads; bytes by the bf16 workload formula; "
                      f"value_1core: 1 example per D on one thread"}


def load_traffic():
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get("ln_rows_bf16_D8192_bytes_per_launch")
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--d-list", type=lambda s: [int(v) for v in s.split(",")], default=SWEEP_D)
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-extra", action="store_true", help="skip the per-width steady runs and the side measurements")
    ap.add_argument("--no-side", action="store_true", help="skip the side measurements (forward, configs 3/4/5)")
    ap.add_argument("--cfg5", type=lambda s: [int(v) for v in s.split(",")], default=[256, 2048, 4096],
                    help="B_global,T,D of the N > 1 strong-scaling step (BASELINE configs[4]; smaller for tests)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
