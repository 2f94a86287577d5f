"""Timeline of the steady LayerNorm-backward step: NL row passes of one width
(distinct buffers) + one grouped reduce, replayed as a CUDA graph, with
per-CTA %globaltimer stamps of every row pass (experiment only).

Per layer: kernel start, griddepcontrol.wait exit, row math end and fold
end, relative to the first layer's start (us).  --notrace: timing only;
--lib=TAG: experiments/libln_sweep_TAG.so (scripts/ab_build.sh).

usage: python experiments/ln_steady_trace.py [D,D,...] [NL] [--plain]
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_00999_b200 as m  # noqa: E402
from paper_2411_00999_b200 import _lib  # noqa: E402

LIBTAG = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--lib=")), None)
sw = ctypes.CDLL(os.path.join(ROOT, "experiments", f"libln_sweep_{LIBTAG}.so" if LIBTAG else "libln_sweep.so"))
_vp, _i64 = ctypes.c_void_p, ctypes.c_int64
sw.sweep_rows_prod.argtypes = [_vp] * 6 + [_i64, _i64, _i64, _vp, ctypes.c_size_t, _vp, _vp]
sw.sweep_rows_prod.restype = ctypes.c_int
sw.sweep_reduce.restype = ctypes.c_int
lib = _lib.lib()
dev = torch.device("cuda")
B, T = 32, 1024
Ds = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1024, 2048]
NL = int(sys.argv[2]) if len(sys.argv) > 2 else 8
PLAIN = "--plain" in sys.argv
NOTRACE = "--notrace" in sys.argv  # timing only (the per-stage stamps perturb the kernel)
NORED = "--noreduce" in sys.argv
REDTRACE = "--redtrace" in sys.argv  # per-CTA stamps of the grouped reduce  # row passes only (the grouped reduce's share of the step)
SMS = torch.cuda.get_device_properties(dev).multi_processor_count
P = lambda t: ctypes.c_void_p(t.data_ptr())

for D in Ds:
    Bv, Mv = (1, B * T) if PLAIN else (B, T)
    layers = []
    for l in range(NL):
        x, dy, gamma, beta = m.synth_ln(B, T, D, torch.bfloat16, dev, b_offset=l * B)
        f = m.layernorm_forward(m.LayerNormLayer(gamma, beta), x)
        nb = m.layers.ctypes_size(Bv, Mv, D, 1)
        L = dict(x=x, dy=dy, gamma=gamma, mean=f.cache.mean, rstd=f.cache.inv_std, dx=torch.empty_like(x),
                 ws=torch.zeros(nb, dtype=torch.uint8, device=dev), dg=torch.empty(D, device=dev),
                 db=torch.empty(D, device=dev), rg=torch.zeros(Bv, dtype=torch.float64, device=dev),
                 rb=torch.zeros(Bv, dtype=torch.float64, device=dev),
                 sums=torch.zeros(4, dtype=torch.float64, device=dev),
                 trace=torch.zeros(SMS * 6, dtype=torch.int64, device=dev))
        layers.append(L)
    pend = (_lib.LnBwdPending * NL)(*[
        _lib.LnBwdPending(L["ws"].data_ptr(), L["ws"].numel(), Bv, Mv, D, 1, L["dg"].data_ptr(), L["db"].data_ptr(),
                          L["rg"].data_ptr(), L["rb"].data_ptr(), L["sums"].data_ptr()) for L in layers])

    rtrace = torch.zeros(4 * SMS * 6, dtype=torch.int64, device=dev)

    def step():
        sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        for L in layers:
            rc = sw.sweep_rows_prod(P(L["x"]), P(L["mean"]), P(L["rstd"]), P(L["dy"]), P(L["gamma"]), P(L["dx"]),
                                    Bv, Mv, D, P(L["ws"]), L["ws"].numel(), sp,
                                    None if NOTRACE else P(L["trace"]))
            assert rc == 0, rc
        if NORED:
            return
        if REDTRACE:
            arr = lambda key: (ctypes.c_void_p * NL)(*[L[key].data_ptr() for L in layers])
            meta = (ctypes.c_int64 * (3 * NL))(*([Bv, Mv, D] * NL))
            assert sw.sweep_reduce(NL, meta, arr("ws"), arr("dg"), arr("db"), arr("rg"), arr("rb"), arr("sums"),
                                   0 if PLAIN else 1, sp, P(rtrace)) == 0
        else:
            assert lib.gnsb_ln_bwd_reduce(pend, NL, 0 if PLAIN else 1, sp) == 0

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            step()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    nbytes = B * T * D * 6 + 8 * B * T
    print(f"[{LIBTAG or 'wt'}] D={D} {'plain' if PLAIN else 'fused'}{' noreduce' if NORED else ''}: step {ms*1e3:.1f} us for {NL} layers -> "
          f"{NL*nbytes/ms/1e6:.0f} GB/s ({NL*nbytes/ms/1e6/6558.1*100:.1f} % of 6558)")
    if REDTRACE:
        g.replay()
        torch.cuda.synchronize()
        rt = rtrace.view(-1, 6).cpu().numpy().astype(np.int64)
        rt = rt[rt[:, 0] > 0]
        t0 = rt[:, 0].min()
        r = (rt - t0) / 1000.0
        q = lambda a: f"{np.min(a):6.2f}/{np.median(a):6.2f}/{np.max(a):6.2f}"
        last = r[rt[:, 3] > 0]
        print(f"  reduce ({len(rt)} CTAs, us from first wait exit, min/med/max): wait-exit {q(r[:,0])} "
              f"first-stage {q(r[:,1])} items {q(r[:,5])} main-end {q(r[:,2])} | last CTAs: start {q(last[:,3])} end {q(last[:,4])}")
        rtrace.zero_()
    if NOTRACE:
        continue
    g.replay()
    torch.cuda.synchronize()
    trs = [L["trace"].view(SMS, 6).cpu().numpy().astype(np.int64) for L in layers]
    t0 = trs[0][:, 0].min()
    prev_end = None
    per_cta_rows = np.array([(c + 1) * B * T // SMS - c * B * T // SMS for c in range(SMS)])
    for l, tr in enumerate(trs):
        r = (tr - t0) / 1000.0
        med = lambda a: float(np.median(a))
        gap = f" gap(prev fold end -> wait exit) {r[:,3].min() - prev_end:5.2f}" if prev_end is not None else ""
        print(f"  L{l}: start {r[:,0].min():7.2f}..{r[:,0].max():7.2f} wait-exit {r[:,3].min():7.2f}..{r[:,3].max():7.2f}"
              f" rows-end {r[:,1].min():7.2f}/{med(r[:,1]):7.2f}/{r[:,1].max():7.2f} fold-end {r[:,2].max():7.2f}{gap}")
        prev_end = r[:, 2].max()
    # is the SM-to-SM spread systematic?  per-CTA row time (wait exit -> rows end)
    # of consecutive layers: correlation and the slowest CTAs
    dur = np.array([(tr[:, 1] - tr[:, 3]) / 1000.0 for tr in trs])
    cc = [float(np.corrcoef(dur[l], dur[l + 1])[0, 1]) for l in range(len(trs) - 1)]
    print(f"  per-CTA row time corr(layer l, l+1): {' '.join(f'{c:.2f}' for c in cc)}")
    print(f"  slowest CTAs L1: {np.argsort(-dur[1])[:12].tolist()}  L5: {np.argsort(-dur[5 % len(trs)])[:12].tolist()}")
    rows = [(c * Bv * Mv // SMS, (c + 1) * Bv * Mv // SMS) for c in range(SMS)]
    bnd = np.array([(r1 - 1) // Mv != r0 // Mv for r0, r1 in rows])
    mdur = dur.mean(0)
    print(f"  mean row time: CTAs with an example boundary {mdur[bnd].mean():.2f} us (n={int(bnd.sum())}, "
          f"max {mdur[bnd].max():.2f}), without {mdur[~bnd].mean():.2f} us (n={int((~bnd).sum())}, max {mdur[~bnd].max():.2f})")
    fold = np.array([(tr[:, 2] - tr[:, 1]) / 1000.0 for tr in trs]).mean(0)
    print(f"  mean fold time: boundary CTAs {fold[bnd].mean():.2f} us, others {fold[~bnd].mean():.2f} us")
    print(f"  row time min/med/max per layer: " + " | ".join(f"{d.min():.1f}/{np.median(d):.1f}/{d.max():.1f}" for d in dur))
    for L in layers:
        L.clear()
    torch.cuda.empty_cache()
