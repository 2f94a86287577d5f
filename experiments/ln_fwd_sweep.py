"""LayerNorm forward variants at the cfg2 widths (bf16, B=32 T=1024): the product
gnsb_ln_fwd vs the warp-per-row kernel (vectors per lane x CTAs per SM).  8
distinct buffer sets replayed in one CUDA graph (no L2 reuse between launches),
median over replays; outputs checked against the product kernel."""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_00999_b200 as m  # noqa: E402
from paper_2411_00999_b200 import _lib  # noqa: E402

ex = ctypes.CDLL(os.path.join(ROOT, "experiments", "libln_fwd_sweep.so"))
lib = _lib.lib()
dev = torch.device("cuda")
B, T, NS = 32, 1024, 8


def timed(fn):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(15):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2] / NS


for D in [int(v) for v in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["768", "1024", "2048", "4096"])]:
    N = B * T
    sets = []
    for i in range(NS):
        x, dy, gamma, beta = m.synth_ln(B, T, D, torch.bfloat16, dev, stream0=16 * i)
        del dy
        sets.append(dict(x=x, gamma=gamma, beta=beta, y=torch.empty_like(x), mean=torch.empty(N, device=dev),
                         rstd=torch.empty(N, device=dev)))
    nbytes = N * D * 4 + 8 * N + 8 * D

    def prod():
        sp = torch.cuda.current_stream().cuda_stream
        for s in sets:
            _lib.check(lib.gnsb_ln_fwd(s["x"].data_ptr(), s["gamma"].data_ptr(), s["beta"].data_ptr(),
                                       s["y"].data_ptr(), s["mean"].data_ptr(), s["rstd"].data_ptr(), None, N, D,
                                       1e-5, 1, sp))
    t = timed(prod)
    print(f"D={D} product        : {t*1e3:7.1f} us {nbytes/t/1e6:6.0f} GB/s", flush=True)
    ref = [(s["y"].clone(), s["mean"].clone(), s["rstd"].clone()) for s in sets[:1]]
    for cfg in ({4096: (0, 6, 7, 8), 8192: (10, 14, 16, 17, 18)}.get(D, ())):
        for smax in (8, 16, 32):
            def ring(cfg=cfg, smax=smax):
                sp = torch.cuda.current_stream().cuda_stream
                for s in sets:
                    rc = ex.fwd_ring_run(cfg, smax, ctypes.c_void_p(s["x"].data_ptr()), ctypes.c_void_p(s["gamma"].data_ptr()),
                                         ctypes.c_void_p(s["beta"].data_ptr()), ctypes.c_void_p(s["y"].data_ptr()),
                                         ctypes.c_void_p(s["mean"].data_ptr()), ctypes.c_void_p(s["rstd"].data_ptr()),
                                         ctypes.c_longlong(N), ctypes.c_longlong(D), ctypes.c_void_p(sp))
                    assert rc == 0, (cfg, rc)
            try:
                t = timed(ring)
            except AssertionError as e:
                print(f"D={D} ring cfg={cfg}: {e}")
                continue
            y, mu, rs = ref[0]
            dy_ = (sets[0]["y"].float() - y.float()).abs().max().item()
            print(f"D={D} ring cfg={cfg:2d} smax={smax:2d}: {t*1e3:7.1f} us {nbytes/t/1e6:6.0f} GB/s  |dy|={dy_:.1e}", flush=True)
    vpt = {768: 3, 1024: 4, 2048: 8, 4096: 16}.get(D)
    if vpt is None:
        continue
    combos = {3: [(1, 1), (4, 1), (4, 0), (6, 0)], 4: [(1, 1), (3, 1), (4, 0), (6, 0)],
              8: [(1, 1), (2, 1), (2, 0), (3, 0), (4, 0)], 16: [(1, 0), (2, 0), (3, 0)], 32: [(1, 0)]}[vpt]
    for minb, pf in combos:
        for bps in (1, 2, 3, 4, 6, 8):
            def warp(vpt=vpt, bps=bps, minb=minb, pf=pf):
                sp = torch.cuda.current_stream().cuda_stream
                for s in sets:
                    rc = ex.fwd_warp_run(vpt, minb, pf, bps, ctypes.c_void_p(s["x"].data_ptr()), ctypes.c_void_p(s["gamma"].data_ptr()),
                                         ctypes.c_void_p(s["beta"].data_ptr()), ctypes.c_void_p(s["y"].data_ptr()),
                                         ctypes.c_void_p(s["mean"].data_ptr()), ctypes.c_void_p(s["rstd"].data_ptr()),
                                         ctypes.c_longlong(N), ctypes.c_longlong(D), ctypes.c_void_p(sp))
                    assert rc == 0, rc
            t = timed(warp)
            y, mu, rs = ref[0]
            s = sets[0]
            dy_ = (s["y"].float() - y.float()).abs().max().item()
            print(f"D={D} warp vpt={vpt} minb={minb} pf={pf} bps={bps:2d}: {t*1e3:7.1f} us {nbytes/t/1e6:6.0f} GB/s  |dy|={dy_:.1e}",
                  flush=True)
    del sets
    torch.cuda.empty_cache()
