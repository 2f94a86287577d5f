"""Steady-state sweep of the LN-bwd configurations of experiments/ln_sweep.cu
(bf16, B=32 T=1024): per config, NL row passes of one width (distinct
buffers) + one grouped stage 2, replayed as a CUDA graph -- bench.py's
per-width "steady" measurement, for every config that fits the width.
Fused and plain (B=1 view of the same rows: no per-example bookkeeping).

usage: python experiments/ln_sweep_steady.py D[,D..] [ids] [--lib=TAG]"""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_00999_b200 as m  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
TAG = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--lib=")), None)
sw = ctypes.CDLL(os.path.join(ROOT, "experiments", f"libln_sweep_{TAG}.so" if TAG else "libln_sweep.so"))
VP = ctypes.c_void_p
sw.sweep_step.argtypes = [ctypes.c_int, ctypes.c_int] + [VP] * 11 + [ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                                                     ctypes.c_int64, VP, ctypes.c_size_t, VP]
sw.sweep_step.restype = ctypes.c_int
dev = torch.device("cuda")
B, T, NL = 32, 1024, 8
Ds = [int(v) for v in args[0].split(",")] if args else [768, 1024, 2048]
ids = [int(v) for v in args[1].split(",")] if len(args) > 1 else list(range(sw.sweep_n()))
WS = 64 << 20
for D in Ds:
    L = []
    for l in range(NL):
        x, dy, gamma, beta = m.synth_ln(B, T, D, torch.bfloat16, dev, b_offset=l * B)
        f = m.layernorm_forward(m.LayerNormLayer(gamma, beta), x)
        L.append(dict(x=x, mean=f.cache.mean, rstd=f.cache.inv_std, dy=dy, gamma=gamma, dx=torch.empty_like(x),
                      dg=torch.empty(D, device=dev), db=torch.empty(D, device=dev),
                      rg=torch.zeros(B, dtype=torch.float64, device=dev),
                      rb=torch.zeros(B, dtype=torch.float64, device=dev),
                      sums=torch.zeros(4, dtype=torch.float64, device=dev),
                      ws=torch.zeros(WS, dtype=torch.uint8, device=dev)))
    arr = {k: (VP * NL)(*[e[k].data_ptr() for e in L]) for k in L[0]}
    nbytes = NL * (B * T * D * 6 + 8 * B * T)
    desc = (ctypes.c_int * 6)()
    for i in ids:
        if sw.sweep_desc(i, desc) != 0:
            continue
        gw, vpt, g, rpg, prod, keep = list(desc)
        if gw * 32 * vpt < D // 8 or (gw * 32 * vpt) // 2 >= D // 8:
            continue
        res = {}
        modes = (1, 0, -1, -2) if "--rows" in sys.argv else (1, 0)
        for norms in modes:
            # 1 fused, 0 plain (B=1 view); -1 / -2: their row passes alone (no stage 2)
            Bv, Mv = (B, T) if norms in (1, -1) else (1, B * T)
            nm = -1 if norms < 0 else norms

            def step():
                return sw.sweep_step(i, NL, arr["x"], arr["mean"], arr["rstd"], arr["dy"], arr["gamma"], arr["dx"],
                                     arr["dg"], arr["db"], arr["rg"], arr["rb"], arr["sums"], nm, Bv, Mv, D,
                                     arr["ws"], WS, VP(torch.cuda.current_stream().cuda_stream))

            rc = step()
            torch.cuda.synchronize()
            if rc:
                res[norms] = None
                continue
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                step()
            torch.cuda.current_stream().wait_stream(s)
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                step()
            for _ in range(3):
                gr.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                gr.replay()
            e1.record()
            torch.cuda.synchronize()
            res[norms] = e0.elapsed_time(e1) / 10
            del gr
        if res.get(1) is None or res.get(0) is None:
            print(f"D={D} cfg{i:2d} gw{gw} vpt{vpt} g{g} rpg{rpg}: failed", flush=True)
            continue
        print(f"D={D} cfg{i:2d} gw{gw:2d} vpt{vpt} g{g:2d} rpg{rpg} prod{prod} keep{keep}: fused {res[1]*1e3:6.1f} us "
              f"{nbytes/res[1]/1e6:5.0f} GB/s ({nbytes/res[1]/1e6/6558.1*100:4.1f} %)  plain {res[0]*1e3:6.1f} us "
              f"({nbytes/res[0]/1e6/6558.1*100:4.1f} %)  ovh {100*(res[1]-res[0])/res[0]:5.2f} %"
              + (f" | rows only: fused {res[-1]*1e3:6.1f} plain {res[-2]*1e3:6.1f} us (ovh {100*(res[-1]-res[-2])/res[-2]:5.2f} %)"
                 if -1 in res else ""), flush=True)
    del L, arr
    torch.cuda.empty_cache()
