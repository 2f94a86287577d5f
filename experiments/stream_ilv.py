"""TMA-ring streaming (read x, dy; write dx; bf16, B=32 T=1024, 8 buffer sets)
with the stage order interleaved across CTAs in chunks of K stages (K=0:
contiguous per-CTA row ranges).  Does DRAM locality of the concurrent
streams set the narrow-width ceiling?  Experiment only."""
import ctypes
import os
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(HERE, "libstream_bench.so"))
f = ctypes.c_float()
B, T, NS = 32, 1024, 8
for D in [int(v) for v in (sys.argv[1:] or ["1024", "2048"])]:
    N = B * T
    sets = [(torch.randn(N, D, device="cuda").bfloat16(), torch.randn(N, D, device="cuda").bfloat16(),
             torch.empty(N, D, device="cuda", dtype=torch.bfloat16)) for _ in range(NS)]
    arr = lambda k: (ctypes.c_void_p * NS)(*[s[k].data_ptr() for s in sets])
    xs, dys, dxs = arr(0), arr(1), arr(2)
    nbytes = 3 * N * D * 2
    for cw in (8, 16):
        for R in (4, 8):
            stage = 2 * R * D * 2
            S = min(12, (200 * 1024) // stage)
            for K in (0, 1, 2, 4, 8, 16, 32):
                rc = lib.run_tma_ilv_sets(cw, xs, dys, dxs, NS, ctypes.c_int64(N), D, R, S, K, ctypes.byref(f), 24)
                print(f"D={D} tma_ilv cw={cw} R={R} S={S} K={K}: {nbytes / f.value / 1e6:.0f} GB/s ({f.value*1e3:.1f} us) rc={rc}", flush=True)
    del sets
    torch.cuda.empty_cache()
