"""Streaming ceiling of the LN-bwd traffic (read x, dy; write dx; bf16, B=32 T=1024)
with 8 distinct buffer sets, one launch per set: no launch finds its inputs in
L2, as in bench.py's per-width "steady" measurement.  Experiment only."""
import ctypes
import os
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(HERE, "libstream_bench.so"))
f = ctypes.c_float()
B, T, NS = 32, 1024, 8
for D in [int(v) for v in (sys.argv[1:] or ["768", "1024", "2048", "4096"])]:
    N = B * T
    sets = [(torch.randn(N, D, device="cuda").bfloat16(), torch.randn(N, D, device="cuda").bfloat16(),
             torch.empty(N, D, device="cuda", dtype=torch.bfloat16)) for _ in range(NS)]
    arr = lambda k: (ctypes.c_void_p * NS)(*[s[k].data_ptr() for s in sets])
    xs, dys, dxs = arr(0), arr(1), arr(2)
    nbytes = 3 * N * D * 2
    for u in (1, 2, 4):
        for bps in (2, 4, 8):
            rc = lib.run_ldg_sets(u, bps, xs, dys, dxs, NS, ctypes.c_int64(N * D // 8), ctypes.byref(f), 24)
            print(f"D={D} sets ldg U={u} blocks/SM={bps}: {nbytes / f.value / 1e6:.0f} GB/s ({f.value*1e3:.1f} us) rc={rc}")
    for cw in (4, 8, 16):
        for R in (2, 4, 8):
            stage = 2 * R * D * 2
            S = min(12, (200 * 1024) // stage)
            if S < 2:
                continue
            rc = lib.run_tma_sets(cw, xs, dys, dxs, NS, ctypes.c_int64(N), D, R, S, ctypes.byref(f), 24)
            print(f"D={D} sets tma cw={cw} R={R} S={S}: {nbytes / f.value / 1e6:.0f} GB/s ({f.value*1e3:.1f} us) rc={rc}")
    del sets
    torch.cuda.empty_cache()
