"""Driver for experiments/stream_bench.cu (memory ceiling of the LN-bwd traffic)."""
import ctypes
import os
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(HERE, "libstream_bench.so"))
f = ctypes.c_float()
B, T = 32, 1024
for D in [int(v) for v in (sys.argv[1:] or ["768", "4096", "8192"])]:
    N = B * T
    x = torch.randn(N, D, device="cuda").bfloat16()
    dy = torch.randn(N, D, device="cuda").bfloat16()
    dx = torch.empty_like(x)
    nbytes = 3 * N * D * 2
    for u in (1, 2, 4, 8):
        for bps in (2, 4, 8):
            rc = lib.run_ldg(u, bps, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(dy.data_ptr()),
                             ctypes.c_void_p(dx.data_ptr()), ctypes.c_int64(N * D // 8), ctypes.byref(f), 20)
            print(f"D={D} ldg U={u} blocks/SM={bps}: {nbytes / f.value / 1e6:.0f} GB/s rc={rc}")
    for cw in (4, 8, 16):
        for R in (1, 2, 4, 8):
            stage = 2 * R * D * 2
            S = min(12, (200 * 1024) // stage)
            if S < 2:
                continue
            for s in sorted({2, 4, S}):
                if s > S:
                    continue
                rc = lib.run_tma(cw, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(dy.data_ptr()),
                                 ctypes.c_void_p(dx.data_ptr()), ctypes.c_int64(N), D, R, s, ctypes.byref(f), 20)
                print(f"D={D} tma cw={cw} R={R} S={s} ({s * stage // 1024} KB ring): {nbytes / f.value / 1e6:.0f} GB/s rc={rc}")
