"""Time the linear-layer GEMMs (gnsb_linear_dx / gnsb_linear_fwd, tcgen05) at
BASELINE config 3 (rows = B*T = 32768, K = L = 4096 bf16) and at shapes with
tile tails; ncu target (experiment only)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_00999_b200 import _lib  # noqa: E402

lib = _lib.lib()
dev = torch.device("cuda")
PEAK = 1647.2
shapes = [(32768, 4096, 4096), (32768, 4096, 16384), (32768, 16384, 4096), (8192, 1024, 4096), (32768, 768, 50264),
          (30000, 4000, 4000)]
DT = torch.bfloat16
if "--fp32" in sys.argv:  # fp32 rows and weights: the 3xTF32 kernel
    DT = torch.float32
    sys.argv.remove("--fp32")
    shapes = [(32768, 4096, 4096), (8192, 1024, 4096), (30000, 4000, 4000)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in sys.argv[1:4])]
GD = 0 if DT == torch.float32 else 1
for rows, K, L in shapes:
    a_fwd = torch.randn(rows, K, device=dev).to(DT)
    a_dx = torch.randn(rows, L, device=dev).to(DT)
    W = (torch.randn(K, L, device=dev) / K ** 0.5).to(DT)
    y = torch.empty(rows, L, device=dev, dtype=DT)
    dx = torch.empty(rows, K, device=dev, dtype=DT)
    sp = torch.cuda.current_stream().cuda_stream
    for name, fn in (("dx ", lambda: lib.gnsb_linear_dx(a_dx.data_ptr(), W.data_ptr(), dx.data_ptr(), rows, K, L, GD, GD,
                                                         None, 0, sp)),
                     ("fwd", lambda: lib.gnsb_linear_fwd(a_fwd.data_ptr(), W.data_ptr(), None, y.data_ptr(), rows, K,
                                                         L, GD, GD, None, 0, sp))):
        for _ in range(3):
            assert fn() == 0, lib.gnsb_last_error()
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        t = ts[len(ts) // 2]
        fl = 2.0 * rows * K * L
        ref = torch.cuda.Event(enable_timing=True)
        print(f"rows={rows} K={K} L={L} {name}: {t*1e3:8.1f} us {fl/t/1e9:7.0f} TFLOP/s ({fl/t/1e9/PEAK*100:.1f}% of "
              f"{PEAK})", flush=True)
    # cuBLAS for the same products (library reference point)
    for name, fn in (("cublas dx ", lambda: torch.matmul(a_dx, W.t(), out=dx)),
                     ("cublas fwd", lambda: torch.matmul(a_fwd, W, out=y))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 10
        print(f"rows={rows} K={K} L={L} {name}: {t*1e3:8.1f} us {2.0*rows*K*L/t/1e9:7.0f} TFLOP/s", flush=True)
    del a_fwd, a_dx, W, y, dx
    torch.cuda.empty_cache()
