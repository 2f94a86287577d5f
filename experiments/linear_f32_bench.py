"""fp32 rows: per-example weight-gradient norms (+ dW) on the 3xTF32 path
(linear_f32.cu) at BASELINE config 3's shape (B=16 T=2048 K=L=4096) and a
smaller shape; GNSB_LINEAR_F32_GENERIC=1 times the generic kernels instead
(smaller shape only).  CUDA events around one call, median of 5.  Experiment only."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_00999_b200 as m  # noqa: E402
from paper_2411_00999_b200 import linear  # noqa: E402

dev = torch.device("cuda")
generic = os.environ.get("GNSB_LINEAR_F32_GENERIC") is not None
shapes = [(4, 1024, 1024, 1024)] + ([] if generic else [(16, 2048, 4096, 4096)])
for B, T, K, L in shapes:
    x, g = m.synth_linear(B, T, K, L, torch.float32, dev)
    layer = linear.LinearLayer(torch.zeros(K, L, device=dev))
    for form in ("weight_grad", "gram"):
        def call():
            if form == "gram":
                return linear.linear_perexample_sqnorm_frobenius(x, g)
            return linear.linear_backward_simultaneous(layer, x, g, form="weight_grad", need_input_grad=False)
        call()
        torch.cuda.synchronize()
        ts = []
        for _ in range(3 if generic else 5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            call()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        t = ts[len(ts) // 2]
        fl = 2.0 * B * T * K * L
        print(f"{'generic' if generic else '3xTF32 '} B={B} T={T} K={K} L={L} fp32 form={form:11s}: {t:9.3f} ms  "
              f"{fl / t / 1e9:8.1f} TFLOP/s (2BTKL)", flush=True)
