"""Form dispatch evidence: the per-example linear norms
at K = L = 4096 bf16 with B*T = 32768 tokens fixed, T swept 128..8192.
Per T: the weight-gradient form with dW (wgrad_norms_kernel), the Gram form
(norms only), and a plain dW GEMM (cuBLAS via torch, the "Gram + plain dW"
alternative).  Prints which form wins for norms only and for norms + dW, next
to the FLOP model's crossover (Gram iff T*(K+L) < 2*K*L, i.e. T < 4096 here).
Experiment only."""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_00999_b200 as m  # noqa: E402
from paper_2411_00999_b200 import _lib  # noqa: E402

lib = _lib.lib()
dev = torch.device("cuda")
K = L = 4096
NTOK = 32768


def t_ms(fn, reps=7):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


print(f"K=L={K}, B*T={NTOK} tokens, bf16; FLOP-model crossover T = {2 * K * L / (K + L):.0f}")
for T in (128, 256, 512, 1024, 2048, 4096, 8192):
    B = NTOK // T
    x, g = m.synth_linear(B, T, K, L, torch.bfloat16, dev)
    dW = torch.empty(K, L, device=dev)
    raw = torch.empty(B, dtype=torch.float64, device=dev)
    n = ctypes.c_size_t()
    _lib.check(lib.gnsb_linear_pe_workspace_size(B, T, K, L, 1, ctypes.byref(n)))
    ws = torch.zeros(n.value, dtype=torch.uint8, device=dev)
    sp = torch.cuda.current_stream().cuda_stream

    def form(f, with_dw):
        _lib.check(lib.gnsb_linear_pe_norms(x.data_ptr(), g.data_ptr(), dW.data_ptr() if with_dw else None,
                                            raw.data_ptr(), None, B, T, K, L, f, 1, ws.data_ptr(), ws.numel(), sp))

    tw = t_ms(lambda: form(1, True))
    ta = t_ms(lambda: form(0, True))
    tg = t_ms(lambda: form(2, False))
    xf, gf = x.reshape(NTOK, K), g.reshape(NTOK, L)
    tgemm = t_ms(lambda: torch.matmul(xf.t(), gf))
    norms_only = "gram" if tg < tw else "weight-grad"
    with_dw = "gram + dW GEMM" if tg + tgemm < tw else "weight-grad"
    model = "gram" if T * (K + L) < 2 * K * L else "weight-grad"
    print(f"T={T:5d} B={B:4d}: weight-grad+dW {tw*1e3:8.1f} us | gram {tg*1e3:8.1f} us | dW GEMM {tgemm*1e3:7.1f} us"
          f" | norms only -> {norms_only:11s} (model: {model}) | norms + dW -> {with_dw:15s} | auto(+dW) {ta*1e3:7.1f} us",
          flush=True)
    del x, g, dW, ws
    torch.cuda.empty_cache()
