"""Time the per-example linear norm kernels at BASELINE config 3 (B=16 T=2048 K=L=4096 bf16):
weight-gradient form (dW + norms) and Gram form (norms only), both on tcgen05."""
import ctypes, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_00999_b200 as m
from paper_2411_00999_b200 import _lib
B, T, K, L = (int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (16, 2048, 4096, 4096)))
dev = torch.device("cuda")
x, g = m.synth_linear(B, T, K, L, torch.bfloat16, dev)
dW = torch.empty(K, L, device=dev)
raw = torch.empty(B, dtype=torch.float64, device=dev)
sums = torch.zeros(4, dtype=torch.float64, device=dev)
n = ctypes.c_size_t()
_lib.check(_lib.lib().gnsb_linear_pe_workspace_size(B, T, K, L, 1, ctypes.byref(n)))
ws = torch.zeros(n.value, dtype=torch.uint8, device=dev)
sp = torch.cuda.current_stream().cuda_stream
def run(form):
    _lib.check(_lib.lib().gnsb_linear_pe_norms(x.data_ptr(), g.data_ptr(), dW.data_ptr() if form == 1 else None,
                                               raw.data_ptr(), sums.data_ptr(), B, T, K, L, form, 1, ws.data_ptr(),
                                               ws.numel(), sp))
res = {}
for form, name in ((1, "weight-grad"), (2, "gram")):
    for _ in range(3): run(form)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); run(form); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort(); t = ts[len(ts)//2]
    res[form] = raw.clone()
    fl = 2.0 * B * T * K * L if form == 1 else 1.0 * B * T * T * (K + L)  # algorithmic (Gram: symmetric half)
    print(f"B={B} T={T} K={K} L={L}: {name:11s} form {t*1e3:8.1f} us  {fl/t/1e9:6.0f} TFLOP/s algorithmic"
          f" ({fl/t/1e9/1671.9*100:.1f}% of measured 1671.9)", flush=True)
print("max rel diff between forms:", float(((res[1] - res[2]).abs() / res[1].abs()).max()))
