"""Time the per-example linear norm kernels at BASELINE config 3 (B=16 T=2048 K=L=4096 bf16)."""
import ctypes, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_00999_b200 as m
from paper_2411_00999_b200 import _lib, linear
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
def run():
    _lib.check(_lib.lib().gnsb_linear_pe_norms(x.data_ptr(), g.data_ptr(), dW.data_ptr(), raw.data_ptr(), sums.data_ptr(),
                                               B, T, K, L, 1, 1, ws.data_ptr(), ws.numel(), sp))
for _ in range(3): run()
torch.cuda.synchronize()
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); run(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
ts.sort(); t = ts[len(ts)//2]
fl = 2.0 * B * T * K * L
print(f"B={B} T={T} K={K} L={L}: weight-grad form {t*1e3:.1f} us  {fl/t/1e9:.0f} TFLOP/s  ({fl/t/1e9/1671.9*100:.1f}% of measured 1671.9)")
