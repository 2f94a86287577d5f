"""One embedding per-example-norms call at GPT-2 size (for an ncu launch list).  Experiment only."""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_00999_b200 import _lib  # noqa: E402
from paper_2411_00999_b200.layers import gnsb_dtype  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
T, V, D, dt = 1024, 50257, 768, torch.bfloat16
lib = _lib.lib()
dev = torch.device("cuda")
gen = torch.Generator(device="cpu").manual_seed(0)
ids = torch.randint(0, V, (B, T), generator=gen, dtype=torch.int32).to(dev)
g = torch.randn(B, T, D, generator=gen).to(dev, dt)
n = ctypes.c_size_t()
_lib.check(lib.gnsb_embedding_pe_workspace_size(B, T, V, D, gnsb_dtype(dt), ctypes.byref(n)))
ws = torch.zeros(n.value, dtype=torch.uint8, device=dev)
dW = torch.empty(V, D, dtype=torch.float32, device=dev)
raw = torch.empty(B, dtype=torch.float64, device=dev)
sums = torch.zeros(4, dtype=torch.float64, device=dev)
for _ in range(3):
    _lib.check(lib.gnsb_embedding_pe(ids.data_ptr(), g.data_ptr(), dW.data_ptr(), raw.data_ptr(), sums.data_ptr(),
                                     B, T, V, D, gnsb_dtype(dt), ws.data_ptr(), ws.numel(), None,
                                     torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
