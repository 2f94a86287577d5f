"""Embedding per-example norms (gnsb_embedding_pe) at GPT-2-like sizes: time
per call (CUDA graph replay of one call, median), algorithmic bytes
g + ids in, dW out, and the share of each kernel (torch profiler-free: two
graphs, with and without the table pass, are not separable here, so only the
total is reported).  Experiment only."""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_00999_b200 import _lib  # noqa: E402
from paper_2411_00999_b200.layers import gnsb_dtype, stat_dtype  # noqa: E402

lib = _lib.lib()
dev = torch.device("cuda")


def run(B, T, V, D, dt):
    gen = torch.Generator(device="cpu").manual_seed(0)
    ids = torch.randint(0, V, (B, T), generator=gen, dtype=torch.int32).to(dev)
    g = torch.randn(B, T, D, generator=gen).to(dev, dt)
    sd = stat_dtype(dt)
    n = ctypes.c_size_t()
    _lib.check(lib.gnsb_embedding_pe_workspace_size(B, T, V, D, gnsb_dtype(dt), ctypes.byref(n)))
    ws = torch.zeros(n.value, dtype=torch.uint8, device=dev)
    dW = torch.empty(V, D, dtype=sd, device=dev)
    raw = torch.empty(B, dtype=torch.float64, device=dev)
    sums = torch.zeros(4, dtype=torch.float64, device=dev)

    def call():
        _lib.check(lib.gnsb_embedding_pe(ids.data_ptr(), g.data_ptr(), dW.data_ptr(), raw.data_ptr(), sums.data_ptr(),
                                         B, T, V, D, gnsb_dtype(dt), ws.data_ptr(), ws.numel(), None,
                                         torch.cuda.current_stream().cuda_stream))

    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        call()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        call()
    ts = []
    for _ in range(12):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        gr.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    t = ts[len(ts) // 2]
    alg = B * T * D * g.element_size() + B * T * 4 + V * D * dW.element_size()
    print(f"B={B} T={T} V={V} D={D} {str(dt):15s}: {t*1e3:8.1f} us  {alg/t/1e6:6.0f} GB/s algorithmic "
          f"(g + ids in, dW out; workspace {n.value/1e6:.0f} MB)", flush=True)


for args in [(32, 1024, 50257, 768, torch.bfloat16), (32, 1024, 50257, 768, torch.float32),
             (8, 1024, 50257, 768, torch.bfloat16), (64, 1024, 50257, 768, torch.bfloat16),
             (32, 1024, 8192, 768, torch.bfloat16)]:
    run(*args)
