"""PyTorch's own LayerNorm backward (aten::native_layer_norm_backward, bf16 rows,
the paper's baseline) on the cfg2 shapes: NL layers of one
width back to back (distinct buffers) in one CUDA graph (experiment only)."""
import sys

import torch

dev = torch.device("cuda")
B, T = 32, 1024
Ds = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [768, 1024, 2048, 4096, 8192]
NL = 8
for D in Ds:
    sets = []
    for _ in range(NL):
        x = torch.randn(B, T, D, device=dev, dtype=torch.bfloat16)
        w = torch.randn(D, device=dev, dtype=torch.bfloat16)
        b = torch.randn(D, device=dev, dtype=torch.bfloat16)
        y, mean, rstd = torch.ops.aten.native_layer_norm(x, [D], w, b, 1e-5)
        sets.append((torch.randn_like(x), x, mean, rstd, w, b))

    def step():
        for g, x, mean, rstd, w, b in sets:
            torch.ops.aten.native_layer_norm_backward(g, x, [D], mean, rstd, w, b, [True, True, True])

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            step()
    torch.cuda.current_stream().wait_stream(s)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        step()
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    nbytes = B * T * D * 6 + 8 * B * T
    print(f"aten D={D}: {ms*1e3/NL:.1f} us per layer, {NL*nbytes/ms/1e6:.0f} GB/s", flush=True)
