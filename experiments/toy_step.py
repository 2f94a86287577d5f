"""The reference toy model (embedding -> n x [LN -> fc1 -> tanh -> fc2 +
residual] -> LN -> head, proj/src/model.cpp) at GPT-2-small width, one
training step's forward + backward:
  ours  : ToyModelPE.forward_backward with bf16 activations (fp32 parameters)
          -- every op on the library's kernels AND every layer's per-example
          gradient norms -- plus the device GNS step (GnsTracker);
  torch : the same architecture in torch (cuBLAS GEMMs, torch LayerNorm /
          embedding / cross-entropy, bf16 autocast, autograd), WITHOUT
          per-example norms -- an uninstrumented training step.
Both timed with CUDA events over replays of a captured CUDA graph.
Experiment only.  usage: python experiments/toy_step.py [B T]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_00999_b200.model import ToyModelPE  # noqa: E402
from paper_2411_00999_b200.nn import GnsTracker  # noqa: E402

dev = torch.device("cuda")
V, D, HM, NB = 50304, 768, 4, 12
B, T = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (8, 1024)
gen = torch.Generator(device="cpu").manual_seed(0)
ids = torch.randint(0, V, (B, T), generator=gen, dtype=torch.int32).to(dev)
targets = torch.randint(0, V, (B, T), generator=gen, dtype=torch.int32).to(dev)


def time_graph(fn, reps=10):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


model = ToyModelPE(V, D, HM, NB, seed=1, device=dev)
layers = model.instrumented_layers()
tracker = GnsTracker([m for _, m in layers], alpha=0.9)
nparam = sum(p.numel() for p in model.parameters())


def ours():
    model.forward_backward(ids, targets, rows_dtype=torch.bfloat16, validate=False)
    tracker.step()


ms_ours = time_graph(ours)


class Torch(torch.nn.Module):
    def __init__(self):
        super().__init__()
        H = D * HM
        self.emb = torch.nn.Embedding(V, D)
        self.lns = torch.nn.ModuleList([torch.nn.LayerNorm(D) for _ in range(NB)])
        self.fc1 = torch.nn.ModuleList([torch.nn.Linear(D, H) for _ in range(NB)])
        self.fc2 = torch.nn.ModuleList([torch.nn.Linear(H, D) for _ in range(NB)])
        self.lnf = torch.nn.LayerNorm(D)
        self.head = torch.nn.Linear(D, V)

    def forward(self, ids):
        x = self.emb(ids)
        for ln, f1, f2 in zip(self.lns, self.fc1, self.fc2):
            x = x + f2(torch.tanh(f1(ln(x))))
        return self.head(self.lnf(x))


tm = Torch().to(dev)


def plain():
    for p in tm.parameters():
        p.grad = None
    with torch.autocast("cuda", dtype=torch.bfloat16):
        logits = tm(ids.long())
        loss = torch.nn.functional.cross_entropy(logits.reshape(-1, V).float(), targets.reshape(-1).long())
    loss.backward()


ms_torch = time_graph(plain)
flops = 6.0 * nparam * B * T
print(f"toy model V={V} D={D} H={D*HM} blocks={NB} B={B} T={T}: {nparam/1e6:.1f} M params, "
      f"{flops/1e12:.2f} TFLOP per step (6 N tokens)")
print(f"  ours  (library kernels + per-example norms of every layer + GNS step): {ms_ours:8.3f} ms "
      f"({flops/ms_ours/1e9:.0f} TFLOP/s)")
print(f"  torch (cuBLAS + autograd, bf16 autocast, no per-example norms)       : {ms_torch:8.3f} ms "
      f"({flops/ms_torch/1e9:.0f} TFLOP/s)")
print(f"  ratio ours/torch: {ms_ours/ms_torch:.3f}")
