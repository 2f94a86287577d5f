"""GPU toy model (paper_2411_00999_b200/model.py) against plain PyTorch fp32.

The reference toy model (proj/include/gnstk/model.hpp:14-31) with every layer's
backward on the B200 kernels.  The check is torch.func: per-example gradients
of the mean-reduced loss (vmap over examples of grad(loss_b) / B) give, for every
instrumented layer and parameter, ||grad_b||^2, which must equal the kernels'
raw per-example norms (1e-4 relative); the parameter gradients must equal
torch autograd's (1e-4 relative to max|grad|); the device GNS step must equal
the reference arithmetic on the layers' records.
"""
import numpy as np
import pytest
import torch

from conftest import close

pytestmark = pytest.mark.gpu


def _functional_loss(p, ids, targets, n_blocks):
    """The same forward in plain torch ops, one example (ids [T])."""
    F = torch.nn.functional
    x = p["embed.weight"][ids.long()]
    for i in range(n_blocks):
        h = F.layer_norm(x, (x.shape[-1],), p[f"lns.{i}.weight"], p[f"lns.{i}.bias"], 1e-5)
        h = torch.tanh(h @ p[f"fc1.{i}.weight"] + p[f"fc1.{i}.bias"])
        x = x + (h @ p[f"fc2.{i}.weight"] + p[f"fc2.{i}.bias"])
    h = F.layer_norm(x, (x.shape[-1],), p["final_ln.weight"], p["final_ln.bias"], 1e-5)
    logits = h @ p["head.weight"] + p["head.bias"]
    return F.cross_entropy(logits, targets.long(), reduction="mean")


@pytest.mark.parametrize("path", ["autograd", "explicit"])
def test_toy_model_per_example_norms_and_gns(cuda, path):
    from paper_2411_00999_b200 import gns
    from paper_2411_00999_b200.model import ToyModelPE
    from paper_2411_00999_b200.nn import GnsTracker

    V, D, HM, NB, B, T = 64, 32, 2, 2, 4, 16
    model = ToyModelPE(V, D, HM, NB, seed=3, device=cuda)
    with torch.no_grad():  # non-trivial LN / bias parameters
        for name, prm in model.named_parameters():
            if name.endswith("bias") or ".lns." in f".{name}" or name.startswith("final_ln"):
                prm.add_(0.1 * torch.randn_like(prm))
    gen = torch.Generator(device="cpu").manual_seed(7)
    ids = torch.randint(0, V, (B, T), generator=gen, dtype=torch.int32).to(cuda)
    targets = torch.randint(0, V, (B, T), generator=gen, dtype=torch.int32).to(cuda)
    if path == "autograd":
        loss = model.loss(ids, targets)
        loss.backward()
    else:  # model_backward on the library kernels (fused epilogues, gnsb_xent, grouped LN stage 2)
        loss = model.forward_backward(ids, targets)
    torch.cuda.synchronize()

    params = {k: v.detach() for k, v in model.named_parameters()}
    ref_loss = torch.stack([_functional_loss(params, ids[b], targets[b], NB) for b in range(B)]).mean()
    assert close(float(loss.detach()), float(ref_loss), 1e-5)
    per_ex = torch.func.vmap(torch.func.grad(_functional_loss), in_dims=(None, 0, 0, None))(params, ids, targets, NB)
    full = torch.func.grad(lambda p: torch.stack([_functional_loss(p, ids[b], targets[b], NB)
                                                  for b in range(B)]).mean())(params)

    def raw_of(name):
        g = per_ex[name].double() / B  # gradient of the mean-reduced loss, example b's share
        return (g.reshape(B, -1) ** 2).sum(1).cpu().numpy()

    names = {"embed": ["embed.weight"], "final_ln": ["final_ln.weight", "final_ln.bias"],
             "head": ["head.weight", "head.bias"]}
    for i in range(NB):
        names[f"block{i}.ln"] = [f"lns.{i}.weight", f"lns.{i}.bias"]
        names[f"block{i}.fc1"] = [f"fc1.{i}.weight", f"fc1.{i}.bias"]
        names[f"block{i}.fc2"] = [f"fc2.{i}.weight", f"fc2.{i}.bias"]
    layers = model.instrumented_layers()
    assert [n for n, _ in layers][:2] == ["embed", "block0.ln"]
    for lname, mod in layers:
        keys = list(mod.per_example_raw)
        for key, pname in zip(keys, names[lname]):
            got = mod.per_example_raw[key].cpu().numpy()
            assert close(got, raw_of(pname), 1e-4), (lname, key)
        for pname in names[lname]:
            prm = dict(model.named_parameters())[pname]
            ref = full[pname]
            assert close(prm.grad.cpu().numpy(), ref.cpu().numpy(), 1e-4, 1e-4 * float(ref.abs().max())), pname

    tracker = GnsTracker([m for _, m in layers], alpha=1.0)
    groups, per_layer = tracker.step()
    torch.cuda.synchronize()
    recs = tracker.records.cpu().numpy()
    types = [m.layer_type for _, m in layers]
    g = groups.cpu().numpy()
    for gi, flt in enumerate([None, "embedding", "linear", "layernorm"]):
        big = small = 0.0
        for r, t in zip(recs, types):
            if flt is None or t == flt:
                big += r[3] + r[2]
                small += r[1] * B + r[0] * B
        st = gns.GradStats(big, small, B, 1, B)
        assert close(g[gi, 0], gns.estimate_g2(st), 1e-10), gi
        assert close(g[gi, 1], gns.estimate_s(st), 1e-10), gi


def test_toy_model_trains(cuda):
    """A few SGD steps on a fixed synthetic batch lower the loss; the GNS
    estimate is finite every step (the GNS-logged training loop of Trainer::step)."""
    from paper_2411_00999_b200.model import ToyModelPE
    from paper_2411_00999_b200.nn import GnsTracker

    V, D, B, T = 32, 32, 8, 16
    model = ToyModelPE(V, D, 2, 2, seed=5, device=cuda)
    gen = torch.Generator(device="cpu").manual_seed(11)
    ids = torch.randint(0, V, (B, T), generator=gen, dtype=torch.int32).to(cuda)
    targets = torch.roll(ids, -1, dims=1)
    opt = torch.optim.SGD(model.parameters(), lr=0.3)
    tracker = GnsTracker([m for _, m in model.instrumented_layers()], alpha=0.5)
    losses = []
    for _ in range(12):
        opt.zero_grad()
        loss = model.loss(ids, targets)
        loss.backward()
        groups, _ = tracker.step()
        opt.step()
        losses.append(float(loss.detach()))
        assert bool(torch.isfinite(groups[0, :3]).all())
    assert losses[-1] < 0.8 * losses[0], losses


def test_toy_model_bf16_rows_on_tensor_cores(cuda):
    """forward_backward with bf16 activations (fp32 parameters): the linear
    layers run the tcgen05 GEMMs with fused epilogues and the tcgen05 norm
    kernels; the result tracks the fp32 run within bf16 rounding."""
    from paper_2411_00999_b200.model import ToyModelPE

    V, D, HM, NB, B, T = 256, 128, 2, 2, 4, 64
    model = ToyModelPE(V, D, HM, NB, seed=9, device=cuda)
    gen = torch.Generator(device="cpu").manual_seed(13)
    ids = torch.randint(0, V, (B, T), generator=gen, dtype=torch.int32).to(cuda)
    targets = torch.randint(0, V, (B, T), generator=gen, dtype=torch.int32).to(cuda)
    l32 = float(model.forward_backward(ids, targets))
    g32 = {k: v.grad.clone() for k, v in model.named_parameters()}
    n32 = {n: m.norm_record.clone() for n, m in model.instrumented_layers()}
    l16 = float(model.forward_backward(ids, targets, rows_dtype=torch.bfloat16))
    torch.cuda.synchronize()
    assert close(l16, l32, 2e-2)
    for k, v in model.named_parameters():
        ref = g32[k]
        assert close(v.grad.cpu().numpy(), ref.cpu().numpy(), 5e-2, 5e-2 * float(ref.abs().max())), k
    for n, m in model.instrumented_layers():
        assert close(m.norm_record[:2].cpu().numpy(), n32[n][:2].cpu().numpy(), 1e-1), n
