"""LayerNormPE (paper_2411_00999_b200/nn.py): the fused kernel behind torch autograd.

Numerics are checked against a plain PyTorch fp32 reference of the same op
(torch.nn.functional.layer_norm + autograd); the per-example norms against
per-example autograd passes (loss_b / B, i.e. the mean-reduced loss split by
example). Tolerances: fp32 rows 1e-5 relative (atol 1e-5 * max|ref|), norms
1e-4; bf16 rows dx 2^-8 relative to max|ref|.
"""
import numpy as np
import pytest
import torch

from conftest import close


def _ref(x, w, b, c, eps=1e-5):
    """fp32 torch reference: loss = mean_b sum(y_b * c_b); grads and per-example norms."""
    x = x.detach().float().requires_grad_(True)
    w = w.detach().float().requires_grad_(True)
    b = b.detach().float().requires_grad_(True)
    y = torch.nn.functional.layer_norm(x, (x.shape[-1],), w, b, eps)
    B = x.shape[0]
    loss = (y * c.float()).flatten(1).sum(1).mean()
    dx, dw, db = torch.autograd.grad(loss, (x, w, b))
    raw_w, raw_b = [], []
    for i in range(B):
        wi = w.detach().clone().requires_grad_(True)
        bi = b.detach().clone().requires_grad_(True)
        yi = torch.nn.functional.layer_norm(x[i:i + 1].detach(), (x.shape[-1],), wi, bi, eps)
        li = (yi * c[i:i + 1].float()).sum() / B
        gw, gb = torch.autograd.grad(li, (wi, bi))
        raw_w.append(float((gw.double() ** 2).sum()))
        raw_b.append(float((gb.double() ** 2).sum()))
    return dx, dw, db, np.array(raw_w), np.array(raw_b)


@pytest.mark.gpu
@pytest.mark.parametrize("dt,shape", [(torch.float32, (4, 33, 256)), (torch.float32, (3, 2, 5, 768)),
                                      (torch.bfloat16, (4, 64, 1024))])
def test_layernorm_pe_matches_torch(cuda, dt, shape):
    from paper_2411_00999_b200.nn import LayerNormPE

    torch.manual_seed(0)
    D = shape[-1]
    ln = LayerNormPE(D, device=cuda)
    with torch.no_grad():
        ln.weight.copy_(1.0 + 0.1 * torch.randn(D, device=cuda))
        ln.bias.copy_(0.1 * torch.randn(D, device=cuda))
    x = (torch.randn(shape, device=cuda) + 0.5).to(dt).requires_grad_(True)
    c = torch.randn(shape, device=cuda).to(dt)
    y = ln(x)
    B = shape[0]
    loss = (y.float() * c.float()).flatten(1).sum(1).mean()
    loss.backward()
    rdx, rdw, rdb, rraw_w, rraw_b = _ref(x, ln.weight, ln.bias, c)
    torch.cuda.synchronize()
    tol = 1e-5 if dt == torch.float32 else 2.0 ** -8
    assert close(x.grad.float().cpu().numpy(), rdx.cpu().numpy(), tol, tol * float(rdx.abs().max()))
    gtol = 1e-5 if dt == torch.float32 else 1e-4
    assert close(ln.weight.grad.cpu().numpy(), rdw.cpu().numpy(), gtol, gtol * float(rdw.abs().max()))
    assert close(ln.bias.grad.cpu().numpy(), rdb.cpu().numpy(), gtol, gtol * float(rdb.abs().max()))
    assert close(ln.per_example_raw["gamma"].cpu().numpy(), rraw_w, 1e-4)
    assert close(ln.per_example_raw["beta"].cpu().numpy(), rraw_b, 1e-4)
    rec = ln.norm_record.cpu().numpy()
    assert close(rec[0], rraw_w.sum(), 1e-4) and close(rec[1], rraw_b.sum(), 1e-4)
    assert close(rec[2], float((rdw.double() ** 2).sum()), 1e-4)
    assert close(rec[3], float((rdb.double() ** 2).sum()), 1e-4)
    assert ln.batch_size == B


@pytest.mark.gpu
def test_gns_tracker_over_two_layers(cuda):
    """Two LayerNormPE layers in a tiny residual stack; the tracker's device GNS
    step equals the reference arithmetic on the layers' records."""
    from paper_2411_00999_b200 import gns
    from paper_2411_00999_b200.nn import GnsTracker, LayerNormPE

    torch.manual_seed(1)
    B, T, D = 8, 16, 128
    l1, l2 = LayerNormPE(D, device=cuda), LayerNormPE(D, device=cuda)
    lin = torch.nn.Linear(D, D, device=cuda)
    x = torch.randn(B, T, D, device=cuda)
    h = l2(lin(l1(x)) + x)
    loss = (h ** 2).flatten(1).sum(1).mean()
    loss.backward()
    tr = GnsTracker([l1, l2], alpha=1.0)
    groups, layers = tr.step()
    torch.cuda.synchronize()
    big = small = 0.0
    for r in tr.records.cpu().numpy():
        big += r[3] + r[2]
        small += r[1] * B + r[0] * B
    st = gns.GradStats(big, small, B, 1, B)
    g = groups.cpu().numpy()
    assert close(g[0, 0], gns.estimate_g2(st), 1e-10)
    assert close(g[0, 1], gns.estimate_s(st), 1e-10)
    assert close(g[3, :2], g[0, :2], 0.0)
    # records are consumed: a step whose backward skipped a tracked layer fails loudly
    assert l1.norm_record is None and l2.norm_record is None
    l1(x).sum().backward()
    with pytest.raises(RuntimeError, match="no norm record"):
        tr.step()


def test_layernorm_pe_rejects_cpu_and_bad_shapes():
    """CPU: the module refuses host tensors (no eager fallback) and bad shapes."""
    from paper_2411_00999_b200.nn import LayerNormPE

    with pytest.raises(ValueError, match="epsilon"):
        LayerNormPE(8, eps=0.0)
    with pytest.raises(ValueError, match="trailing extent >= 2"):
        LayerNormPE(1)
    ln = LayerNormPE(8)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        ln(torch.zeros(2, 3, 8))
    with pytest.raises(ValueError, match="trailing extent"):
        ln(torch.zeros(2, 3, 7))
