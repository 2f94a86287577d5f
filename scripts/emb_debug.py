import os, sys, torch, numpy as np, subprocess
sys.path.insert(0, os.getcwd())
code = r'''
import sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_2411_00999_b200.embedding import embedding_backward_simultaneous
B,T,V,D = 8,512,1000,256
gen = torch.Generator(device="cpu").manual_seed(B * 1000 + T)
ids = (torch.rand(B, T, generator=gen) ** 3 * V).to(torch.int32).clamp_(0, V - 1)
g = torch.randn(B, T, D, generator=gen)
r = embedding_backward_simultaneous(ids.cuda(), g.cuda(), V)
torch.cuda.synchronize()
np.savez(sys.argv[1], dW=r.weight_grads["weight"].cpu().numpy(), raw=r.per_example_sqnorms_raw["weight"].cpu().numpy(), s=r.sums4.cpu().numpy())
'''
open('gpurun_out/embdbg_inner.py','w').write(code)
for impl in ('fast','slow'):
    subprocess.run([sys.executable, 'gpurun_out/embdbg_inner.py', f'gpurun_out/emb_{impl}.npz'], env=dict(os.environ, GNSB_EMB_IMPL=impl), check=True)
a = np.load('gpurun_out/emb_fast.npz'); b = np.load('gpurun_out/emb_slow.npz')
d = np.abs(a['dW'] - b['dW'])
print('dW max diff', d.max(), 'rows differing', np.unique(np.nonzero(d > 1e-6)[0])[:20], 'count', (d.max(1) > 1e-6).sum())
print('raw fast', a['raw']); print('raw slow', b['raw']); print('sums', a['s'], b['s'])
