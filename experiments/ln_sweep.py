"""Time every LN-bwd configuration of experiments/ln_sweep.cu (bf16, B=32 T=1024)."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_00999_b200 as m  # noqa: E402

lib = ctypes.CDLL(os.path.join(ROOT, "experiments", "libln_sweep.so"))
_vp, _i64 = ctypes.c_void_p, ctypes.c_int64
lib.sweep_run.argtypes = [ctypes.c_int] + [_vp] * 11 + [ctypes.c_int, _i64, _i64, _i64, _vp, ctypes.c_size_t, _vp, _vp, _vp]
lib.sweep_run.restype = ctypes.c_int
dev = torch.device("cuda")
B, T = int(os.environ.get('SWEEP_B', '32')), 1024
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
TRACE = os.environ.get("SWEEP_TRACE") == "1"
mk = ctypes.CDLL(os.path.join(ROOT, "experiments", "liblaunch_overhead.so"))
marks = torch.zeros(2, dtype=torch.int64, device=dev)
FLUSH = os.environ.get("SWEEP_FLUSH", "write")
flush_sink = torch.zeros((), dtype=torch.int64, device=dev)
trace = torch.zeros(148 * 6, dtype=torch.int64, device=dev)
trace2 = torch.zeros(148 * 6, dtype=torch.int64, device=dev)
Ds = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [768, 1024, 2048, 4096, 8192]
ids = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else list(range(lib.sweep_n()))
for D in Ds:
    x, dy, gamma, beta = m.synth_ln(B, T, D, torch.bfloat16, dev)
    f = m.layernorm_forward(m.LayerNormLayer(gamma, beta), x)
    ref = m.layernorm_backward_simultaneous(m.LayerNormLayer(gamma, beta), f.cache, dy)
    dx = torch.empty_like(x)
    dg = torch.empty(D, device=dev)
    db = torch.empty(D, device=dev)
    rg = torch.empty(B, dtype=torch.float64, device=dev)
    rb = torch.empty(B, dtype=torch.float64, device=dev)
    sums = torch.empty(4, dtype=torch.float64, device=dev)
    ws = torch.zeros(256 << 20, dtype=torch.uint8, device=dev)
    nbytes = B * T * D * 6 + 8 * B * T + 12 * D + 16 * B
    desc = (ctypes.c_int * 6)()
    for i in ids:
        if lib.sweep_desc(i, desc) != 0:
            continue
        gw, vpt, g, rpg, prod, keep = list(desc)
        if gw * 32 * vpt < D // 8 or (gw * 32 * vpt) // 2 >= D // 8:
            continue  # config does not fit this width (or wastes > half the lanes)
        res = {}
        for norms in (1, 0):
            ts = []
            for r in range(12):
                if FLUSH == "write":
                    flush.zero_()
                elif FLUSH == "read":
                    flush_sink.copy_(flush.view(torch.int64).sum())
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                if TRACE:
                    mk.marker(ctypes.c_void_p(marks.data_ptr()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
                rc = lib.sweep_run(i, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(f.cache.mean.data_ptr()),
                                   ctypes.c_void_p(f.cache.inv_std.data_ptr()), ctypes.c_void_p(dy.data_ptr()),
                                   ctypes.c_void_p(gamma.data_ptr()), ctypes.c_void_p(dx.data_ptr()),
                                   ctypes.c_void_p(dg.data_ptr()), ctypes.c_void_p(db.data_ptr()),
                                   ctypes.c_void_p(rg.data_ptr()), ctypes.c_void_p(rb.data_ptr()),
                                   ctypes.c_void_p(sums.data_ptr()), norms, B, T, D, ctypes.c_void_p(ws.data_ptr()),
                                   ctypes.c_size_t(ws.numel()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream),
                                   ctypes.c_void_p(trace.data_ptr() if TRACE else 0),
                                   ctypes.c_void_p(trace2.data_ptr() if TRACE else 0))
                if TRACE:
                    mk.marker(ctypes.c_void_p(marks.data_ptr() + 8), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
                e1.record()
                if rc:
                    break
                torch.cuda.synchronize()
                if r >= 2:
                    ts.append(e0.elapsed_time(e1))
            if rc:
                res[norms] = f"rc={rc}"
                continue
            ts.sort()
            res[norms] = ts[len(ts) // 2]
            if TRACE:
                tr = trace.view(-1, 6).cpu().numpy().astype("int64")
                t2 = trace2.view(-1, 6).cpu().numpy().astype("int64")
                trace2.zero_()
                mks = marks.cpu().numpy().astype("int64")
                t0 = tr[:, 0].min()
                last = max(tr[:, 2].max(), t2.max())
                t2 = np.where(t2 == 0, t0, t2)
                rel = (tr - t0) / 1000.0
                r2 = (t2 - t0) / 1000.0
                print(f"   {'fused' if norms else 'plain'}: launch->start {(t0 - mks[0]) / 1000:.1f} us; last->marker {(mks[1] - last) / 1000:.1f} us"
                      f" | rowmath end min {rel[:,1].min():.1f} med {sorted(rel[:,1])[len(rel)//2]:.1f} max {rel[:,1].max():.1f}"
                      f" | fold end {rel[:,2].max():.1f} | red wait-out {r2[:,0].min():.1f}..{r2[:,0].max():.1f}"
                      f" | loads {r2[:,1].max():.1f} | red end {r2[:,2].max():.1f} | final {r2[:,3].max():.1f}->{r2[:,4].max():.1f}")
        ok = ""
        if not isinstance(res.get(1), str):
            err = (dx.float() - ref.input_grad.float()).abs().max().item()
            nerr = ((rg - ref.grads.per_example_sqnorms_raw["gamma"]).abs() / ref.grads.per_example_sqnorms_raw["gamma"]).max().item()
            ok = f"dxerr={err:.1e} nerr={nerr:.1e}"
        if isinstance(res.get(1), str) or isinstance(res.get(0), str):
            print(f"D={D} cfg{i} gw{gw} vpt{vpt} g{g} rpg{rpg} prod{prod} keep{keep}: {res}", flush=True)
            continue
        print(f"D={D} cfg{i:2d} gw{gw:2d} vpt{vpt} g{g} rpg{rpg} prod{prod} keep{keep}: fused {res[1]*1e3:7.1f}us "
              f"{nbytes/res[1]/1e6:6.0f} GB/s  plain {res[0]*1e3:7.1f}us {nbytes/res[0]/1e6:6.0f} GB/s "
              f"ovh {100*(res[1]-res[0])/res[0]:5.1f}%  {ok}", flush=True)
