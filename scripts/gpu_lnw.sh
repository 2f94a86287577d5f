#!/bin/bash
# warp-per-row LN backward row pass: parity, then per-width steady numbers per variant
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_ln_gpu.py -x -q 2>&1 | tail -5
B="python bench.py --steps 10 --warmup 3 --no-cpu --no-side --d-list 768,1024,2048"
show() { python -c "
import json,sys
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
print('$2', ' '.join(f\"D={s['D']}: steady {s['steady_fused_GBps']:.0f} ({100*s['steady_frac_of_measured_peak']:.1f}%) ovh {s['steady_overhead_pct']:.1f}% cold {s['fused_GBps']:.0f}\" for s in d['sweep']))
"; }
GNSB_LN_BWD_IMPL=ring timeout 300 $B > gpurun_out/lnw_ring.json 2>gpurun_out/lnw_ring.err; show gpurun_out/lnw_ring.json ring
for v in 0 1 2 3; do
  GNSB_LNW_VARIANT=$v timeout 300 $B > gpurun_out/lnw_v$v.json 2>gpurun_out/lnw_v$v.err; show gpurun_out/lnw_v$v.json v$v
done
for c in 1 3 4; do
  GNSB_LNW_CPS=$c timeout 300 $B > gpurun_out/lnw_c$c.json 2>gpurun_out/lnw_c$c.err; show gpurun_out/lnw_c$c.json cps$c
done
