#!/bin/bash
# A/B of an environment switch on the per-width steady numbers:  bash scripts/gpu_ab.sh VAR "v1 v2 ..." [d-list]
VAR=$1; VALS=$2; DL=${3:-768,1024,2048,4096,8192}
mkdir -p gpurun_out
[ -z "$NO_TEST" ] && timeout 600 python -m pytest tests/test_ln_gpu.py -x -q 2>&1 | tail -2
show() { python -c "
import json
d=json.loads([l for l in open('$1') if l.startswith('{')][-1])
print('$2', 'step %.1f%%' % (100*d['roofline_step']['frac']), ' '.join(f\"D={s['D']}: {100*s['steady_frac_of_measured_peak']:.1f}% ovh {s['steady_overhead_pct']:.1f} cold {100*s['frac_of_measured_peak']:.1f}%\" for s in d['sweep']))
"; }
for rep in 1 2; do
for v in $VALS; do
  env $VAR=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-side --d-list $DL > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err; show gpurun_out/ab_$v.json "$VAR=$v"
done
done
