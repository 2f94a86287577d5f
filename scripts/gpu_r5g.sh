# LN row pass: early fold of the CTA's first example (GNSB_LN_EARLYFOLD=1 variant) vs production, interleaved
mkdir -p gpurun_out
for i in 1 2 3; do
  for v in base early; do
    if [ $v = base ]; then timeout 600 python bench.py --no-cpu --no-side > gpurun_out/r5g_$v$i.log 2>&1
    else GNSB_LIB_VARIANT=early timeout 600 python bench.py --no-cpu --no-side > gpurun_out/r5g_$v$i.log 2>&1; fi
  done
done
GNSB_LIB_VARIANT=early timeout 900 python -m pytest tests/test_ln_gpu.py -q -x 2>&1 | tail -3 > gpurun_out/r5g_pytest_early.log
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r5g_*[0-9].log')):
    l=[x for x in open(f) if x.startswith('{')]
    if not l: print(f,'no json'); continue
    d=json.loads(l[-1])
    sw=d.get('sweep',[])
    print(f, 'value %.0f'%d['value'], 'ovh %.2f'%d.get('overhead_pct',0), ' '.join('%d:%.1f'%(c['D'],100*c.get('steady_frac_of_measured_peak',0)) for c in sw))
PY
cat gpurun_out/r5g_pytest_early.log
