#!/bin/bash
# CTA-pair weight-gradient kernel: parity, timing of both kernels, one ncu capture
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_linear_gpu.py -x -q 2>&1 | tail -15
for impl in 0 1; do GNSB_WGRAD_IMPL=$impl timeout 300 python experiments/linear_bench.py 2>&1 | tail -4; done
GNSB_WGRAD_IMPL=0 timeout 300 python experiments/linear_bench.py 8 1024 4096 4096 2>&1 | tail -4
GNSB_WGRAD_IMPL=1 timeout 300 python experiments/linear_bench.py 8 1024 4096 4096 2>&1 | tail -4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wgrad_norms_kernel -c 1 \
  -o gpurun_out/prof_wgrad_pair -f python experiments/linear_bench.py > gpurun_out/ncu_wgrad.log 2>&1
tail -3 gpurun_out/ncu_wgrad.log
