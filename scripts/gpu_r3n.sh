mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_ln_gpu.py tests/test_nn_gpu.py -x -q 2>&1 | grep -E "Error|assert|passed|failed" | head -10 > gpurun_out/r3n.log
timeout 900 python experiments/ln_fwd_sweep.py >> gpurun_out/r3n.log 2>&1
