mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
SWEEP_TRACE=1 timeout 300 python experiments/ln_sweep.py 768,1024,2048,4096,8192 15,10,6,0,2 > gpurun_out/trace.log 2>&1
timeout 120 python experiments/launch_overhead.py > gpurun_out/launch_overhead.log 2>&1
