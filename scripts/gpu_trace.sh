mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
SWEEP_TRACE=1 timeout 300 python experiments/ln_sweep.py 768,1024,2048,4096,8192 15,10,5,0,2 > gpurun_out/trace.log 2>&1
timeout 600 python bench.py --no-cpu --no-extra > gpurun_out/bench.log 2>&1
