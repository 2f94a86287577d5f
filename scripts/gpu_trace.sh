mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench.log 2>&1
