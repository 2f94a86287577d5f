mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
timeout 300 python experiments/linear_bench.py > gpurun_out/linear_bench.log 2>&1
