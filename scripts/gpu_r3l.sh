mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_model_gpu.py -x -q 2>&1 | grep -E "Error|assert|passed|failed" | head -10 > gpurun_out/r3l.log
timeout 600 python experiments/gemm_bench.py 8192 768 50304 >> gpurun_out/r3l.log 2>&1
timeout 600 python experiments/gemm_bench.py 32768 768 50264 >> gpurun_out/r3l.log 2>&1
GNSB_GEMM_NOSPLIT=1 timeout 600 python experiments/gemm_bench.py 8192 768 50304 >> gpurun_out/r3l.log 2>&1
timeout 600 python experiments/toy_step.py >> gpurun_out/r3l.log 2>&1
