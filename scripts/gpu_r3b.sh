mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_model_gpu.py -x -q 2>&1 | grep -E "Error|assert|passed|failed" | head -20 > gpurun_out/r3b_pytest.log
timeout 600 python experiments/gemm_bench.py --fp32 > gpurun_out/r3b_gemm_fp32.log 2>&1
