mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_model_gpu.py tests/test_trainer_gpu.py -q 2>&1 | grep -E "Error|assert|passed|failed" | head -20 > gpurun_out/r3c_pytest.log
