mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_model_gpu.py -x -q 2>&1 | tail -5 > gpurun_out/r2o_pytest.log
timeout 600 python experiments/gemm_bench.py > gpurun_out/r2o_gemm.log 2>&1
