mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_model_gpu.py tests/test_trainer_gpu.py -x -q 2>&1 | grep -E "Error|assert|passed|failed" | head -20 > gpurun_out/r3g_pytest.log
timeout 600 python experiments/toy_step.py > gpurun_out/r3g_toy.log 2>&1
timeout 900 python bench.py > gpurun_out/r3g_bench.log 2>&1
