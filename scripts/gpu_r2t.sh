mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_linear_gpu.py tests/test_model_gpu.py tests/test_trainer_gpu.py -x -q 2>&1 | tail -3 > gpurun_out/r2t_pytest.log
timeout 800 python experiments/form_sweep.py > gpurun_out/r2t_forms.log 2>&1
