# fp32 rows on the 3xTF32 per-example weight-gradient path: parity + timing vs the generic kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_linear_gpu.py tests/test_nn_gpu.py tests/test_model_gpu.py tests/test_trainer_gpu.py -q -x 2>&1 | tail -6 > gpurun_out/r5i_pytest.log
timeout 600 python experiments/linear_f32_bench.py > gpurun_out/r5i_f32.log 2>&1
GNSB_LINEAR_F32_GENERIC=1 timeout 600 python experiments/linear_f32_bench.py >> gpurun_out/r5i_f32.log 2>&1
cat gpurun_out/r5i_pytest.log; cat gpurun_out/r5i_f32.log
