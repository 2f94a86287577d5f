# model on library kernels + reference suites + GEMM timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_model_gpu.py tests/test_trainer_gpu.py tests/test_linear_gpu.py -x -q 2>&1 | tail -30 > gpurun_out/r2j_pytest.log
LD_LIBRARY_PATH=paper_2411_00999_b200/lib timeout 600 ./tests/cpp/_ref/unit_tests -ts=layers > gpurun_out/r2j_ref_layers.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_ref_layers.log
LD_LIBRARY_PATH=paper_2411_00999_b200/lib timeout 900 ./tests/cpp/_ref/unit_tests -ts=trainer > gpurun_out/r2j_ref_trainer.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_ref_trainer.log
LD_LIBRARY_PATH=paper_2411_00999_b200/lib timeout 1500 ./tests/cpp/_ref/acceptance > gpurun_out/r2j_ref_acceptance.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_ref_acceptance.log
