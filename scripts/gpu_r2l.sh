# fp64 reference-order per-example params: the reference's own suites + our GPU tests
mkdir -p gpurun_out
export LD_LIBRARY_PATH=paper_2411_00999_b200/lib
timeout 600 ./tests/cpp/_ref/unit_tests -ts=layers > gpurun_out/r2l_ref_layers.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_ref_layers.log
timeout 900 ./tests/cpp/_ref/unit_tests -ts=trainer > gpurun_out/r2l_ref_trainer.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_ref_trainer.log
timeout 300 ./tests/cpp/test_dropin > gpurun_out/r2l_cpp.log 2>&1; echo "rc=$?" >> gpurun_out/r2l_cpp.log
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/r2l_pytest.log
