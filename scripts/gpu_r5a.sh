# Re-entry validation: GPU tests, C++ drop-in, smoke, bench (both arms)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r5a_gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r5a_pytest.log
LD_LIBRARY_PATH=paper_2411_00999_b200/lib timeout 300 ./tests/cpp/test_dropin > gpurun_out/r5a_cpp.log 2>&1; echo "rc=$?" >> gpurun_out/r5a_cpp.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5a_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r5a_smoke.log
timeout 900 python bench.py > gpurun_out/r5a_bench.log 2>&1
tail -3 gpurun_out/r5a_pytest.log; tail -2 gpurun_out/r5a_smoke.log; tail -c 600 gpurun_out/r5a_bench.log
