# Last check of the committed state: full GPU tests, smoke, C++ drop-in, bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/r5s_pytest.log
LD_LIBRARY_PATH=paper_2411_00999_b200/lib timeout 300 ./tests/cpp/test_dropin > gpurun_out/r5s_cpp.log 2>&1; echo "rc=$?" >> gpurun_out/r5s_cpp.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5s_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r5s_smoke.log
timeout 900 python bench.py > gpurun_out/r5s_bench.log 2>&1
cat gpurun_out/r5s_pytest.log; tail -1 gpurun_out/r5s_cpp.log; tail -2 gpurun_out/r5s_smoke.log
