# Round 2 first GPU call: full GPU tests (incl. the new full-size parity tests), C++ drop-in, smoke, bench.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.log
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15 2>&1 | tail -60 > gpurun_out/r2a_pytest.log
LD_LIBRARY_PATH=paper_2411_00999_b200/lib timeout 300 ./tests/cpp/test_dropin > gpurun_out/r2a_cpp.log 2>&1; echo "rc=$?" >> gpurun_out/r2a_cpp.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2a_smoke.log
timeout 900 python bench.py > gpurun_out/r2a_bench.log 2>&1
tail -3 gpurun_out/r2a_*.log
