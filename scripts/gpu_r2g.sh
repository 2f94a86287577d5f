# Round-2 state check after re-entry: GPU tests, C++ drop-in, smoke, bench, launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2g_smi.log
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/r2g_pytest.log
LD_LIBRARY_PATH=paper_2411_00999_b200/lib timeout 300 ./tests/cpp/test_dropin > gpurun_out/r2g_cpp.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_cpp.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_smoke.log
timeout 900 python bench.py > gpurun_out/r2g_bench.log 2>&1
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum -c 700 --csv --log-file gpurun_out/r2g_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-extra > /dev/null 2>&1
tail -3 gpurun_out/r2g_*.log | cut -c1-400
