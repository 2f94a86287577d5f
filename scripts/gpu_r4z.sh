# round-end style validation: all GPU tests, C++ drop-in, smoke, both bench arms, launch list
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/r4z_pytest.log
LD_LIBRARY_PATH=paper_2411_00999_b200/lib timeout 300 ./tests/cpp/test_dropin > gpurun_out/r4z_cpp.log 2>&1; echo "rc=$?" >> gpurun_out/r4z_cpp.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4z_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r4z_smoke.log
timeout 900 python bench.py --impl reference > gpurun_out/r4z_bench_ref.log 2>&1
timeout 900 python bench.py > gpurun_out/r4z_bench.log 2>&1
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum -c 700 --csv --log-file gpurun_out/r4z_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-extra > /dev/null 2>&1
