# Round-end evidence in one call: full GPU tests, C++ drop-in, smoke, both bench arms,
# the launch list of the bench step and ncu captures of the current top kernels.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/final_pytest.log
LD_LIBRARY_PATH=paper_2411_00999_b200/lib timeout 300 ./tests/cpp/test_dropin > gpurun_out/final_cpp.log 2>&1; echo "rc=$?" >> gpurun_out/final_cpp.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/final_bench_ref.log 2>&1
timeout 900 python bench.py > gpurun_out/final_bench.log 2>&1
NCU="ncu --clock-control none"
timeout 600 $NCU --metrics gpu__time_duration.sum -c 700 --csv --log-file gpurun_out/final_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-extra > /dev/null 2>&1
timeout 600 $NCU --set full --import-source on -k regex:ln_bwd_kernel -s 9 -c 1 -o gpurun_out/final_rows_d8192 \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-extra --d-list 8192 > /dev/null 2>&1
timeout 600 $NCU --set full --import-source on -k regex:ln_fwd_ring -s 1 -c 1 -o gpurun_out/final_fwd_d4096 \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-extra --d-list 4096 > /dev/null 2>&1
ls -la gpurun_out/final_*
