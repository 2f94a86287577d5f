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
timeout 600 $NCU --set full --import-source on -k regex:ln_fwd -s 1 -c 1 -o gpurun_out/final_fwd_d1024 \
    python bench.py --steps 1 --warmup 3 --no-cpu --d-list 1024 > /dev/null 2>&1
ls -la gpurun_out/final_*
# memcheck over the kernels changed since the last sanitizer pass (CTA-pair wgrad, warp forward)
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_linear_gpu.py -q -k "weight_grad_form_matches" > gpurun_out/final_memcheck_lin.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_ln_gpu.py -q -k "forward or edge or oracle" > gpurun_out/final_memcheck_ln.log 2>&1
tail -n 3 gpurun_out/final_memcheck_*.log
