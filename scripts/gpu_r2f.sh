mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/r2f_pytest.log
timeout 900 python bench.py > gpurun_out/r2f_bench.log 2>&1
tail -2 gpurun_out/r2f_bench.log | cut -c1-300
