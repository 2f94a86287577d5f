mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_linear_gpu.py -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_lin.log
GNSB_GRAM_IMPL=1 timeout 600 python -m pytest tests/test_linear_gpu.py -m gpu -q -k gram 2>&1 | tail -3 >> gpurun_out/pytest_lin.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 ncu --clock-control none --set full --import-source on -k regex:gram2 -s 1 -c 1 -o gpurun_out/prof_gram2b python experiments/linear_bench.py > /dev/null 2>&1
