mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_linear_gpu.py tests/test_embedding_gpu.py tests/test_model_gpu.py -x -q 2>&1 | tail -3 > gpurun_out/r2u_pytest.log
timeout 300 python experiments/linear_bench.py > gpurun_out/r2u_linear.log 2>&1
timeout 800 python experiments/form_sweep.py > gpurun_out/r2u_forms.log 2>&1
timeout 600 ncu --clock-control none --set full -k regex:wgrad_norms -s 1 -c 1 -o gpurun_out/r2u_wgrad python experiments/linear_bench.py > /dev/null 2>&1
