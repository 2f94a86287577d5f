# LN no-fold A/B (steady trace + per-CTA spread), LN parity, embedding + GEMM bench side numbers
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_ln_gpu.py tests/test_parity_full.py tests/test_embedding_gpu.py tests/test_gns_gpu.py tests/test_nn_gpu.py -x -q 2>&1 | tail -5 > gpurun_out/r2k_pytest.log
python experiments/ln_steady_trace.py 1024 8 > gpurun_out/r2k_trace.log 2>&1
python experiments/ln_steady_trace.py 768,1024,2048,4096,8192 8 --notrace >> gpurun_out/r2k_trace.log 2>&1
python experiments/ln_steady_trace.py 768,1024,2048 8 --notrace --plain >> gpurun_out/r2k_trace.log 2>&1
GNSB_LN_FOLD=1 python experiments/ln_steady_trace.py 768,1024,2048 8 --notrace >> gpurun_out/r2k_trace.log 2>&1
GNSB_LN_FOLD=1 python experiments/ln_steady_trace.py 768,1024,2048 8 --notrace --plain >> gpurun_out/r2k_trace.log 2>&1
timeout 900 python bench.py > gpurun_out/r2k_bench.log 2>&1
