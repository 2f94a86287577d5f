# GEMM parity + LN after the warp-per-example square fold in stage 2.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -30 > gpurun_out/r2i_gemm.log
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2i_pytest.log
python experiments/ln_steady_trace.py 768,1024,2048,4096,8192 8 --notrace > gpurun_out/r2i_trace.log 2>&1
python experiments/ln_steady_trace.py 768,1024,2048,4096,8192 8 --notrace --plain >> gpurun_out/r2i_trace.log 2>&1
tail -3 gpurun_out/r2i_*.log
