mkdir -p gpurun_out
python experiments/ln_steady_trace.py 768,1024,2048,4096,8192 8 > gpurun_out/r2c_trace.log 2>&1
python experiments/ln_steady_trace.py 1024,2048 8 --plain >> gpurun_out/r2c_trace.log 2>&1
