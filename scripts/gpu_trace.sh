mkdir -p gpurun_out
SWEEP_TRACE=1 timeout 600 python experiments/ln_sweep.py 768,1024,2048,4096 15,10,5,0 > gpurun_out/trace_small.log 2>&1
timeout 600 python experiments/ln_sweep.py 768,1024,2048,4096 15,10,5,0 > gpurun_out/sweep_small.log 2>&1
