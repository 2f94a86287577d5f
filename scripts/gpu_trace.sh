mkdir -p gpurun_out
timeout 600 python experiments/ln_sweep.py 768,1024,2048,4096 15,35,36,37,38,41,10,5,39,40,0 > gpurun_out/sweep_cps.log 2>&1
