# steady sweep of every LN-bwd configuration at D=1024/2048 with the 4-stage ring
mkdir -p gpurun_out
timeout 1200 python experiments/ln_sweep_steady.py 1024,2048 > gpurun_out/r2v_sweep.log 2>&1
timeout 300 python experiments/linear_bench.py > gpurun_out/r2v_linear.log 2>&1
