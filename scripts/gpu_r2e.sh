mkdir -p gpurun_out
python experiments/ln_steady_trace.py 768,1024,2048,4096,8192 8 --notrace > gpurun_out/r2e_time.log 2>&1
python experiments/ln_steady_trace.py 1024,2048 8 --plain --notrace >> gpurun_out/r2e_time.log 2>&1
NCU="ncu --clock-control none"
timeout 600 $NCU --set full --import-source on -k regex:ln_bwd_kernel -s 3 -c 1 -o gpurun_out/r2e_rows_d1024 \
    python experiments/ln_steady_trace.py 1024 1 --notrace > /dev/null 2>&1
ls gpurun_out
