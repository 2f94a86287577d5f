# Final-build ncu of the dominant kernel (D=8192 LN row pass): full set, for roofline.traffic
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ln_bwd_kernel -s 9 -c 1 -o gpurun_out/r5q_rows_d8192 \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-extra --d-list 8192 > gpurun_out/r5q_ncu.log 2>&1
ls -la gpurun_out/r5q_rows_d8192.ncu-rep
