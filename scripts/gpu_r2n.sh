# Evidence: GEMM timings vs cuBLAS, ncu of the GEMM (dx) and the LN row pass at D=1024, bench launch list
mkdir -p gpurun_out
timeout 600 python experiments/gemm_bench.py > gpurun_out/r2n_gemm.log 2>&1
NCU="ncu --clock-control none"
timeout 600 $NCU --set full --import-source on -k regex:gemm_kernel -s 2 -c 1 -o gpurun_out/r2n_gemm_dx \
    python experiments/gemm_bench.py 32768 4096 4096 > /dev/null 2>&1
timeout 600 $NCU --set full --import-source on -k regex:ln_bwd_kernel -s 3 -c 1 -o gpurun_out/r2n_rows_d1024 \
    python experiments/ln_steady_trace.py 1024 1 --notrace > /dev/null 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum -c 700 --csv --log-file gpurun_out/r2n_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-extra > /dev/null 2>&1
ls -la gpurun_out/r2n*
