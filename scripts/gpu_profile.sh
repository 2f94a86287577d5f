# Round-1 ncu evidence: launch list of the bench step, full captures of the
# LayerNorm row kernel (D=4096 and D=768), the stage-2 reduce kernel, and the
# two tcgen05 linear kernels.  Numbers printed under ncu are never bench values.
mkdir -p gpurun_out
NCU="ncu --clock-control none"
timeout 600 $NCU --metrics gpu__time_duration.sum -c 600 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-extra > gpurun_out/launches_bench.log 2>&1
timeout 600 $NCU --set full --import-source on -k regex:ln_bwd_kernel -s 6 -c 1 -o gpurun_out/prof_rows_d4096 \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-extra --d-list 4096 > /dev/null 2>&1
timeout 600 $NCU --set full --import-source on -k regex:ln_bwd_kernel -s 6 -c 1 -o gpurun_out/prof_rows_d768 \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-extra --d-list 768 > /dev/null 2>&1
timeout 600 $NCU --set full --import-source on -k regex:ln_bwd_reduce -s 6 -c 1 -o gpurun_out/prof_reduce_d4096 \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-extra --d-list 4096 > /dev/null 2>&1
timeout 600 $NCU --set full --import-source on -k regex:gram_norms -s 3 -c 1 -o gpurun_out/prof_gram \
    python experiments/linear_bench.py > /dev/null 2>&1
timeout 600 $NCU --set full --import-source on -k regex:wgrad_norms -s 3 -c 1 -o gpurun_out/prof_wgrad \
    python experiments/linear_bench.py > /dev/null 2>&1
ls -la gpurun_out
