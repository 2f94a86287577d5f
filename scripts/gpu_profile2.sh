mkdir -p gpurun_out
NCU="ncu --clock-control none"
timeout 600 $NCU --metrics gpu__time_duration.sum -c 600 --csv --log-file gpurun_out/launches_c.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-extra > /dev/null 2>&1
timeout 600 $NCU --set full --import-source on -k regex:gram_norms -s 3 -c 1 -o gpurun_out/prof_gram_v2 \
    python experiments/linear_bench.py > /dev/null 2>&1
timeout 600 $NCU --set full --import-source on -k regex:ln_bwd_reduce_group -s 3 -c 1 -o gpurun_out/prof_reduce_group \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-extra > /dev/null 2>&1
timeout 600 $NCU --set full --import-source on -k regex:ln_bwd_kernel -s 9 -c 1 -o gpurun_out/prof_rows_d8192 \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-extra --d-list 8192 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
