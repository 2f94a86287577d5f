# Round-2 evidence: bench (both arms), launch list, ncu full of the GEMM and the embedding kernels, smoke
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2p_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2p_smoke.log
timeout 900 python bench.py > gpurun_out/r2p_bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/r2p_bench_ref.log 2>&1
NCU="ncu --clock-control none"
timeout 600 $NCU --metrics gpu__time_duration.sum -c 700 --csv --log-file gpurun_out/r2p_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-extra > /dev/null 2>&1
timeout 600 $NCU --set full --import-source on -k regex:gemm_kernel -s 2 -c 1 -o gpurun_out/r2p_gemm_dx \
    python experiments/gemm_bench.py 32768 4096 4096 > /dev/null 2>&1
timeout 600 $NCU --set full --import-source on -k regex:emb_ -s 3 -c 3 -o gpurun_out/r2p_emb \
    python experiments/embedding_bench.py > /dev/null 2>&1
timeout 600 $NCU --set full --import-source on -k regex:ln_bwd_kernel -s 3 -c 1 -o gpurun_out/r2p_rows_d1024 \
    python experiments/ln_steady_trace.py 1024 1 --notrace > /dev/null 2>&1
ls -la gpurun_out/r2p*
