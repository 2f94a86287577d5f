mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_embedding_gpu.py tests/test_model_gpu.py -x -q 2>&1 | tail -3 > gpurun_out/r2x.log
python experiments/embedding_bench.py >> gpurun_out/r2x.log 2>&1
GNSB_EMB_SORT=bitonic python experiments/embedding_bench.py >> gpurun_out/r2x.log 2>&1
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum -k regex:emb_ -c 12 python experiments/embedding_bench.py 2>/dev/null | grep -E "emb_|gpu__time" | head -30 >> gpurun_out/r2x.log
