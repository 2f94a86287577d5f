mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_embedding_gpu.py -x -q 2>&1 | tail -2 > gpurun_out/r2y.log
python experiments/embedding_bench.py >> gpurun_out/r2y.log 2>&1
