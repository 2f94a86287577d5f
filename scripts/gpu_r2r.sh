mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_embedding_gpu.py tests/test_model_gpu.py tests/test_trainer_gpu.py -x -q 2>&1 | tail -3 > gpurun_out/r2r_pytest.log
python experiments/embedding_bench.py > gpurun_out/r2r_emb.log 2>&1
timeout 600 ncu --clock-control none --set full -k regex:emb_ -s 3 -c 3 -o gpurun_out/r2r_emb python experiments/embedding_bench.py > /dev/null 2>&1
