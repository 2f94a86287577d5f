# Embedding: raw kernel folds the sums and the flag (one launch instead of three + a copy)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_embedding_gpu.py tests/test_nn_gpu.py tests/test_trainer_gpu.py -q -x 2>&1 | tail -15 > gpurun_out/r5e_pytest.log
for i in 1 2; do
  echo "== default" >> gpurun_out/r5e_ab.log; timeout 300 python experiments/embedding_bench.py >> gpurun_out/r5e_ab.log 2>&1
done
cat gpurun_out/r5e_pytest.log | tail -3; cat gpurun_out/r5e_ab.log
