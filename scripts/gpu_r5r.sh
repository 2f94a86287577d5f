# Embedding: two sort CTAs per example (id halves) vs one (GNSB_EMB_SORT_HALVES=0), parity
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_embedding_gpu.py tests/test_nn_gpu.py -q -x 2>&1 | tail -3 > gpurun_out/r5r_pytest.log
for i in 1 2; do
  echo "== halves" >> gpurun_out/r5r_ab.log; timeout 300 python experiments/embedding_bench.py >> gpurun_out/r5r_ab.log 2>&1
  echo "== one" >> gpurun_out/r5r_ab.log; GNSB_EMB_SORT_HALVES=0 timeout 300 python experiments/embedding_bench.py >> gpurun_out/r5r_ab.log 2>&1
done
cat gpurun_out/r5r_pytest.log; grep -E "==|V=50257 D=768 torch.bfloat16" gpurun_out/r5r_ab.log
