# Embedding mask walk v2: parity, A/B (policy default vs cursor; 768-thread occupancy; 4-row blocks)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_embedding_gpu.py -q -x 2>&1 | tail -15 > gpurun_out/r5d_pytest.log
for i in 1 2; do
  echo "== default" >> gpurun_out/r5d_ab.log; timeout 300 python experiments/embedding_bench.py >> gpurun_out/r5d_ab.log 2>&1
  echo "== cursor" >> gpurun_out/r5d_ab.log; GNSB_EMB_WALK=cursor timeout 300 python experiments/embedding_bench.py >> gpurun_out/r5d_ab.log 2>&1
  echo "== mocc768" >> gpurun_out/r5d_ab.log; GNSB_LIB_VARIANT=mocc768 timeout 300 python experiments/embedding_bench.py >> gpurun_out/r5d_ab.log 2>&1
  echo "== rpw4 (forced mask)" >> gpurun_out/r5d_ab.log; GNSB_EMB_WALK=mask GNSB_LIB_VARIANT=rpw4 timeout 300 python experiments/embedding_bench.py >> gpurun_out/r5d_ab.log 2>&1
done
cat gpurun_out/r5d_pytest.log | tail -3; cat gpurun_out/r5d_ab.log
