# Embedding: PDL chain (sort -> walk -> raw) vs no PDL (variant), parity
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_embedding_gpu.py tests/test_nn_gpu.py -q -x 2>&1 | tail -4 > gpurun_out/r5h_pytest.log
for i in 1 2; do
  echo "== pdl" >> gpurun_out/r5h_ab.log; timeout 300 python experiments/embedding_bench.py >> gpurun_out/r5h_ab.log 2>&1
  echo "== nopdl" >> gpurun_out/r5h_ab.log; GNSB_LIB_VARIANT=nopdl timeout 300 python experiments/embedding_bench.py >> gpurun_out/r5h_ab.log 2>&1
done
cat gpurun_out/r5h_pytest.log | tail -2; cat gpurun_out/r5h_ab.log
