# Embedding mask walk: first-token rows in flight per batch (PB = 4 default, 6, 8), parity of the default
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_embedding_gpu.py -q -x 2>&1 | tail -3 > gpurun_out/r5l_pytest.log
for i in 1 2; do
  for v in default pb6 pb8; do
    echo "== $v" >> gpurun_out/r5l_ab.log
    if [ $v = default ]; then timeout 300 python experiments/embedding_bench.py >> gpurun_out/r5l_ab.log 2>&1
    else GNSB_LIB_VARIANT=$v timeout 300 python experiments/embedding_bench.py >> gpurun_out/r5l_ab.log 2>&1; fi
  done
done
cat gpurun_out/r5l_pytest.log; grep -E "==|V=50257 D=768 torch.bfloat16" gpurun_out/r5l_ab.log
