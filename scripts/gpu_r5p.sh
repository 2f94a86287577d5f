# Embedding mask walk: the batch's per-pair squares reduced with interleaved butterflies
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_embedding_gpu.py -q -x 2>&1 | tail -3 > gpurun_out/r5p_pytest.log
for i in 1 2; do timeout 300 python experiments/embedding_bench.py >> gpurun_out/r5p_ab.log 2>&1; done
cat gpurun_out/r5p_pytest.log; grep "V=50257" gpurun_out/r5p_ab.log
