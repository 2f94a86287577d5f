# Embedding mask walk at 24 warps per SM (85 registers; forced mask walk) vs the default 16
mkdir -p gpurun_out
for i in 1 2; do
  echo "== default" >> gpurun_out/r5o_ab.log; timeout 300 python experiments/embedding_bench.py >> gpurun_out/r5o_ab.log 2>&1
  echo "== m768 (mask forced)" >> gpurun_out/r5o_ab.log; GNSB_EMB_WALK=mask GNSB_LIB_VARIANT=m768 timeout 300 python experiments/embedding_bench.py >> gpurun_out/r5o_ab.log 2>&1
  echo "== m768pb2 (mask forced)" >> gpurun_out/r5o_ab.log; GNSB_EMB_WALK=mask GNSB_LIB_VARIANT=m768pb2 timeout 300 python experiments/embedding_bench.py >> gpurun_out/r5o_ab.log 2>&1
done
grep -E "==|V=50257 D=768 torch.bfloat16" gpurun_out/r5o_ab.log
