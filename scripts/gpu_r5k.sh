# Embedding sort: bucket count (default <= 4096 buckets; bk1 / bk2: <= 1 / 2 buckets per padded key)
mkdir -p gpurun_out
for i in 1 2; do
  for v in default bk1 bk2; do
    echo "== $v" >> gpurun_out/r5k_ab.log
    if [ $v = default ]; then timeout 300 python experiments/embedding_bench.py >> gpurun_out/r5k_ab.log 2>&1
    else GNSB_LIB_VARIANT=$v timeout 300 python experiments/embedding_bench.py >> gpurun_out/r5k_ab.log 2>&1; fi
  done
done
cat gpurun_out/r5k_ab.log
