# Embedding: the raw kernel's ||dW||^2 fold CTA with 8 load chains (it was the call's last CTA)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_embedding_gpu.py -q -x 2>&1 | tail -3 > gpurun_out/r5n_pytest.log
for i in 1 2; do timeout 300 python experiments/embedding_bench.py >> gpurun_out/r5n_ab.log 2>&1; done
timeout 600 ncu --set full --clock-control none -k regex:emb_ -c 3 -o gpurun_out/r5n_emb python experiments/emb_one.py > /dev/null 2>&1
ncu -i gpurun_out/r5n_emb.ncu-rep --page details --csv > gpurun_out/r5n_emb_details.csv 2>/dev/null
cat gpurun_out/r5n_pytest.log; cat gpurun_out/r5n_ab.log
