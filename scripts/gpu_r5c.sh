# Embedding mask walk: parity (oracle + bitwise vs the cursor walk), A/B timing, ncu of the walk
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_embedding_gpu.py -q -x 2>&1 | tail -15 > gpurun_out/r5c_pytest.log
for walk in mask cursor mask cursor; do
  echo "== $walk" >> gpurun_out/r5c_ab.log
  GNSB_EMB_WALK=$walk timeout 300 python experiments/embedding_bench.py >> gpurun_out/r5c_ab.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:emb_ -c 6 -o gpurun_out/r5c_emb \
   python experiments/emb_one.py > gpurun_out/r5c_ncu.log 2>&1
ncu -i gpurun_out/r5c_emb.ncu-rep --page details --csv > gpurun_out/r5c_emb_details.csv 2>/dev/null
cat gpurun_out/r5c_pytest.log | tail -3; cat gpurun_out/r5c_ab.log
