# park A/B at D=1024/2048 (steady, fused+plain), embedding CTA-size A/B, LN parity
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_ln_gpu.py tests/test_parity_full.py tests/test_embedding_gpu.py -x -q 2>&1 | tail -3 > gpurun_out/r2q_pytest.log
for i in 1 2; do
python experiments/ln_steady_trace.py 1024,2048 8 --notrace >> gpurun_out/r2q_trace.log 2>&1
GNSB_LN_PARK=0 python experiments/ln_steady_trace.py 1024,2048 8 --notrace >> gpurun_out/r2q_trace.log 2>&1
done
python experiments/ln_steady_trace.py 1024,2048 8 --notrace --plain >> gpurun_out/r2q_trace.log 2>&1
python experiments/embedding_bench.py > gpurun_out/r2q_emb.log 2>&1
GNSB_EMB_CTA=64 python experiments/embedding_bench.py >> gpurun_out/r2q_emb.log 2>&1
