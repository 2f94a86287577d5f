mkdir -p gpurun_out
for v in "" rpw4 rpw2; do echo "== variant '$v'" >> gpurun_out/r2w_emb.log; GNSB_LIB_VARIANT=$v python experiments/embedding_bench.py >> gpurun_out/r2w_emb.log 2>&1; done
GNSB_LIB_VARIANT=rpw2 timeout 600 python -m pytest tests/test_embedding_gpu.py -x -q 2>&1 | tail -2 >> gpurun_out/r2w_emb.log
