mkdir -p gpurun_out
for bn in 256 128; do
echo "== BN=$bn" >> gpurun_out/r3j.log
GNSB_GEMM_BN=$bn timeout 600 python experiments/gemm_bench.py 8192 768 3072 >> gpurun_out/r3j.log 2>&1
GNSB_GEMM_BN=$bn timeout 600 python experiments/gemm_bench.py 8192 3072 768 >> gpurun_out/r3j.log 2>&1
GNSB_GEMM_BN=$bn timeout 600 python experiments/gemm_bench.py 8192 768 50304 >> gpurun_out/r3j.log 2>&1
GNSB_GEMM_BN=$bn timeout 600 python experiments/toy_step.py >> gpurun_out/r3j.log 2>&1
done
