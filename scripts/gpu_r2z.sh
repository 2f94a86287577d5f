# memcheck / racecheck of the kernels added this round
mkdir -p gpurun_out
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gemm_gpu.py -q -k "forward_and_dx or rank3 or fp64_forward or embedding_forward" > gpurun_out/r2z_memcheck_gemm.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_model_gpu.py -q > gpurun_out/r2z_memcheck_model.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_embedding_gpu.py -q -k "matches_oracle" > gpurun_out/r2z_memcheck_emb.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_ln_gpu.py -q -k "batch_invariant or edge_cases" > gpurun_out/r2z_memcheck_ln.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_linear_gpu.py -q -k "auto_form or tcgen05_weight_grad_form_matches_oracle and 100" > gpurun_out/r2z_memcheck_lin.log 2>&1
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_embedding_gpu.py -q -k "uniform" > gpurun_out/r2z_racecheck_emb.log 2>&1
tail -n 4 gpurun_out/r2z_*.log
