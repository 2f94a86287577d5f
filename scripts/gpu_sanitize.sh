mkdir -p gpurun_out
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 --error-exitcode 9 \
    python -m pytest tests/test_ln_gpu.py -m gpu -q -x -k "test_backward_matches_oracle or deferred or plain_equals" > gpurun_out/sanitize_ln.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_ln.log
timeout 900 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 --error-exitcode 9 \
    python -m pytest tests/test_embedding_gpu.py tests/test_linear_gpu.py -m gpu -q -x -k "not cfg3" > gpurun_out/sanitize_lin.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_lin.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 --error-exitcode 9 \
    python -m pytest tests/test_ln_gpu.py -m gpu -q -x -k "test_backward_matches_oracle and (dt0 or dt6 or dt9)" > gpurun_out/racecheck_ln.log 2>&1; echo "rc=$?" >> gpurun_out/racecheck_ln.log
