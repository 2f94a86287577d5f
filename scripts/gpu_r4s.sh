# memcheck / racecheck of this round's LN row-pass slot stores, stage-2 bulk staging and the embedding grid change
mkdir -p gpurun_out
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_ln_gpu.py -q -k "test_backward_matches_oracle or grouped_reduce_one_example or deferred_grouped or many_examples_blocked" > gpurun_out/r4s_memcheck_ln.log 2>&1
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_ln_gpu.py -q -k "test_backward_matches_oracle and (bfloat16-4-64-1024 or bfloat16-3-50-2048 or float32-2-33-1024 or float32-1-1000-256) or grouped_reduce_one_example" > gpurun_out/r4s_racecheck_ln.log 2>&1
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_ln_gpu.py -q -k "test_backward_matches_oracle and (bfloat16-4-64-1024 or float32-1-1000-256)" > gpurun_out/r4s_synccheck_ln.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_embedding_gpu.py -q -k "matches_oracle" > gpurun_out/r4s_memcheck_emb.log 2>&1
tail -n 3 gpurun_out/r4s_*.log
