mkdir -p gpurun_out
python experiments/ln_steady_trace.py 768,1024,2048,4096 8 > gpurun_out/r2b_trace.log 2>&1
python experiments/ln_steady_trace.py 1024,2048 8 --plain >> gpurun_out/r2b_trace.log 2>&1
python experiments/aten_ln_bwd.py > gpurun_out/r2b_aten.log 2>&1
python experiments/stream_sets.py > gpurun_out/r2b_stream.log 2>&1
tail -5 gpurun_out/r2b_*.log
