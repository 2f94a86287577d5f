# LN backward steady timeline at narrow/wide widths, fused vs plain (per-CTA phase stamps).
mkdir -p gpurun_out
python experiments/ln_steady_trace.py 1024,8192 8 > gpurun_out/r2h_trace.log 2>&1
python experiments/ln_steady_trace.py 1024,8192 8 --plain >> gpurun_out/r2h_trace.log 2>&1
python experiments/ln_steady_trace.py 768,1024,2048,4096,8192 8 --notrace >> gpurun_out/r2h_trace.log 2>&1
python experiments/ln_steady_trace.py 768,1024,2048,4096,8192 8 --notrace --plain >> gpurun_out/r2h_trace.log 2>&1
python experiments/stream_sets.py > gpurun_out/r2h_stream.log 2>&1
tail -3 gpurun_out/r2h_*.log
