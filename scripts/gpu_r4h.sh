python experiments/ln_steady_trace.py 768,1024,2048,4096,8192 8 --lib=r2 --notrace --redtrace
