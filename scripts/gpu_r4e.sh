for t in wt w2 wt w2; do python experiments/ln_steady_trace.py 768,1024,2048,4096,8192 8 --lib=$t --notrace; done
python experiments/ln_steady_trace.py 1024,2048,4096 8 --lib=w2 | grep -v "  L[0-9]"
python -m pytest tests/test_ln_gpu.py -q -x 2>&1 | tail -2
