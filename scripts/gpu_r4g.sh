for t in w2 r2 w2 r2; do python experiments/ln_steady_trace.py 768,1024,2048,4096,8192 8 --lib=$t --notrace; done
python experiments/ln_steady_trace.py 1024,8192 8 --lib=r2 --notrace --noreduce
python -m pytest tests/test_ln_gpu.py tests/test_gns_gpu.py tests/test_nn_gpu.py tests/test_model_gpu.py -q -x 2>&1 | tail -2
