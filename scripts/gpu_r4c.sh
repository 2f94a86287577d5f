python experiments/ln_steady_trace.py 1024,2048 8 --lib=wt
GNSB_LN_PARK=1 python experiments/ln_steady_trace.py 1024,2048 8 --lib=wt
GNSB_LN_PARK=1 python experiments/ln_steady_trace.py 1024,2048 8 --lib=wt --notrace
python experiments/ln_steady_trace.py 1024,2048 8 --lib=wt --notrace
