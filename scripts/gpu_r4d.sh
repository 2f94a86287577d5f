for t in wt u4 wt u4; do python experiments/ln_steady_trace.py 768,1024,2048,4096 8 --lib=$t --notrace; done
python experiments/ln_steady_trace.py 1024,2048 8 --lib=u4 | grep -v "  L[0-9]"
