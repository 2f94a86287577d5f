for t in w2 xa xb w2 xa xb; do python experiments/ln_steady_trace.py 2048 8 --lib=$t --notrace; done
for t in xa xb; do python experiments/ln_steady_trace.py 2048 8 --lib=$t | grep -v "  L[0-9]"; done
