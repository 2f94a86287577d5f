set -x
for a in "" "--noreduce"; do
  python experiments/ln_steady_trace.py 768,1024,2048,4096,8192 8 --notrace --lib=wt $a
done
python experiments/ln_steady_trace.py 1024 8 --lib=wt
