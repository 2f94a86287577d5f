# same-box A/B of the LN row pass (steady 8 layers + grouped reduce), interleaved twice
# AB_TAGS: "tag" or "tag:maxstages" entries
mkdir -p gpurun_out
for rep in 1 2; do
for t in $AB_TAGS; do
lib=${t%%:*}; st=${t#*:}; [ "$st" = "$t" ] && st=8
GNSB_LN_MAX_STAGES=$st python experiments/ln_steady_trace.py ${AB_DS:-768,1024,2048,4096,8192} 8 --notrace --lib=$lib | sed "s/^/S$st /"
done
done > gpurun_out/ab_${AB_NAME:-x}.log 2>&1
