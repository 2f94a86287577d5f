# Build the experiment-only shared libraries (not part of the product).
set -e
cd "$(dirname "$0")/../experiments"
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -shared -I../include"
$NV -o libln_sweep.so ln_sweep.cu ../paper_2411_00999_b200/csrc/ln_reduce.cu &
$NV -o liblaunch_overhead.so launch_overhead.cu &
$NV -o libstream_bench.so stream_bench.cu &
$NV -o libln_fwd_sweep.so ln_fwd_sweep.cu &
wait
