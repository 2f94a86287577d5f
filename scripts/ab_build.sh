# Build experiments/libln_sweep_<tag>.so from the csrc of git revision <rev>
# (or "wt" = the working tree) with the CURRENT experiments/ln_sweep.cu, for
# same-box A/B timing (experiments/ln_steady_trace.py --lib <tag>).
#   bash scripts/ab_build.sh <rev|wt> <tag> [extra nvcc flags]
set -e
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
REV="$1"; TAG="$2"; shift 2
W=/tmp/ab_$TAG
rm -rf "$W"; mkdir -p "$W/experiments" "$W/paper_2411_00999_b200"
if [ "$REV" = "wt" ]; then
  cp -r "$ROOT/paper_2411_00999_b200/csrc" "$W/paper_2411_00999_b200/"
else
  (cd "$ROOT" && git archive "$REV" paper_2411_00999_b200/csrc) | tar -x -C "$W"
fi
cp "$ROOT/experiments/ln_sweep.cu" "$W/experiments/"
cd "$W/experiments"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC \
  -shared -I"$ROOT/include" "$@" -o "$ROOT/experiments/libln_sweep_$TAG.so" ln_sweep.cu ../paper_2411_00999_b200/csrc/ln_reduce.cu
