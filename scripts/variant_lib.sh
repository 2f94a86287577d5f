# Build paper_2411_00999_b200/lib/libgnsb_<tag>.so: the product library with ONE
# translation unit recompiled with extra flags (A/B experiments; load it with
# GNSB_LIB_VARIANT=<tag>).   bash scripts/variant_lib.sh <tag> <unit.cu> [nvcc flags]
set -e
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
TAG="$1"; UNIT="$2"; shift 2
cd "$ROOT"
make -s lib
mkdir -p build/var_$TAG
base=$(basename "$UNIT" .cu)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-O3 \
  -Iinclude "$@" -c paper_2411_00999_b200/csrc/$base.cu -o build/var_$TAG/$base.o
objs=$(ls build/obj/*.o build/obj/host/*.o | grep -v "/$base.o$")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2411_00999_b200/lib/libgnsb_$TAG.so $objs build/var_$TAG/$base.o -lrt -ldl -lpthread
echo built paper_2411_00999_b200/lib/libgnsb_$TAG.so
