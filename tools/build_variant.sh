#!/bin/bash
# Build an experiment variant of libpolar_b200.so with extra -D flags:
#   tools/build_variant.sh NAME -DPS_SHA_STAGES=6 -DPS_SHA_CTAS=2
# -> tools/micro/libpolar_NAME.so (load with PS_LIB_PATH=...).
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/build/variant_$name
mkdir -p "$out"
for f in "$root"/paper_2505_14884_b200/csrc/*.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -I "$root/include" "$@" -c "$f" -o "$out/$(basename "$f" .cu).o" &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$root/tools/micro/libpolar_$name.so" "$out"/*.o
echo "built tools/micro/libpolar_$name.so"
