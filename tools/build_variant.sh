#!/bin/bash
# Build a libskx.so variant with extra -D flags for A/B timing (never replaces
# the in-tree library; select it with SKX_LIBSKX=tools/variants/libskx_<name>.so):
#   bash tools/build_variant.sh <name> -DSKX_HIST_SAMPLED=0 ...
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/tools/variants
obj=$out/obj_$name
mkdir -p "$obj"
src=${SKX_VARIANT_SRC:-$root/paper_1910_10063_b200/csrc}  # e.g. a copy holding an older kernel
for s in "$src"/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC \
       -I"$root/include" -I"$src" "$@" -c "$s" -o "$obj/$(basename "${s%.cu}").o" &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out/libskx_$name.so" "$obj"/*.o \
     -lcudart_static -lnccl -lrt -lpthread -ldl
rm -rf "$obj"
echo "$out/libskx_$name.so"
