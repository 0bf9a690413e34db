#!/bin/bash
# A/B timing of libskx.so variants on the GPU box:
#   bash tools/ab.sh "<command>" orig <variant> ...
# 'orig' is the in-tree build; <variant> is tools/variants/libskx_<variant>.so,
# selected through SKX_LIBSKX (paper_1910_10063_b200/_native.py) -- the in-tree
# library is never overwritten, so an interrupted run cannot leave a variant
# in place.
cmd="$1"; shift
for v in "$@"; do
  if [ "$v" = orig ]; then unset SKX_LIBSKX
  else export SKX_LIBSKX="$PWD/tools/variants/libskx_$v.so"; fi
  echo "== $v"
  timeout 300 bash -c "$cmd" 2>&1 | tail -${AB_TAIL:-2}
done
