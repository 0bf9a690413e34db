#!/bin/bash
# A/B timing of libskx.so variants on the GPU box:
#   bash tools/ab.sh "<command>" orig <variant> ...
# 'orig' is the in-tree build; <variant> is tools/variants/libskx_<variant>.so.
cmd="$1"; shift
cp paper_1910_10063_b200/libskx.so /tmp/ab_orig.so
for v in "$@"; do
  if [ "$v" = orig ]; then cp /tmp/ab_orig.so paper_1910_10063_b200/libskx.so
  else cp "tools/variants/libskx_$v.so" paper_1910_10063_b200/libskx.so; fi
  echo "== $v"
  timeout 300 bash -c "$cmd" 2>&1 | tail -${AB_TAIL:-2}
done
cp /tmp/ab_orig.so paper_1910_10063_b200/libskx.so
