cp paper_1910_10063_b200/libskx.so /tmp/orig.so
for v in orig h1024_14_1 h512_14_1 h256_13_6; do
  if [ $v = orig ]; then cp /tmp/orig.so paper_1910_10063_b200/libskx.so; else cp tools/variants/libskx_$v.so paper_1910_10063_b200/libskx.so; fi
  echo "== $v"; timeout 120 python tools/index_sweep.py 2>&1 | tail -1 | cut -c1-100
done
cp /tmp/orig.so paper_1910_10063_b200/libskx.so
