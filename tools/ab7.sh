# C3 group-by: rows per thread per iteration x stream pipelining (macro builds), alternated
for rep in 1 2; do
for v in orig u2p0 u2p1 u1p0; do
  if [ $v = orig ]; then unset SKX_LIBSKX; else export SKX_LIBSKX=$PWD/tools/variants/libskx_$v.so; fi
  python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --configs c3 > gpurun_out/ab7_$v.json 2>gpurun_out/ab7_$v.err
  python -c "import json;d=json.load(open('gpurun_out/ab7_$v.json'));print('$v', 'c3', round(d['groupby_c3']['ms_per_step'],3))"
done
done
