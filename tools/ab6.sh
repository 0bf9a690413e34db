# C5 launch-shape variants (macro builds) vs in-tree, alternated
for rep in 1 2; do
for v in orig per8 smem192 smem64 grp2; do
  if [ $v = orig ]; then unset SKX_LIBSKX; else export SKX_LIBSKX=$PWD/tools/variants/libskx_$v.so; fi
  python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --configs c5 > gpurun_out/ab6_$v.json 2>gpurun_out/ab6_$v.err
  python -c "import json;d=json.load(open('gpurun_out/ab6_$v.json'));print('$v', 'c5', round(d['select_c5']['ms_per_step'],3))"
done
done
