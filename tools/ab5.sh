# C4 histogram: software-pipelined FK stream + one-branch lookup (in-tree) vs previous (variant)
for rep in 1 2; do
for v in orig histprev; do
  if [ $v = orig ]; then unset SKX_LIBSKX; else export SKX_LIBSKX=$PWD/tools/variants/libskx_$v.so; fi
  python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --configs c4 > gpurun_out/ab5_$v.json 2>gpurun_out/ab5_$v.err
  python -c "import json;d=json.load(open('gpurun_out/ab5_$v.json'));print('$v', 'c4', round(d['index_build_c4']['ms_per_build'],3), d['index_build_c4']['phases_ms'])"
done
done
unset SKX_LIBSKX
python -m pytest tests/test_gpu_parity.py -q -x -k "hist or count or rebuild or golden or kat or scratch" 2>&1 | tail -2
python -m pytest tests/test_gpu_scale.py -q -x -k "c4" 2>&1 | tail -2
