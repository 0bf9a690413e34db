# C5: pass-1 scan/store rework (in-tree) vs the previous pass 1 (variant), alternated
for rep in 1 2; do
for v in orig selprev; do
  if [ $v = orig ]; then unset SKX_LIBSKX; else export SKX_LIBSKX=$PWD/tools/variants/libskx_$v.so; fi
  python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --configs c5 > gpurun_out/ab3_$v.json 2>gpurun_out/ab3_$v.err
  python -c "import json;d=json.load(open('gpurun_out/ab3_$v.json'));print('$v', 'c5', round(d['select_c5']['ms_per_step'],3), d['select_c5']['roofline_frac'])"
done
done
unset SKX_LIBSKX
python -m pytest tests/test_gpu_parity.py -q -x -k "select or golden or kat" 2>&1 | tail -2
python -m pytest tests/test_gpu_scale.py -q -x -k c5 2>&1 | tail -2
