# C5 compact records (in-tree) vs sparse records (variant); C4 histogram top key in a register
# (variant topreg) vs in-tree; alternated.  Then parity of the in-tree build.
for rep in 1 2; do
for v in orig sparse topreg; do
  if [ $v = orig ]; then unset SKX_LIBSKX; else export SKX_LIBSKX=$PWD/tools/variants/libskx_$v.so; fi
  python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --configs c4,c5 > gpurun_out/ab4_$v.json 2>gpurun_out/ab4_$v.err
  python -c "import json;d=json.load(open('gpurun_out/ab4_$v.json'));print('$v', 'c4', round(d['index_build_c4']['ms_per_build'],3), d['index_build_c4']['phases_ms']['histogram'], 'c5', round(d['select_c5']['ms_per_step'],3))"
done
done
unset SKX_LIBSKX
python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x 2>&1 | tail -2
python -m pytest tests/test_gpu_scale.py -q -x -k "c5 or c4" 2>&1 | tail -2
SKX_LIBSKX=$PWD/tools/variants/libskx_topreg.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -k "hist or count or rebuild or c4 or golden" 2>&1 | tail -2
