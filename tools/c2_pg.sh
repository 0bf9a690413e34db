# C2 step time per gather policy and skew (partitioned 8321 vs one-pass 129)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "${PG_TESTS:-partitioned or store_policies}" 2>&1 | tail -5
for pol in ${PG_POLS:-8321 129}; do for z in ${PG_ZS:-1.0 0.5 1.5}; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu --no-e2e --policy $pol --z $z > gpurun_out/c2_$pol_$z.log 2>&1
echo "pol=$pol z=$z $(tail -1 gpurun_out/c2_$pol_$z.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], round(d['roofline']['frac'],3))" 2>&1 | tail -1)"
done; done
