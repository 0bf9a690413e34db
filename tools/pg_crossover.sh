# One-pass (129) vs forced partitioned (24705) vs planned (8321) C2 step per skew: where the
# plan's 30% threshold sits against the measured crossover
mkdir -p gpurun_out
for z in ${PG_ZS:-0.75 0.9}; do for pol in 129 24705 8321; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu --no-e2e --policy $pol --z $z 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('z=$z pol=$pol', round(d['ms_per_step'],3), d['config']['gather_path'])"
done; done
