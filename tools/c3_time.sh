# C3 group-by step time of bench.py (for tools/ab.sh A/B runs of library variants)
python bench.py --steps 10 --warmup 3 --configs c3 --no-cpu --no-e2e 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); g=d.get('groupby_c3',{}); print(g.get('ms_per_step'), g.get('phases_ms'))"
