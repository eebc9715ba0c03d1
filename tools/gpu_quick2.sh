timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for w in c2 c3 c1; do timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['phases_ms'].items()})"; done
