set -x
mkdir -p gpurun_out/q8
timeout 900 python -m pytest tests/test_gpu_build_parity.py tests/test_gpu_northstar.py tests/test_gpu_threads.py -q -x 2>&1 | tail -2
B="python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-nf --workload"
for w in c2 c3 c4; do timeout 300 $B $w > gpurun_out/q8/$w.log 2>&1; python -c "
import json
d=json.loads(open('gpurun_out/q8/$w.log').read().strip().splitlines()[-1]); print('$w', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})"; done
