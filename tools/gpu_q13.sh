set -x
mkdir -p gpurun_out/q13
timeout 1200 python -m pytest tests/test_gpu_build_parity.py tests/test_gpu_northstar.py tests/test_gpu_golden.py tests/test_gpu_threads.py tests/test_gpu_errors.py tests/test_gpu_properties.py -q -x 2>&1 | tail -2
B="python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-nf --workload"
for w in c2 c4 c1 c3; do timeout 300 $B $w > gpurun_out/q13/$w.log 2>&1; python -c "
import json
d=json.loads(open('gpurun_out/q13/$w.log').read().strip().splitlines()[-1]); print('$w', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})"; done
timeout 300 python tools/c1_latency.py c1 2>&1 | head -2
