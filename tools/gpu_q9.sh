set -x
mkdir -p gpurun_out/q9
B="python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-nf --workload"
for i in 1 2 3; do timeout 300 $B c2 > gpurun_out/q9/c2_$i.log 2>&1; python -c "
import json
d=json.loads(open('gpurun_out/q9/c2_$i.log').read().strip().splitlines()[-1]); print('c2', round(d['ms_per_step'],3), round(d['build_ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})"; done
FMMB_TRACE=1 timeout 300 python tools/trace_build.py c2 > gpurun_out/q9/trace.log 2>&1; cat gpurun_out/q9/trace.log
