set -x
mkdir -p gpurun_out/ab7
B="python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-nf --workload"
for w in c3 c2 c4; do
timeout 300 $B $w > gpurun_out/ab7/base_$w.log 2>&1
FMMB_SIDE_PRIO=1 timeout 300 $B $w > gpurun_out/ab7/prio_$w.log 2>&1
done
FMMB_SCATTER_AFTER_COUNT=1 timeout 300 $B c3 > gpurun_out/ab7/sac_c3.log 2>&1
FMMB_SIDE_PRIO=1 FMMB_TRACE=1 timeout 300 python tools/trace_build.py c3 > gpurun_out/ab7/trace_prio_c3.log 2>&1
FMMB_TRACE=1 timeout 300 python tools/trace_build.py c3 > gpurun_out/ab7/trace_c3.log 2>&1
for f in gpurun_out/ab7/*_c?.log; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})"; done
cat gpurun_out/ab7/trace_c3.log gpurun_out/ab7/trace_prio_c3.log
