set -x
mkdir -p gpurun_out/ab6
B="python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-nf --workload"
for w in c2 c4; do
timeout 300 $B $w > gpurun_out/ab6/base_$w.log 2>&1
FMMB_LC_PER_SM=1 timeout 300 $B $w > gpurun_out/ab6/lc1_$w.log 2>&1
FMMB_LC_PER_SM=3 timeout 300 $B $w > gpurun_out/ab6/lc3_$w.log 2>&1
done
FMMB_TRACE=1 FMMB_LC_PER_SM=1 timeout 300 python tools/trace_build.py c2 > gpurun_out/ab6/trace_lc1.log 2>&1
for f in gpurun_out/ab6/*_c?.log; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})"; done
cat gpurun_out/ab6/trace_lc1.log
