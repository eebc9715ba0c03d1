set -x
mkdir -p gpurun_out/ab8
B="python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-nf --workload"
for w in c2 c4; do
timeout 300 $B $w > gpurun_out/ab8/base_$w.log 2>&1
FMMB_LOCAL_AFTER=1 timeout 300 $B $w > gpurun_out/ab8/after_$w.log 2>&1
FMMB_LOCAL_AFTER=1 FMMB_LC_PER_SM=3 timeout 300 $B $w > gpurun_out/ab8/after3_$w.log 2>&1
done
for f in gpurun_out/ab8/*_c?.log; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})"; done
