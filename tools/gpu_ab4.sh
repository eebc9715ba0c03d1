set -x
mkdir -p gpurun_out/ab4
B="python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-nf --workload"
timeout 300 $B c3 > gpurun_out/ab4/base_c3.log 2>&1
FMMB_SCATTER_EARLY=1 timeout 300 $B c3 > gpurun_out/ab4/sce_c3.log 2>&1
FMMB_LC_PER_SM=2 timeout 300 $B c3 > gpurun_out/ab4/lc2_c3.log 2>&1
FMMB_SCATTER_EARLY=1 FMMB_LC_PER_SM=2 timeout 300 $B c3 > gpurun_out/ab4/sce_lc2_c3.log 2>&1
FMMB_LATE_OCC=1 timeout 300 $B c3 > gpurun_out/ab4/late_c3.log 2>&1
for f in gpurun_out/ab4/*.log; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})"; done
