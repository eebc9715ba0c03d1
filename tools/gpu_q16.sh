set -x
mkdir -p gpurun_out/q16
B="python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-nf --workload"
for w in c2 c3 c4 c2; do timeout 300 $B $w > gpurun_out/q16/$w.log 2>&1; python -c "
import json
d=json.loads(open('gpurun_out/q16/$w.log').read().strip().splitlines()[-1]); print('$w', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_lists_cscan|k_rank" --csv --log-file gpurun_out/q16/l_c2.csv python tools/profile_build.py c2 1 > /dev/null 2>&1; python tools/launches.py gpurun_out/q16/l_c2.csv | tail -4
FMMB_TRACE=1 timeout 300 python tools/trace_build.py c2 > gpurun_out/q16/trace_c2.log 2>&1; tail -25 gpurun_out/q16/trace_c2.log
timeout 1200 python -m pytest tests/test_gpu_build_parity.py tests/test_gpu_northstar.py tests/test_gpu_distributed.py -q -x 2>&1 | tail -2
