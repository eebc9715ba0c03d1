D=gpurun_out/${Q:-q22}
mkdir -p $D
B="python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-nf --workload"
for w in c1 c2 c3 c4; do timeout 300 $B $w > $D/$w.log 2>&1; python -c "
import json
d=json.loads(open('$D/$w.log').read().strip().splitlines()[-1]); print('$w', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})"; done
for w in c2 c3; do timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_lists_cscan" --csv --log-file $D/l_$w.csv python tools/profile_build.py $w 1 > /dev/null 2>&1; python tools/launches.py $D/l_$w.csv | tail -3 | head -1; done
FMMB_TRACE=1 timeout 300 python tools/trace_build.py c3 > $D/trace_c3.log 2>&1; tail -13 $D/trace_c3.log
timeout 1200 python -m pytest tests/test_gpu_build_parity.py tests/test_gpu_northstar.py tests/test_gpu_distributed.py -q -x 2>&1 | tail -2
