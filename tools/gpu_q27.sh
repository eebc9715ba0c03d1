D=gpurun_out/${Q:-q27}
mkdir -p $D
B="python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-nf --workload"
for w in c2 c3 c4 c2 c3; do timeout 300 $B $w > $D/$w.log 2>&1; python -c "
import json
d=json.loads(open('$D/$w.log').read().strip().splitlines()[-1]); print('$w', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})"; done
for w in c2 c3; do timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_bkt_local" --csv --log-file $D/l_$w.csv python tools/profile_build.py $w 1 > /dev/null 2>&1; python tools/launches.py $D/l_$w.csv | tail -3 | head -1; done
timeout 900 python -m pytest tests/test_gpu_northstar.py tests/test_gpu_build_parity.py -q -x 2>&1 | tail -2
