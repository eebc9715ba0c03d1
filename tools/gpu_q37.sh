D=gpurun_out/${Q:-q37}
mkdir -p $D
timeout 600 python -m pytest tests/test_gpu_workload.py -q -x 2>&1 | tail -2
B="python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-nf --workload"
for w in c4 c4; do timeout 300 $B $w > $D/$w.log 2>&1; python -c "
import json
d=json.loads(open('$D/$w.log').read().strip().splitlines()[-1]); print('$w', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})"; done
timeout 600 python tools/c4_trajectory.py > $D/traj.log 2>&1; tail -1 $D/traj.log | cut -c1-420
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_perturb" --csv --log-file $D/l.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-nf --workload c4 > /dev/null 2>&1; python tools/launches.py $D/l.csv | head -4
