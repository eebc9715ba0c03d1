# A/B: near-dense list windows (default) vs none (FMMB_DENSE_ROWS=2)
D=gpurun_out/${Q:-q30}
mkdir -p $D
B="python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-nf --workload"
run() { tag=$1; shift; for w in c2 c3 c4; do env "$@" timeout 300 $B $w > $D/${tag}_$w.log 2>&1; python -c "
import json
d=json.loads(open('$D/${tag}_$w.log').read().strip().splitlines()[-1]); print('$tag $w', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})"; done; }
run near X=1
run nonear FMMB_DENSE_ROWS=2
run near X=1
run nonear FMMB_DENSE_ROWS=2
for w in c2 c4; do timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_lists_write" --csv --log-file $D/l_$w.csv python tools/profile_build.py $w 1 > /dev/null 2>&1; python tools/launches.py $D/l_$w.csv | tail -3 | head -1; done
timeout 900 python -m pytest tests/test_gpu_northstar.py tests/test_gpu_build_parity.py -q -x 2>&1 | tail -2
