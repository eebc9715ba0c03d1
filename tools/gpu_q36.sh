# bench timing: settle time after the clock sampler starts (c1 is host-latency bound)
D=gpurun_out/${Q:-q36}
mkdir -p $D
B="python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-nf --workload"
for rep in 1 2; do
for st in 0 0.5; do for w in c1 c2; do FMMB_BENCH_SETTLE_S=$st timeout 300 $B $w > $D/s${st}_$w.log 2>&1; python -c "
import json
d=json.loads(open('$D/s${st}_$w.log').read().strip().splitlines()[-1]); print('settle $st $w', round(d['ms_per_step'],4), d['clocks'])"; done; done
done
