# A/B: dense list writer (line-aligned runs vs rows) x local-pass CTAs per SM, in-step c2/c4
D=gpurun_out/${Q:-q20}
mkdir -p $D
B="python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-nf --workload"
run() { tag=$1; shift; for w in c2 c4; do env "$@" timeout 300 $B $w > $D/${tag}_$w.log 2>&1; python -c "
import json
d=json.loads(open('$D/${tag}_$w.log').read().strip().splitlines()[-1]); print('$tag $w', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})"; done; }
for rep in 1 2; do
run runs X=1
run rows FMMB_DENSE_ROWS=1
run runs_lc3 FMMB_LC_PER_SM=3
run rows_lc3 FMMB_DENSE_ROWS=1 FMMB_LC_PER_SM=3
run runs_lc1 FMMB_LC_PER_SM=1
done
