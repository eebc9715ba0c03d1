# A/B: list-count grid (persistent CTAs per SM) and scatter CTAs
D=gpurun_out/${Q:-q34}
mkdir -p $D
B="python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-nf --workload"
run() { tag=$1; shift; for w in c2 c3 c4; do env "$@" timeout 300 $B $w > $D/${tag}_$w.log 2>&1; python -c "
import json
d=json.loads(open('$D/${tag}_$w.log').read().strip().splitlines()[-1]); print('$tag $w', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})"; done; }
for rep in 1 2; do
run base X=1
run cs4 FMMB_CS_PER_SM=4
run cs16 FMMB_CS_PER_SM=16
run sc132 FMMB_SCATTER_CTAS=132
done
