# A/B: list-write grid (CTAs per SM) and local-pass CTAs per SM, c2/c4 in-step
D=gpurun_out/${Q:-q31}
mkdir -p $D
B="python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-nf --workload"
run() { tag=$1; shift; for w in c2 c4; do env "$@" timeout 300 $B $w > $D/${tag}_$w.log 2>&1; python -c "
import json
d=json.loads(open('$D/${tag}_$w.log').read().strip().splitlines()[-1]); print('$tag $w', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})"; done; }
for rep in 1 2; do
run lw16 X=1
run lw4 FMMB_LW_PER_SM=4
run lw8 FMMB_LW_PER_SM=8
run lw32 FMMB_LW_PER_SM=32
run lw64 FMMB_LW_PER_SM=64
done
