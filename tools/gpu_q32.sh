D=gpurun_out/${Q:-q32}
mkdir -p $D
B="python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-nf --workload"
run() { tag=$1; shift; for w in c1 c2 c3 c4; do env "$@" timeout 300 $B $w > $D/${tag}_$w.log 2>&1; python -c "
import json
d=json.loads(open('$D/${tag}_$w.log').read().strip().splitlines()[-1]); print('$tag $w', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})"; done; }
for rep in 1 2; do
run lw32 X=1
run lw16 FMMB_LW_PER_SM=16
run lw256 FMMB_LW_PER_SM=256
done
