# A/B at the final state: ordering / priority variants
D=gpurun_out/${Q:-q35}
mkdir -p $D
B="python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-nf --workload"
run() { tag=$1; shift; for w in c2 c4; do env "$@" timeout 300 $B $w > $D/${tag}_$w.log 2>&1; python -c "
import json
d=json.loads(open('$D/${tag}_$w.log').read().strip().splitlines()[-1]); print('$tag $w', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})"; done; }
for rep in 1 2; do
run base X=1
run lafter FMMB_LOCAL_AFTER=1
run prio FMMB_SIDE_PRIO=1
run early FMMB_EARLY_OCC=1
done
