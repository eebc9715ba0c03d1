set -x
mkdir -p gpurun_out/fin1
timeout 900 python tools/c4_trajectory.py > gpurun_out/fin1/c4_trajectory.log 2>&1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533"
timeout 1500 $R bench.py --partitioned --workload c5 --steps 3 --warmup 3 > gpurun_out/fin1/part_c5.log 2>&1
timeout 900 $R bench.py --partitioned --workload c2 --steps 5 --warmup 3 --no-cpu > gpurun_out/fin1/part_c2.log 2>&1
for w in c2 c3 c4; do FMMB_TRACE=1 timeout 300 python tools/trace_build.py $w > gpurun_out/fin1/trace_$w.log 2>&1; done
tail -1 gpurun_out/fin1/c4_trajectory.log | cut -c1-700
for f in gpurun_out/fin1/part_*.log; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],3), d.get('e2e'), {k: round(v,3) for k,v in d['phases_ms'].items()})"; done
cat gpurun_out/fin1/trace_c2.log
