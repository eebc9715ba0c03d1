set -x
mkdir -p gpurun_out/d2
timeout 900 python -m pytest tests/test_gpu_distributed.py -q -x 2>&1 | tail -3 > gpurun_out/d2/pytest.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533"
timeout 900 $R bench.py --partitioned --workload c2 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/d2/part_c2.log 2>&1
timeout 900 $R bench.py --partitioned --workload c5 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/d2/part_c5.log 2>&1
cat gpurun_out/d2/pytest.log
for f in gpurun_out/d2/part_*.log; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], {k: round(v,3) for k,v in d['phases_ms'].items()})"; done
