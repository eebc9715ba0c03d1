# partitioned path at P=1: c2 shard and the c5 shard (2^27 + 2^27, L=8)
set -x
mkdir -p gpurun_out/r2g
timeout 600 python -m pytest tests/test_gpu_workload.py tests/test_gpu_distributed.py -q -x 2>&1 | tail -3 > gpurun_out/r2g/pytest.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533"
timeout 900 $R bench.py --partitioned --workload c2 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2g/part_c2.log 2>&1
timeout 1500 $R bench.py --partitioned --workload c5 --steps 3 --warmup 3 > gpurun_out/r2g/part_c5.log 2>&1
timeout 300 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu --no-e2e --no-nf > gpurun_out/r2g/c4.log 2>&1
cat gpurun_out/r2g/pytest.log
tail -2 gpurun_out/r2g/part_c2.log | cut -c1-2500
tail -3 gpurun_out/r2g/part_c5.log | cut -c1-3000
tail -1 gpurun_out/r2g/c4.log | cut -c1-600
