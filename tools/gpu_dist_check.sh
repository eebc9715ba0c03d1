# 2 ranks of the partitioned bench on ONE GPU over gloo (host-staged): exercises
# run_partitioned end to end where NCCL cannot put two ranks on one device.
set -x
FMMB_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 2 --warmup 3 --workload c1 \
  > gpurun_out/dist_bench.log 2>&1
tail -3 gpurun_out/dist_bench.log
