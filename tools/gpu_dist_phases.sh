mkdir -p gpurun_out
for P in 1 2; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29611 tools/dist_phases.py ${WL:-c2} 5 2>&1 | grep '^{' 
done
