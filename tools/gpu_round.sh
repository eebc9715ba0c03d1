# round artefacts: full GPU suite, official bench line (c2), all workloads,
# ncu launch list of one c2 build, one --set full capture of the top kernels,
# near-field capture, partitioned-step phases
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_all.log
timeout 900 python bench.py > gpurun_out/bench_official.log 2>&1
for w in c1 c3 c4; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$w.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/profile_build.py c2 1 > /dev/null 2>&1
for k in k_lists_write k_bkt_scatter k_bkt_local; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/full_$k python tools/profile_build.py c2 2 > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_near_field -s 1 -c 1 -o gpurun_out/full_k_near_field python tools/bench_nearfield.py c2 1 > /dev/null 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29615 tools/dist_phases.py c2 5 2>&1 | grep '^{' > gpurun_out/dist_phases.log
tail -3 gpurun_out/pytest_all.log
tail -1 gpurun_out/bench_official.log
