# round validation: smoke, full GPU suite, official bench line, reference arm, c1-c4 lines
set -x
mkdir -p gpurun_out/val
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/val/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/val/pytest_all.log
timeout 900 python bench.py > gpurun_out/val/bench_official.log 2>&1
B="python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-nf"
for w in c1 c3 c4; do timeout 300 $B --workload $w > gpurun_out/val/$w.log 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/val/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-nf > /dev/null 2>&1
cat gpurun_out/val/smoke.log gpurun_out/val/pytest_all.log
tail -1 gpurun_out/val/bench_official.log | cut -c1-400
for f in gpurun_out/val/c?.log; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})"; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/val/bench_ref.log 2>&1
tail -1 gpurun_out/val/bench_ref.log | cut -c1-600
timeout 300 python tools/c1_latency.py c1 > gpurun_out/val/c1_latency.log 2>&1; head -2 gpurun_out/val/c1_latency.log
timeout 600 python tools/c4_trajectory.py > gpurun_out/val/c4_trajectory.log 2>&1; tail -1 gpurun_out/val/c4_trajectory.log | cut -c1-400
for w in c2 c3 c4; do FMMB_TRACE=1 timeout 300 python tools/trace_build.py $w > gpurun_out/val/trace_$w.log 2>&1; done
for w in c3 c4; do timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/val/launches_$w.csv python tools/profile_build.py $w 1 > /dev/null 2>&1; done
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533"
timeout 900 $R bench.py --partitioned --workload c2 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/val/part_c2.log 2>&1; tail -1 gpurun_out/val/part_c2.log | cut -c1-300
timeout 1200 $R bench.py --partitioned --workload c5 --steps 3 --warmup 3 > gpurun_out/val/part_c5.log 2>&1; tail -1 gpurun_out/val/part_c5.log | cut -c1-300
