# checkpoint: full GPU suite, c1 latency, official bench, reference arm, c4 trajectory
set -x
mkdir -p gpurun_out/r2f
timeout 300 python tools/c1_latency.py c1 > gpurun_out/r2f/c1_latency.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/r2f/pytest_all.log
timeout 900 python bench.py > gpurun_out/r2f/bench_official.log 2>&1
B="python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-nf"
for w in c3 c4 c1; do timeout 300 $B --workload $w > gpurun_out/r2f/$w.log 2>&1; done
timeout 900 python tools/c4_trajectory.py > gpurun_out/r2f/c4_trajectory.log 2>&1
cat gpurun_out/r2f/pytest_all.log gpurun_out/r2f/c1_latency.log | head -40
tail -1 gpurun_out/r2f/bench_official.log | cut -c1-1500
for f in gpurun_out/r2f/c?.log; do echo $f; python -c "
import json,sys
for l in open('$f'):
    if l.startswith('{'):
        d=json.loads(l); print(round(d['ms_per_step'],3), round(d['build_ms_per_step'],3), {k:round(v,3) for k,v in d['phases_ms'].items()})
"; done
tail -1 gpurun_out/r2f/c4_trajectory.log | cut -c1-900
