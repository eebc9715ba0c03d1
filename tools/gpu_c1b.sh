set -x
mkdir -p gpurun_out/c1b
timeout 1200 python -m pytest tests/test_gpu_northstar.py tests/test_gpu_build_parity.py tests/test_gpu_distributed.py tests/test_gpu_plugin.py tests/test_gpu_threads.py tests/test_gpu_container.py -q -x 2>&1 | tail -3 > gpurun_out/c1b/pytest.log
timeout 300 python tools/c1_latency.py c1 > gpurun_out/c1b/lat.log 2>&1
timeout 300 python bench.py --steps 50 --warmup 10 --no-cpu --no-e2e --no-nf --workload c1 > gpurun_out/c1b/c1.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-nf --workload c1 > gpurun_out/c1b/c1_10.log 2>&1
cat gpurun_out/c1b/pytest.log; head -3 gpurun_out/c1b/lat.log
for f in gpurun_out/c1b/c1*.log; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})"; done
