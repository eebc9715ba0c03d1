# parity subset + c2/c3 device bench
set -x
timeout 1200 python -m pytest tests -m gpu -q -x -k "build_all or bucket or overflow or crowded or distributed or sort_points or golden" 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
for w in ${WLS:-c2 c3}; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$w.log 2>&1
done
tail -3 gpurun_out/pytest_gpu.log
for w in ${WLS:-c2 c3}; do tail -1 gpurun_out/bench_$w.log | cut -c1-200; done
