# full GPU test suite + device-resident bench of every single-GPU workload
set -x
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_all.log
for w in c1 c2 c3 c4; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$w.log 2>&1
done
tail -3 gpurun_out/pytest_all.log
for w in c1 c2 c3 c4; do tail -1 gpurun_out/bench_$w.log | cut -c1-260; done
