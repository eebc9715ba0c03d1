# round 2, first GPU pass: new parity (north-star hashes, deep levels,
# threads), the full GPU suite, the official bench line (c2 with the
# reference on identical arrays), and the reference arm
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_northstar.py tests/test_gpu_threads.py -q -k "not nothing" -x 2>&1 | tail -15 > gpurun_out/pytest_new.log
timeout 600 python -m pytest tests/test_gpu_build_parity.py -q -k deep 2>&1 | tail -15 >> gpurun_out/pytest_new.log
timeout 600 python bench.py > gpurun_out/bench_official.log 2>&1
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_all.log
tail -5 gpurun_out/pytest_new.log
tail -3 gpurun_out/pytest_all.log
tail -1 gpurun_out/bench_official.log | cut -c1-600
tail -1 gpurun_out/bench_ref.log | cut -c1-400
