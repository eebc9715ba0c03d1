# GPU session: parity first, then bench, then the ncu launch list (+ optional full captures).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python tools/profile_build.py ${WL:-c2} 3 > gpurun_out/profile_build.log 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_build.py ${WL:-c2} 1 > gpurun_out/ncu_run.log 2>&1
for k in $FULL; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 1 -c 1 \
    -o gpurun_out/full_$k python tools/profile_build.py ${WL:-c2} 2 > gpurun_out/ncu_full_$k.log 2>&1
done
tail -5 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/bench.log; cat gpurun_out/profile_build.log
