# near-field parity + timing; scatter A/B (speculative vs histogram regions)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nearfield.py -q -x 2>&1 | tail -15 > gpurun_out/pytest_nf.log
for w in c1 c2 c3; do timeout 300 python tools/bench_nearfield.py $w 5 >> gpurun_out/nf_bench.log 2>&1; done
for sp in auto bucket_hist; do
  timeout 600 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu --no-e2e --sort-path $sp > gpurun_out/ab_$sp.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_nf.csv python tools/bench_nearfield.py c2 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_near_field -s 1 -c 1 -o gpurun_out/full_k_near_field python tools/bench_nearfield.py c2 1 > /dev/null 2>&1
FMMB_SORT_PATH=bucket_hist timeout 900 ncu --set full --clock-control none -k regex:k_bkt_scatter -s 1 -c 1 -o gpurun_out/full_scatter_hist python tools/profile_build.py c2 1 > /dev/null 2>&1
FMMB_SORT_PATH=auto timeout 900 ncu --set full --clock-control none -k regex:k_bkt_scatter -s 1 -c 1 -o gpurun_out/full_scatter_spec python tools/profile_build.py c2 1 > /dev/null 2>&1
cat gpurun_out/pytest_nf.log | tail -3
cat gpurun_out/nf_bench.log
for sp in auto bucket_hist; do tail -1 gpurun_out/ab_$sp.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$sp', d['ms_per_step'], d['phases_ms'])"; done
