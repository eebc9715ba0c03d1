# A/B: early occupancy (histogram pass sets the bits, sort beside the lists)
# vs the r01 structure, scatter grid caps; parity subset first
set -x
mkdir -p gpurun_out/ab2
timeout 900 python -m pytest tests/test_gpu_northstar.py tests/test_gpu_build_parity.py tests/test_gpu_golden.py tests/test_gpu_plugin.py -q -x 2>&1 | tail -4 > gpurun_out/ab2/pytest.log
B="python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-nf"
for w in c2 c3 c4 c1; do timeout 300 $B --workload $w > gpurun_out/ab2/$w.early.log 2>&1; done
for w in c2 c3 c4; do FMMB_LATE_OCC=1 timeout 300 $B --workload $w > gpurun_out/ab2/$w.late.log 2>&1; done
for k in 120 100 74; do FMMB_SCATTER_CTAS=$k timeout 300 $B --workload c2 > gpurun_out/ab2/c2.sc$k.log 2>&1; done
FMMB_SCATTER_CTAS=100 timeout 300 $B --workload c3 > gpurun_out/ab2/c3.sc100.log 2>&1
timeout 600 nsys --version > /dev/null 2>&1 || true
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ab2/launches_c2.csv python tools/profile_build.py c2 1 > /dev/null 2>&1
cat gpurun_out/ab2/pytest.log
for f in gpurun_out/ab2/*.log; do echo $f; python -c "
import json,sys
for l in open('$f'):
    if l.startswith('{'):
        d=json.loads(l); print(round(d['ms_per_step'],3), round(d['build_ms_per_step'],3), {k:round(v,3) for k,v in d['phases_ms'].items()})
"; done
