# A/B session: parity subset on the current build, then the c2/c3/c4 device
# builds under the scheduling / writer knobs (bench.py, CUDA events)
set -x
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests/test_gpu_northstar.py tests/test_gpu_build_parity.py tests/test_gpu_golden.py tests/test_gpu_threads.py -q -x 2>&1 | tail -6 > gpurun_out/ab/pytest.log
B="python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-nf"
for w in c2 c3 c4 c1; do
  timeout 300 $B --workload $w > gpurun_out/ab/$w.base.log 2>&1
done
FMMB_LW=0 timeout 300 $B --workload c2 > gpurun_out/ab/c2.lw0.log 2>&1
FMMB_LW=0 timeout 300 $B --workload c3 > gpurun_out/ab/c3.lw0.log 2>&1
FMMB_LOCAL_AFTER=1 timeout 300 $B --workload c2 > gpurun_out/ab/c2.after.log 2>&1
FMMB_LC_PER_SM=2 timeout 300 $B --workload c2 > gpurun_out/ab/c2.lc2.log 2>&1
FMMB_NO_OVERLAP=1 timeout 300 $B --workload c2 > gpurun_out/ab/c2.serial.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ab/launches_c2.csv python tools/profile_build.py c2 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ab/launches_c3.csv python tools/profile_build.py c3 1 > /dev/null 2>&1
cat gpurun_out/ab/pytest.log
for f in gpurun_out/ab/*.log; do echo $f; python -c "
import json,sys
for l in open('$f'):
    if l.startswith('{'):
        d=json.loads(l); print(round(d['ms_per_step'],3), round(d['build_ms_per_step'],3), {k:round(v,3) for k,v in d['phases_ms'].items()})
"; done
