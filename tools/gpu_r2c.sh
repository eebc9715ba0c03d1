# parity subset + timelines of the structure variants + bench lines
set -x
mkdir -p gpurun_out/r2c
timeout 900 python -m pytest tests/test_gpu_northstar.py tests/test_gpu_build_parity.py tests/test_gpu_golden.py tests/test_gpu_plugin.py tests/test_gpu_threads.py -q -x 2>&1 | tail -4 > gpurun_out/r2c/pytest.log
for w in c2 c3 c4; do
  FMMB_TRACE=1 timeout 300 python tools/trace_build.py $w > gpurun_out/r2c/trace_$w.log 2>&1
  FMMB_TRACE=1 FMMB_SCATTER_EARLY=1 timeout 300 python tools/trace_build.py $w > gpurun_out/r2c/trace_${w}_scearly.log 2>&1
  FMMB_TRACE=1 FMMB_REC_IDX=1 timeout 300 python tools/trace_build.py $w > gpurun_out/r2c/trace_${w}_recidx.log 2>&1
  FMMB_TRACE=1 FMMB_LATE_OCC=1 timeout 300 python tools/trace_build.py $w > gpurun_out/r2c/trace_${w}_late.log 2>&1
done
B="python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-nf"
for w in c2 c3 c4 c1; do timeout 300 $B --workload $w > gpurun_out/r2c/$w.log 2>&1; done
cat gpurun_out/r2c/pytest.log
for f in gpurun_out/r2c/trace_*.log; do echo "== $f"; tail -14 $f | sort -n | tail -3; done
for f in gpurun_out/r2c/c?.log; do echo $f; python -c "
import json,sys
for l in open('$f'):
    if l.startswith('{'):
        d=json.loads(l); print(round(d['ms_per_step'],3), round(d['build_ms_per_step'],3), {k:round(v,3) for k,v in d['phases_ms'].items()})
"; done
