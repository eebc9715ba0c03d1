set -x
mkdir -p gpurun_out/r2h
timeout 900 python -m pytest tests/test_gpu_northstar.py tests/test_gpu_build_parity.py tests/test_gpu_golden.py tests/test_gpu_distributed.py tests/test_gpu_nearfield.py -q -x 2>&1 | tail -3 > gpurun_out/r2h/pytest.log
B="python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-nf"
for w in c2 c3 c4 c1; do timeout 300 $B --workload $w > gpurun_out/r2h/$w.log 2>&1; done
for w in c2 c3 c4; do FMMB_TRACE=1 timeout 300 python tools/trace_build.py $w > gpurun_out/r2h/trace_$w.log 2>&1; done
for w in c3 c4; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2h/launches_$w.csv python tools/profile_build.py $w 1 > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bkt_scatter" -s 1 -c 1 -o gpurun_out/r2h/full_c3_scatter python tools/profile_build.py c3 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bkt_local" -s 1 -c 1 -o gpurun_out/r2h/full_c3_local python tools/profile_build.py c3 2 > /dev/null 2>&1
cat gpurun_out/r2h/pytest.log
for f in gpurun_out/r2h/c?.log; do echo $f; python -c "
import json,sys
for l in open('$f'):
    if l.startswith('{'):
        d=json.loads(l); print(round(d['ms_per_step'],3), round(d['build_ms_per_step'],3), {k:round(v,3) for k,v in d['phases_ms'].items()}, round(d['roofline']['frac'],3))
"; done
