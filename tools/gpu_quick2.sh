# parity subset + c2/c3/c4 device lines + kernel launch list at c2
set -x
mkdir -p gpurun_out/q2
timeout 900 python -m pytest tests/test_gpu_northstar.py tests/test_gpu_build_parity.py tests/test_gpu_golden.py tests/test_gpu_distributed.py -q -x 2>&1 | tail -3 > gpurun_out/q2/pytest.log
B="python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-nf"
for w in c2 c3 c4; do timeout 300 $B --workload $w > gpurun_out/q2/$w.log 2>&1; done
for w in c2; do FMMB_OCC_RED=1 timeout 300 $B --workload $w > gpurun_out/q2/${w}_occred.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_lists_write|k_bkt_local|k_bkt_scatter|k_lists_cscan|k_bkt_hist" --csv --log-file gpurun_out/q2/l_c2.csv python tools/profile_build.py c2 1 > /dev/null 2>&1
cat gpurun_out/q2/pytest.log
python tools/launches.py gpurun_out/q2/l_c2.csv
for f in gpurun_out/q2/c*.log; do echo $f; python -c "
import json,sys
for l in open('$f'):
    if l.startswith('{'):
        d=json.loads(l); print(round(d['ms_per_step'],3), round(d['build_ms_per_step'],3), {k:round(v,3) for k,v in d['phases_ms'].items()}, round(d['roofline']['frac'],3))
"; done
