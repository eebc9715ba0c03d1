set -x
mkdir -p gpurun_out/q10
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_lists_write" --csv --log-file gpurun_out/q10/l_c2.csv python tools/profile_build.py c2 2 > /dev/null 2>&1
python3 - gpurun_out/q10/l_c2.csv <<'PY'
import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
i=[k for k,r in enumerate(rows) if r and r[0]=="ID"][0]; h=rows[i]
mi,vi,idi=(h.index(x) for x in ("Metric Name","Metric Value","ID"))
d={}
for r in rows[i+1:]:
    d.setdefault(r[idi],{})[r[mi]]=r[vi]
for it in list(d.values())[-1:]: print(it)
PY
timeout 900 python -m pytest tests/test_gpu_build_parity.py tests/test_gpu_northstar.py tests/test_gpu_distributed.py -q -x 2>&1 | tail -2
B="python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-nf --workload"
for w in c2 c4; do timeout 300 $B $w > gpurun_out/q10/$w.log 2>&1; python -c "
import json
d=json.loads(open('gpurun_out/q10/$w.log').read().strip().splitlines()[-1]); print('$w', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})"; done
