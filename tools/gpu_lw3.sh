set -x
mkdir -p gpurun_out/lw3
for v in base out; do
  E="FMMB_X=1"; [ $v = out ] && E="FMMB_LW_OUT=1"
  for w in c2 c3; do
    env $E timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex_op_write.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_lists_write" --csv --log-file gpurun_out/lw3/l_${v}_$w.csv python tools/profile_build.py $w 2 > /dev/null 2>&1
  done
  env $E timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-nf --workload c2 > gpurun_out/lw3/b_${v}_c2.log 2>&1
  env $E timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-nf --workload c4 > gpurun_out/lw3/b_${v}_c4.log 2>&1
done
FMMB_LW_OUT=1 timeout 900 python -m pytest tests/test_gpu_northstar.py tests/test_gpu_build_parity.py -q -x 2>&1 | tail -3 > gpurun_out/lw3/pytest.log
cat gpurun_out/lw3/pytest.log
for f in gpurun_out/lw3/l_*.csv; do echo $f; python3 - $f <<'PY'
import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
i=[k for k,r in enumerate(rows) if r and r[0]=="ID"][0]; h=rows[i]
ki,mi,vi,idi=(h.index(x) for x in ("Kernel Name","Metric Name","Metric Value","ID"))
d={}
for r in rows[i+1:]:
    d.setdefault(r[idi],{})[r[mi]]=r[vi]
for it in list(d.values())[-1:]: print(it)
PY
done
for f in gpurun_out/lw3/b_*.log; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})"; done
