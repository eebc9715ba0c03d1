for v in off on off on; do
  if [ $v = on ]; then export FMMB_SCATTER_BMP=1; else unset FMMB_SCATTER_BMP; fi
  timeout 600 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_sbmp_$v.log 2>&1
  tail -1 gpurun_out/ab_sbmp_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['phases_ms'].items()})"
done
