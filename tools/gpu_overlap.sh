mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for v in on off on off; do
  if [ $v = off ]; then export FMMB_NO_OVERLAP=1; else unset FMMB_NO_OVERLAP; fi
  for w in c2 c3; do
    timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ov_${w}_$v.log 2>&1
    tail -1 gpurun_out/ov_${w}_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w $v', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['phases_ms'].items()})"
  done
done
unset FMMB_NO_OVERLAP
timeout 600 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-220
