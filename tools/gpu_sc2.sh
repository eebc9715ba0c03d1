set -x
mkdir -p gpurun_out/sc2
for lib in paper_1301_1704_b200/libfmmb200.so build/lib_s236.so build/lib_s337.so build/lib_s427.so; do
  t=$(basename $lib .so)
  FMMB_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_bkt_scatter" --csv --log-file gpurun_out/sc2/l_$t.csv python tools/profile_build.py c2 2 > /dev/null 2>&1
  echo $t; python tools/launches.py gpurun_out/sc2/l_$t.csv | tail -4
  FMMB_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-nf --workload c2 > gpurun_out/sc2/b_$t.log 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/sc2/b_$t.log').read().strip().splitlines()[-1]); print('$t', round(d['ms_per_step'],3))"
done
