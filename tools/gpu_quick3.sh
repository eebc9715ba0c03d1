set -x
mkdir -p gpurun_out/q3
for w in c2 c4; do
  FMMB_TRACE=1 FMMB_EARLY_OCC=1 timeout 300 python tools/trace_build.py $w > gpurun_out/q3/early_$w.log 2>&1
  FMMB_TRACE=1 FMMB_EARLY_OCC=1 FMMB_SCATTER_EARLY=1 timeout 300 python tools/trace_build.py $w > gpurun_out/q3/early_sce_$w.log 2>&1
  FMMB_TRACE=1 timeout 300 python tools/trace_build.py $w > gpurun_out/q3/late_$w.log 2>&1
done
FMMB_EARLY_OCC=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/q3/l_c2_early.csv python tools/profile_build.py c2 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/q3/l_c2_early.csv | head -16
for f in gpurun_out/q3/*.log; do echo "== $f"; tail -12 $f | sort -n | tail -1; done
cat gpurun_out/q3/early_c2.log
