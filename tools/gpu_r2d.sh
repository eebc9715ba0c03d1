set -x
mkdir -p gpurun_out/r2d
T="timeout 300 python tools/trace_build.py"
for w in c2 c4 c3; do
  FMMB_TRACE=1 FMMB_SIDE_PRIO=1 $T $w > gpurun_out/r2d/A_$w.log 2>&1
  FMMB_TRACE=1 FMMB_SIDE_PRIO=1 FMMB_LC_PER_SM=2 $T $w > gpurun_out/r2d/B_$w.log 2>&1
  FMMB_TRACE=1 FMMB_SIDE_PRIO=1 FMMB_REC_IDX=1 $T $w > gpurun_out/r2d/C_$w.log 2>&1
  FMMB_TRACE=1 FMMB_SIDE_PRIO=1 FMMB_LATE_OCC=1 $T $w > gpurun_out/r2d/D_$w.log 2>&1
  FMMB_TRACE=1 FMMB_SIDE_PRIO=1 FMMB_SCATTER_EARLY=1 $T $w > gpurun_out/r2d/E_$w.log 2>&1
done
for f in gpurun_out/r2d/*.log; do echo "== $f"; tail -12 $f | sort -n | tail -1; done
cat gpurun_out/r2d/A_c2.log gpurun_out/r2d/B_c2.log
