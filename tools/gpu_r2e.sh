set -x
mkdir -p gpurun_out/r2e
timeout 900 python -m pytest tests/test_gpu_northstar.py tests/test_gpu_build_parity.py tests/test_gpu_golden.py tests/test_gpu_distributed.py -q -x 2>&1 | tail -4 > gpurun_out/r2e/pytest.log
T="timeout 300 python tools/trace_build.py"
for w in c2 c3 c4; do
  FMMB_TRACE=1 $T $w > gpurun_out/r2e/early_$w.log 2>&1
  FMMB_TRACE=1 FMMB_LATE_OCC=1 $T $w > gpurun_out/r2e/late_$w.log 2>&1
  FMMB_TRACE=1 FMMB_SCATTER_EARLY=1 $T $w > gpurun_out/r2e/scearly_$w.log 2>&1
  FMMB_TRACE=1 FMMB_LIB=build/lib_minb3.so $T $w > gpurun_out/r2e/minb3_$w.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2e/launches_c2.csv python tools/profile_build.py c2 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lists_write -s 1 -c 1 -o gpurun_out/r2e/full_lw python tools/profile_build.py c2 2 > /dev/null 2>&1
cat gpurun_out/r2e/pytest.log
for f in gpurun_out/r2e/*_c?.log; do echo "== $f"; tail -12 $f | sort -n | tail -1; done
python tools/launches.py gpurun_out/r2e/launches_c2.csv | head -16
