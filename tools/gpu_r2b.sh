# timeline (trace events) of the overlapped build at c2/c3/c4 + scatter caps,
# plugin tests, and --set full captures of the kernels on the critical path
set -x
mkdir -p gpurun_out/r2b
timeout 600 python -m pytest tests/test_gpu_plugin.py -q -x 2>&1 | tail -3 > gpurun_out/r2b/pytest.log
for w in c2 c3 c4; do FMMB_TRACE=1 timeout 300 python tools/trace_build.py $w > gpurun_out/r2b/trace_$w.log 2>&1; done
FMMB_TRACE=1 FMMB_LATE_OCC=1 timeout 300 python tools/trace_build.py c2 > gpurun_out/r2b/trace_c2_late.log 2>&1
for k in 100 74; do FMMB_TRACE=1 FMMB_SCATTER_CTAS=$k timeout 300 python tools/trace_build.py c2 > gpurun_out/r2b/trace_c2_sc$k.log 2>&1; done
for k in k_lists_write k_bkt_local k_bkt_scatter k_bkt_hist; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 1 -c 1 \
    -o gpurun_out/r2b/full_$k python tools/profile_build.py c2 2 > gpurun_out/r2b/ncu_full_$k.log 2>&1
done
cat gpurun_out/r2b/pytest.log gpurun_out/r2b/trace_*.log
