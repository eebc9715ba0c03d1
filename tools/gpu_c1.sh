set -x
mkdir -p gpurun_out/c1
FMMB_TRACE=1 timeout 300 python tools/trace_build.py c1 50 > gpurun_out/c1/trace.log 2>&1
timeout 300 python tools/c1_latency.py c1 > gpurun_out/c1/lat.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c1/l.csv python tools/profile_build.py c1 1 > /dev/null 2>&1
cat gpurun_out/c1/trace.log; head -3 gpurun_out/c1/lat.log; python tools/launches.py gpurun_out/c1/l.csv | tail -16
