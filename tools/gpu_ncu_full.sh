# one --set full capture per named kernel (first launch after one warm build)
set -x
for k in "$@"; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 1 -c 1 \
    -o gpurun_out/full_$k python tools/profile_build.py ${WL:-c2} 2 > gpurun_out/ncu_full_$k.log 2>&1
done
ls -la gpurun_out
