set -x
mkdir -p gpurun_out/sc
for v in main noocc; do
  lib=paper_1301_1704_b200/libfmmb200.so; [ $v = noocc ] && lib=build/lib_noocc.so
  FMMB_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_bkt_scatter|k_bkt_local" --csv --log-file gpurun_out/sc/l_$v.csv python tools/profile_build.py c2 2 > /dev/null 2>&1
  echo $v; python tools/launches.py gpurun_out/sc/l_$v.csv | tail -5
done
FMMB_SORT_PATH=bucket_hist timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_bkt_scatter" --csv --log-file gpurun_out/sc/l_hist.csv python tools/profile_build.py c2 2 > /dev/null 2>&1
echo hist; python tools/launches.py gpurun_out/sc/l_hist.csv | tail -4
