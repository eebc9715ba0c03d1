# list-writer A/B: kernel times (ncu launch list) at c2/c3 + list parity subset
# usage: bash tools/gpu_lw.sh [alt-lib ...]
set -x
mkdir -p gpurun_out/lw
run() {  # tag, lib
  for w in c2 c3; do
    FMMB_LIB=$2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_lists_write|k_bkt_local|k_bkt_scatter|k_lists_cscan" --csv --log-file gpurun_out/lw/l_$1_$w.csv python tools/profile_build.py $w 2 > /dev/null 2>&1
    python tools/launches.py gpurun_out/lw/l_$1_$w.csv | tail -6 > gpurun_out/lw/l_$1_$w.md
  done
}
run main paper_1301_1704_b200/libfmmb200.so
i=0; for lib in "$@"; do i=$((i+1)); run alt$i $lib; done
timeout 900 python -m pytest tests/test_gpu_northstar.py tests/test_gpu_build_parity.py -q -x 2>&1 | tail -3 > gpurun_out/lw/pytest.log
cat gpurun_out/lw/pytest.log; for f in gpurun_out/lw/l_*.md; do echo "== $f"; cat $f; done
