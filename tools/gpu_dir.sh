set -x
mkdir -p gpurun_out/dir
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_pyramid|k_rank|k_lists_plan" --csv --log-file gpurun_out/dir/l_c2.csv python tools/profile_build.py c2 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/dir/l_c2.csv | tail -12
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_rank" -s 1 -c 1 -o gpurun_out/dir/rank python tools/profile_build.py c2 2 > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_build_parity.py tests/test_gpu_northstar.py -q -x 2>&1 | tail -2
