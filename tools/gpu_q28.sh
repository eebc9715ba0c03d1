# ncu --set full of the list writer (c2, c4) and the persistent list count (c3)
D=gpurun_out/q28
mkdir -p $D
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_lists_write" -s 1 -c 1 -o $D/lw_c2 python tools/profile_build.py c2 2 > $D/lw_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_lists_write" -s 1 -c 1 -o $D/lw_c4 python tools/profile_build.py c4 2 > $D/lw_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_lists_cscan" -s 1 -c 1 -o $D/cs_c3 python tools/profile_build.py c3 2 > $D/cs_c3.log 2>&1
ls -la $D
