mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_nearfield.py -q -x 2>&1 | tail -2
for rg in 8 16 32; do echo rg=$rg; FMMB_NF_RG=$rg timeout 300 python tools/bench_nearfield.py c2 5 | cut -c1-160; FMMB_NF_RG=$rg timeout 300 python tools/bench_nearfield.py c3 5 | cut -c1-160; done
