mkdir -p gpurun_out
for v in 0 3 1; do MDLS_BSU=$v timeout 600 python tools/time_bs.py 2>&1 | tail -1; done
MDLS_BSU=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:bs_update_kernel -s 2 -c 1 -o gpurun_out/bsupd4 -f python tools/time_bs.py > gpurun_out/ncu_bs.log 2>&1; tail -1 gpurun_out/ncu_bs.log
MDLS_BSU=3 timeout 600 python -m pytest tests/test_gpu_backsub.py -q -x 2>&1 | tail -2
