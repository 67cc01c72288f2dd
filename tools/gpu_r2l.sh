mkdir -p gpurun_out
timeout 600 python tools/time_bs.py 2>&1 | tail -1
MDLS_BS_BULK=0 timeout 600 python tools/time_bs.py 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_backsub.py tests/test_gpu_qr.py -q -x 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bs_update_kernel -s 2 -c 1 -o gpurun_out/bsupd5 -f python tools/time_bs.py > gpurun_out/ncu_bs.log 2>&1; tail -1 gpurun_out/ncu_bs.log
