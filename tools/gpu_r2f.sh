set -x
mkdir -p gpurun_out
timeout 600 python tools/time_bs.py > gpurun_out/time_bs.txt 2>&1; cat gpurun_out/time_bs.txt
MDLS_PDL=0 timeout 600 python tools/time_bs.py > gpurun_out/time_bs_nopdl.txt 2>&1; cat gpurun_out/time_bs_nopdl.txt
timeout 900 python -m pytest tests/test_gpu_backsub.py tests/test_gpu_double.py tests/test_gpu_qr.py tests/test_gpu_complex.py -x -q 2>&1 | tail -15 > gpurun_out/gpu_tests_f.txt
tail -3 gpurun_out/gpu_tests_f.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bs_launches3.csv python tools/time_bs.py > /dev/null 2>&1; wc -l gpurun_out/bs_launches3.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bs_update_kernel -s 2 -c 1 -o gpurun_out/bsupd3 -f python tools/time_bs.py > gpurun_out/ncu_bs.log 2>&1; tail -2 gpurun_out/ncu_bs.log
