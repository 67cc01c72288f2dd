set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_double.py tests/test_gpu_qr.py tests/test_gpu_backsub.py tests/test_gpu_gemm.py tests/test_gpu_invariants.py tests/test_gpu_arith.py tests/test_gpu_batched.py -x -q -k "d]" or "d-" 2>&1 | tail -15 > gpurun_out/gpu_tests_d.txt
timeout 900 python -m pytest tests/test_gpu_double.py tests/test_gpu_qr.py tests/test_gpu_backsub.py tests/test_gpu_gemm.py tests/test_gpu_invariants.py tests/test_gpu_arith.py tests/test_gpu_batched.py -x -q 2>&1 | tail -15 > gpurun_out/gpu_tests_d.txt
tail -3 gpurun_out/gpu_tests_d.txt
timeout 300 python tools/time_bs.py > gpurun_out/time_bs.txt 2>&1; cat gpurun_out/time_bs.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bs_launches.csv python tools/time_bs.py > /dev/null 2>&1; wc -l gpurun_out/bs_launches.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bs_update_kernel -s 2 -c 1 -o gpurun_out/bsupd -f python tools/time_bs.py > gpurun_out/ncu_bs.log 2>&1; tail -2 gpurun_out/ncu_bs.log
