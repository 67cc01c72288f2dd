set -x
mkdir -p gpurun_out
for v in 0 1 2; do MDLS_BSU=$v timeout 600 python tools/time_bs.py 2>&1 | tail -1 > gpurun_out/time_bs_v$v.txt; cat gpurun_out/time_bs_v$v.txt; done
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/gpu_tests_h.txt
tail -3 gpurun_out/gpu_tests_h.txt
