mkdir -p gpurun_out
timeout 600 python tools/time_batched.py 32 1 2 4 6 8 2>&1 | tail -6
timeout 900 python -m pytest tests/test_gpu_batched.py -q -x 2>&1 | tail -3
tail -3 /dev/null
