timeout 300 python tools/time_bs.py 2>&1 | tail -1
MDLS_BS_FLOW=0 timeout 300 python tools/time_bs.py 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_backsub.py tests/test_gpu_qr.py tests/test_gpu_determinism.py tests/test_gpu_double.py tests/test_gpu_plan.py -q -x 2>&1 | tail -2
