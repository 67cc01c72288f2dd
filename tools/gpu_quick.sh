# quick GPU check: QR/BS parity (with config 2/3 margins) and a short bench
timeout 1200 python -m pytest tests/test_gpu_qr.py tests/test_gpu_backsub.py tests/test_gpu_arith.py tests/test_gpu_sharded.py -x -q -s 2>&1 | grep -v "^$" | tail -25 > gpurun_out/quick_tests.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/quick_bench.json 2> gpurun_out/quick_bench.err
cat gpurun_out/quick_tests.txt; cat gpurun_out/quick_bench.json; tail -5 gpurun_out/quick_bench.err
