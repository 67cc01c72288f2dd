set -x
mkdir -p gpurun_out
timeout 600 python tools/time_bs.py > gpurun_out/time_bs.txt 2>&1; cat gpurun_out/time_bs.txt
timeout 900 python -m pytest tests/test_gpu_backsub.py tests/test_gpu_qr.py tests/test_gpu_determinism.py tests/test_gpu_variants.py -x -q 2>&1 | tail -15 > gpurun_out/gpu_tests_g.txt
tail -3 gpurun_out/gpu_tests_g.txt
timeout 900 python bench.py --no-cpu --steps 10 > gpurun_out/bench_g.json 2> gpurun_out/bench_g.err; tail -c 3000 gpurun_out/bench_g.json; tail -3 gpurun_out/bench_g.err
MDLS_PDL=0 timeout 600 python bench.py --no-cpu --no-extra --steps 10 > gpurun_out/bench_g_nopdl.json 2>&1; head -c 400 gpurun_out/bench_g_nopdl.json
