# Final round measurement: GPU tests, bench (with the oracle cpu baseline), reference arm, launch list
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/gpu_tests_final5.txt; tail -2 gpurun_out/gpu_tests_final5.txt
timeout 1200 python bench.py > gpurun_out/bench_final5.json 2> gpurun_out/bench_final5.err; tail -c 3000 gpurun_out/bench_final5.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref5.json 2>&1; tail -c 600 gpurun_out/bench_ref5.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_dd_final5.csv python bench.py --steps 1 --warmup 1 --no-extra --no-cpu --no-graph > /dev/null 2>&1; wc -l gpurun_out/launches_dd_final5.csv
