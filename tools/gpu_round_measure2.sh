# Second round measurement (after the dd tile change): GPU tests, bench, launch list, roofline GEMM capture
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/gpu_tests_final2.txt; tail -2 gpurun_out/gpu_tests_final2.txt
timeout 1200 python bench.py > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err; tail -c 3000 gpurun_out/bench_final2.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_dd_final2.csv python bench.py --steps 1 --warmup 1 --no-extra --no-cpu --no-graph > /dev/null 2>&1; wc -l gpurun_out/launches_dd_final2.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -c 1 -o gpurun_out/gemm_dd_final2 -f python tools/prof_gemm.py dd 1024 128 1 > /dev/null 2>&1
ls -la gpurun_out/gemm_dd_final2.ncu-rep
