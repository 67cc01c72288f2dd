# Round measurement on one B200 (run under gpurun): bench + reference arm + GPU tests + ncu launch list and
# full captures of the roofline GEMM, the back-substitution update and the dd leaf + compute-sanitizer.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -c 6000 gpurun_out/bench_final.json; tail -3 gpurun_out/bench_final.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; tail -c 800 gpurun_out/bench_ref.json
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/gpu_tests_final.txt; tail -2 gpurun_out/gpu_tests_final.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_dd_final.csv python bench.py --steps 1 --warmup 1 --no-extra --no-cpu --no-graph > /dev/null 2>&1; wc -l gpurun_out/launches_dd_final.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -c 1 -o gpurun_out/gemm_dd_final -f python tools/prof_gemm.py dd 1024 128 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bs_update_kernel -s 2 -c 1 -o gpurun_out/bsupd_final -f python tools/time_bs.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:leaf_reg_kernel -s 20 -c 1 -o gpurun_out/leaf_dd_final -f python tools/time_variants.py dd 1024 128 > /dev/null 2>&1
for t in racecheck synccheck memcheck; do timeout 900 compute-sanitizer --tool $t python tools/sanitize_cfg1.py > gpurun_out/sanitize_$t.txt 2>&1; tail -2 gpurun_out/sanitize_$t.txt; done
ls -la gpurun_out/*.ncu-rep
