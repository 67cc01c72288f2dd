# quick GPU check: all GPU tests (config 2/3 margins printed), a bench line, the roofline GEMM under ncu
timeout 1200 python -m pytest tests -m gpu -x -q -s 2>&1 | grep -v "^$" | tail -25 > gpurun_out/quick_tests.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/quick_bench.json 2> gpurun_out/quick_bench.err
for p in dd qd od; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 1 -o gpurun_out/gemm_roof_$p python tools/prof_gemm.py $p 1024 128 3 > gpurun_out/ncu_gemm_$p.log 2>&1
done
cat gpurun_out/quick_tests.txt; cat gpurun_out/quick_bench.json; tail -5 gpurun_out/quick_bench.err
