# round measurement: GPU tests, default bench (with cpu baseline), launch list, ncu full of the leaf kernel
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/final_tests.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/final_gpu.txt
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv python tools/prof_step.py dd 1024 128 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:leaf_reg_kernel -s 20 -c 1 -o gpurun_out/final_leaf python tools/prof_step.py dd 1024 128 1 > /dev/null 2>&1
timeout 300 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
cat gpurun_out/final_tests.txt; head -c 600 gpurun_out/final_bench.json; echo; cat gpurun_out/final_ref.json | head -c 400
