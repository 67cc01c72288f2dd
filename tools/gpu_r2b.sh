set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 4000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -c 1 -o gpurun_out/gemm_dd_r2 -f python tools/prof_gemm.py dd 1024 128 1 > gpurun_out/ncu_gemm.log 2>&1
tail -3 gpurun_out/ncu_gemm.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_dd.csv python bench.py --steps 1 --warmup 1 --no-extra --no-cpu --no-graph > gpurun_out/ncu_launch.log 2>&1
tail -3 gpurun_out/ncu_launch.log
