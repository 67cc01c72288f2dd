mkdir -p gpurun_out
timeout 900 python bench.py --workload cfg5b --steps 2 --warmup 1 > gpurun_out/bench5b.json 2> gpurun_out/bench5b.err; tail -c 1500 gpurun_out/bench5b.json; tail -3 gpurun_out/bench5b.err
timeout 900 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 2500 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
