mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_plan.py tests/test_gpu_batched.py -q -x 2>&1 | tail -3
timeout 900 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "
import json;d=json.load(open('gpurun_out/bench.json'));print(d['ms_per_step'],d['e2e'],d['gpu_launches'],d['precisions'],d['batch_cfg5b_1gpu'])"; tail -3 gpurun_out/bench.err
timeout 900 python bench.py --workload cfg5b --steps 2 --warmup 1 > gpurun_out/bench5b.json 2> gpurun_out/bench5b.err; python -c "
import json;d=json.load(open('gpurun_out/bench5b.json'));print(d['ms_per_step'],d['value'],d['fp64_peak_frac'],d['e2e'])"; tail -3 gpurun_out/bench5b.err
