timeout 900 python -m pytest tests/test_gpu_backsub.py tests/test_gpu_qr.py -x -q 2>&1 | tail -2
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bs_bench.json 2> gpurun_out/bs_bench.err
python -c "
import json; d=json.load(open('gpurun_out/bs_bench.json')); print('dd', d['ms_per_step'], 'cfg4', d['backsub_cfg4'])" || tail -5 gpurun_out/bs_bench.err
