# dd dev loop: leaf phases, dd parity tests, short dd bench
./tools/leaf_prof 2>&1 | grep -v "^M=.*us$" | head -20 > gpurun_out/leaf_prof.txt
timeout 900 python -m pytest tests/test_gpu_qr.py tests/test_gpu_backsub.py tests/test_gpu_sharded.py -x -q -s -k "dd or spec or zero or nonfinite or singular or config4" 2>&1 | grep -v "^$" | tail -8 > gpurun_out/dd_tests.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-extra > gpurun_out/dd_bench.json 2> gpurun_out/dd_bench.err
cat gpurun_out/leaf_prof.txt gpurun_out/dd_tests.txt; python -c "
import json; d=json.load(open('gpurun_out/dd_bench.json')); print('dd ms', d['ms_per_step'], 'frac', d['fp64_peak_frac'], 'stages', d['stages_ms'], 'family', d['family_ms'])"
