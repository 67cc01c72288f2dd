# dd dev loop: dd parity tests, short dd bench (persistent chain and per-leaf launches)
timeout 900 python -m pytest tests/test_gpu_qr.py tests/test_gpu_backsub.py tests/test_gpu_sharded.py -x -q -s -k "dd or spec or zero or nonfinite or singular or config4" 2>&1 | grep -v "^$" | tail -8 > gpurun_out/dd_tests.txt
cat gpurun_out/dd_tests.txt
for v in "" "MDLS_PERSIST=0"; do
  env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-extra > gpurun_out/dd_bench.json 2> gpurun_out/dd_bench.err
  python -c "
import json; d=json.load(open('gpurun_out/dd_bench.json')); print('$v dd ms', d['ms_per_step'], 'frac', d['fp64_peak_frac'], 'family', d['family_ms'])" || tail -5 gpurun_out/dd_bench.err
done
