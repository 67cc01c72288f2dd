set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
free -g | head -2
timeout 1500 python -m pytest tests -m gpu -q -s -p no:randomly > gpurun_out/gpu_tests.txt 2>&1
tail -40 gpurun_out/gpu_tests.txt
for tool in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cfg1.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -5 gpurun_out/sanitize_$tool.txt
done
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
