mkdir -p gpurun_out
run() { env $1 timeout 300 python bench.py --no-cpu --no-extra --steps 10 > gpurun_out/b.json 2>&1; echo "$1: $(python -c "import json;d=json.load(open('gpurun_out/b.json'));print(d['ms_per_step'],d['e2e']['ms_per_step'],d['fp64_peak_frac'],d['roofline']['frac'])" 2>&1 | tail -1)"; }
run "MDLS_QFORM=backward"
run "MDLS_QFORM=backward MDLS_DEFER=0"
timeout 300 python tools/time_variants.py dd 1024 128 2>&1
MDLS_DEFER=0 timeout 300 python tools/time_variants.py dd 1024 128 2>&1
MDLS_TIMELINE=1 timeout 120 python tools/time_variants.py dd 1024 128 > gpurun_out/timeline_dd.txt 2>&1
