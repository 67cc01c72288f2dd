timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -2
for v in 1 0; do MDLS_STREAMK=$v timeout 300 python bench.py --no-cpu --no-extra --steps 10 > gpurun_out/b.json 2>&1; echo "SK=$v $(python -c "import json;d=json.load(open('gpurun_out/b.json'));print(d['ms_per_step'],d['e2e']['ms_per_step'],d['fp64_peak_frac'],d['roofline']['frac'],d['roofline']['launch_ms'])" 2>&1 | tail -1)"; done
for p in qd od; do for v in 1 0; do MDLS_STREAMK=$v timeout 300 python tools/time_variants.py $p 1024 128 2>&1 | head -1; done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -c 1 -o gpurun_out/gemm_dd_sk -f python tools/prof_gemm.py dd 1024 128 1 > gpurun_out/ncu_gemm.log 2>&1; tail -1 gpurun_out/ncu_gemm.log
timeout 1200 python -m pytest tests -m gpu -q -x -k "qr or invariants or determinism or batched" 2>&1 | tail -2
