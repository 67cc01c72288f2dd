timeout 1200 python -m pytest tests -m gpu -x -q -s 2>&1 | grep -v "^$" | tail -8 > gpurun_out/quick_tests.txt
cat gpurun_out/quick_tests.txt
for p in dd qd od; do python tools/time_variants.py $p 1024 128 2>&1 | tail -2; done
MDLS_FUSED_APPLY=0 python tools/time_variants.py dd 1024 128 2>&1 | sed 's/^/nofused /' | tail -2
