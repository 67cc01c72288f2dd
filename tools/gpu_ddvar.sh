# dd variants: leaf exclusivity / cluster size
for v in "" "MDLS_LEAF_EXCL=1" "MDLS_LEAF_C=8" "MDLS_LEAF_C=8 MDLS_LEAF_EXCL=1"; do
  env $v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-extra > gpurun_out/v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/v.json')); print('$v', 'dd ms', d['ms_per_step'], 'panel', d['family_ms']['panel'], 'gemm', d['family_ms']['gemm'])"
done
