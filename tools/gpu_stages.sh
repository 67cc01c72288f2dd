for w in cfg3qd cfg3od; do
  for c in 1 0; do
    MDLS_CHAIN=$c timeout 600 python bench.py --workload $w --steps 2 --warmup 1 --no-cpu --no-extra > gpurun_out/st.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/st.json')); print('$w chain=$c', d['ms_per_step'], {k:round(v,1) for k,v in d['stages_ms'].items()}, {k:round(v,1) for k,v in d['family_ms'].items()})"
  done
done
