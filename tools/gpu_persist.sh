# qd/od (and dd) solve times with the per-leaf launched chain vs the persistent chain
for p in dd qd od; do
  python tools/time_variants.py $p 1024 128 2>&1 | tail -2
  MDLS_PERSIST=1 python tools/time_variants.py $p 1024 128 2>&1 | sed 's/^/persist /' | tail -2
done
