for v in 0 2 1 3; do MDLS_BSU=$v timeout 600 python tools/time_bs.py 2>&1 | tail -1; done
