for r in 1 2 3; do
MDLS_BS_FLOW=1 timeout 300 python tools/time_bs.py 2>&1 | tail -1 | sed 's/^/flow /'
MDLS_BS_FLOW=0 timeout 300 python tools/time_bs.py 2>&1 | tail -1 | sed 's/^/noflow /'
done
