mkdir -p gpurun_out
timeout 300 python tools/cfg5a_od8192.py 1024 od 2>&1 | tail -5
timeout 1200 python tools/sweeps.py > gpurun_out/sweeps.log 2>&1; tail -60 gpurun_out/sweeps.log
timeout 1500 python tools/cfg5a_od8192.py 8192 od > gpurun_out/cfg5a.txt 2>&1; cat gpurun_out/cfg5a.txt
