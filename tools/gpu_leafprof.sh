mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:leaf_reg_kernel -s 20 -c 1 -o gpurun_out/leaf_dd_r2 -f python tools/time_variants.py dd 1024 128 > gpurun_out/ncu_leaf.log 2>&1
tail -2 gpurun_out/ncu_leaf.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:leaf_reg_kernel -s 20 -c 1 -o gpurun_out/leaf_od_r2 -f python tools/time_variants.py od 1024 128 > gpurun_out/ncu_leaf_od.log 2>&1
tail -2 gpurun_out/ncu_leaf_od.log
