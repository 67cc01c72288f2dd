mkdir -p gpurun_out
for p in dd; do
python tools/time_plan.py $p 1024 128
MDLS_LEAF_C=8 python tools/time_plan.py $p 1024 128
MDLS_LEAF_EXCL=0 python tools/time_plan.py $p 1024 128
MDLS_QFORM=backward python tools/time_plan.py $p 1024 128
MDLS_STREAMK=0 python tools/time_plan.py $p 1024 128
MDLS_DEFER=0 python tools/time_plan.py $p 1024 128
MDLS_PDL=0 python tools/time_plan.py $p 1024 128
done
python tools/time_plan.py qd 1024 128 5
MDLS_LEAF_C=8 python tools/time_plan.py qd 1024 128 5
