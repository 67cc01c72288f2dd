timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 1 --workload cfg5a --size 1024 --steps 2 --warmup 1 2>&1 | grep -v Warning | tail -2
timeout 900 python bench.py --workload cfg5a --size 2048 --steps 1 --warmup 1 2>&1 | tail -1
