"""Time one plan replay (library CUDA graph, as bench.py) per env variant, L2 flushed between replays:
python tools/time_plan.py dd 1024 128 [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_08375_b200 as mdls  # noqa: E402
from paper_2110_08375_b200 import inputs  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "dd"
M = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
nb = int(sys.argv[3]) if len(sys.argv) > 3 else 128
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
A, b = inputs.lstsq_problem(M, M, prec, 0)
plan = mdls.LstsqPlan(prec, M, M, nb, form_q=True)
plan.solve(torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda())
flush = torch.empty(512 * 2 ** 20, dtype=torch.uint8, device="cuda")
ts = []
for i in range(reps + 3):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    plan.run()
    e1.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(e0.elapsed_time(e1))
ts.sort()
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("MDLS_")) or "default"
print(f"{prec} {M} nb={nb} [{env}] median {ts[len(ts) // 2]:.3f} ms min {ts[0]:.3f}", flush=True)
