"""Run a few least-squares solves through the library (for ncu / sanitizer captures).

usage: python tools/prof_step.py [prec] [M] [nb] [iters]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_08375_b200 as mdls  # noqa: E402
from paper_2110_08375_b200 import inputs  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "dd"
M = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
nb = int(sys.argv[3]) if len(sys.argv) > 3 else 128
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 2
A, b = inputs.lstsq_problem(M, M, prec, 0)
A = torch.from_numpy(A).cuda()
b = torch.from_numpy(b).cuda()
for _ in range(iters):
    r = mdls.lstsq(prec, A, b, nb, form_q=True)
torch.cuda.synchronize()
print("info", int(r.info.item()), "launches", mdls.launch_count())
