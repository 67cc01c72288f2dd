"""Time lstsq variants (form_q on/off) for one precision: python tools/time_variants.py dd 1024 128"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_08375_b200 as mdls  # noqa: E402
from paper_2110_08375_b200 import inputs  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "dd"
M = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
nb = int(sys.argv[3]) if len(sys.argv) > 3 else 128
A, b = inputs.lstsq_problem(M, M, prec, 0)
A = torch.from_numpy(A).cuda()
b = torch.from_numpy(b).cuda()
for form_q in (True, False):
    for _ in range(3):
        mdls.lstsq(prec, A, b, nb, form_q=form_q)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 5
    e0.record()
    for _ in range(n):
        mdls.lstsq(prec, A, b, nb, form_q=form_q)
    e1.record()
    torch.cuda.synchronize()
    print(f"{prec} M={M} nb={nb} form_q={form_q}: {e0.elapsed_time(e1) / n:.3f} ms", flush=True)
