"""Print the factorisation timeline (MDLS_TIMELINE=1) of one lstsq: python tools/dbg_timeline.py od 1024 128"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_08375_b200 as mdls  # noqa: E402
from paper_2110_08375_b200 import inputs  # noqa: E402

prec = sys.argv[1]
M = int(sys.argv[2])
nb = int(sys.argv[3])
A, b = inputs.lstsq_problem(M, M, prec, 0)
A = torch.from_numpy(A).cuda()
b = torch.from_numpy(b).cuda()
mdls.lstsq(prec, A, b, nb, form_q=False)
torch.cuda.synchronize()
print("---", flush=True)
