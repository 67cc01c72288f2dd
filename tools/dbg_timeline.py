"""Print the factorisation timeline (MDLS_TIMELINE=1) of lstsq (two calls): python tools/dbg_timeline.py od 1024 128 [q]"""
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
fq = len(sys.argv) > 4 and sys.argv[4] == "q"
for _ in range(2):  # the second call is the representative one (the first loads modules)
    mdls.lstsq(prec, A, b, nb, form_q=fq)
    torch.cuda.synchronize()
    print("---", flush=True)
