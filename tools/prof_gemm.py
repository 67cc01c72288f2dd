"""The roofline GEMM of bench.py (M x M x nb, C += X Y^T) alone, for ncu --set full captures.

usage: python tools/prof_gemm.py [prec] [M] [nb] [reps]
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
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
m_l = {"dd": 2, "qd": 4, "od": 8}[prec]
X = torch.from_numpy(inputs.random_matrix(M, nb, prec, seed=11)).cuda()
Y = torch.from_numpy(inputs.random_matrix(M, nb, prec, seed=12)).cuda()
C = torch.from_numpy(inputs.random_matrix(M, M, prec, seed=13)).cuda()
work = torch.empty(8 * m_l * 8 * M * M, dtype=torch.uint8, device="cuda")
for _ in range(reps):
    mdls.gemm(prec, X, Y, C=C, trans_b=True, mode=1, work=work)
torch.cuda.synchronize()
print("ok", prec, M, nb)
