"""Time qd back substitution at n=17920 (BASELINE config 4): python tools/bs_variants.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_08375_b200 as mdls  # noqa: E402
from paper_2110_08375_b200 import inputs  # noqa: E402

n, nb = 17920, 128
U = inputs.lu_upper_torch(n, "qd", 0)
y = torch.from_numpy(inputs.random_vector(n, "qd", 1)).cuda()
for _ in range(2):
    mdls.backsub("qd", U, y, nb)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    mdls.backsub("qd", U, y, nb)
e1.record()
torch.cuda.synchronize()
print(f"chunk={os.environ.get('MDLS_INV_CHUNK', '16')}: qd backsub n={n}: {e0.elapsed_time(e1) / 5:.3f} ms", flush=True)
