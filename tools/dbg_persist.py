"""Debug the persistent leaf chain on small problems (prints as it goes)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_08375_b200 as mdls  # noqa: E402
from paper_2110_08375_b200 import inputs  # noqa: E402

for (M, nb) in [(64, 8), (128, 16), (1024, 128)]:
    A, b = inputs.lstsq_problem(M, M, "dd", 0)
    A = torch.from_numpy(A).cuda()
    b = torch.from_numpy(b).cuda()
    print("start", M, nb, flush=True)
    r = mdls.lstsq("dd", A, b, nb, form_q=True)
    torch.cuda.synchronize()
    print("done", M, nb, "info", int(r.info.item()), flush=True)
