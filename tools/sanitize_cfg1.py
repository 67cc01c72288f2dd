"""Small solves for compute-sanitizer (racecheck / synccheck / memcheck): BASELINE config 1
(dd 64 x 64, tile 8) plus qd/od shapes that exercise the register leaf's cluster pushes
(st.async + mbarrier), the prologue, split-K GEMMs and the back-substitution chain (nb % 32 == 0:
the dataflow counters and the TMA-staged update; plain double)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2110_08375_b200 as mdls  # noqa: E402
from paper_2110_08375_b200 import inputs  # noqa: E402

dev = torch.device("cuda:0")
for prec, M, K, nb in [("dd", 64, 64, 8), ("qd", 96, 64, 16), ("od", 64, 32, 8), ("dd", 256, 256, 32), ("d", 64, 64, 8),
                       ("qd", 256, 256, 64)]:
    A, b = inputs.lstsq_problem(M, K, prec, 0)
    for fq in (True, False):
        r = mdls.lstsq(prec, torch.from_numpy(A).to(dev), torch.from_numpy(b).to(dev), nb, form_q=fq)
        torch.cuda.synchronize()
        print(prec, M, K, nb, fq, "info", int(r.info.item()), flush=True)
