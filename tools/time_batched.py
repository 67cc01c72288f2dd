"""Batched dd least squares throughput on one GPU: python tools/time_batched.py [B] [groups...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_08375_b200 as mdls  # noqa: E402
from paper_2110_08375_b200 import inputs  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
glist = [int(g) for g in sys.argv[2:]] or [1, 2, 4, 6, 8]
prec, M, nb = os.environ.get("PREC", "dd"), 1024, 128
base = [inputs.lstsq_problem(M, M, prec, s) for s in range(min(B, 8))]
A = torch.from_numpy(np.stack([base[p % len(base)][0] for p in range(B)])).cuda()
b = torch.from_numpy(np.stack([base[p % len(base)][1] for p in range(B)])).cuda()
flops = mdls.counts(prec, 2, M, M, nb)["total_flops"]
for G in glist:
    work = torch.empty(mdls.batch_workspace_bytes(prec, 2, M, M, nb, G), dtype=torch.uint8, device="cuda")
    for _ in range(2):
        x, info = mdls.lstsq_batched(prec, A, b, nb, groups=G, work=work)
    torch.cuda.synchronize()
    assert info.cpu().tolist() == [0] * B
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        x, info = mdls.lstsq_batched(prec, A, b, nb, groups=G, work=work)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 3
    e0.record()
    for _ in range(n):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"{prec} B={B} groups={G}: {ms:.2f} ms per batch, {ms / B:.3f} ms per solve, "
          f"{flops * B / (ms * 1e-3) / 1e12:.2f} TFLOP/s ({flops * B / (ms * 1e-3) / 1e12 / 37.22:.3f} of peak)",
          flush=True)
    del g, work
