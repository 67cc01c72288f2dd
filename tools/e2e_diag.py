"""Where the end-to-end time goes: plan replay alone, copies alone, both (dd 1024)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_08375_b200 as mdls  # noqa: E402
from paper_2110_08375_b200 import inputs  # noqa: E402

A_h, b_h = inputs.lstsq_problem(1024, 1024, "dd", 0)
A_p, b_p = torch.from_numpy(A_h).pin_memory(), torch.from_numpy(b_h).pin_memory()
plan = mdls.LstsqPlan("dd", 1024, 1024, 128)
x_p = torch.empty(tuple(plan.x.shape), dtype=torch.float64).pin_memory()


def t(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


print("plan.run            %.3f ms" % t(plan.run))
print("H2D A,b             %.3f ms" % t(lambda: (plan.A.copy_(A_p, non_blocking=True), plan.b.copy_(b_p, non_blocking=True))))
print("solve(A_p,b_p)+D2H  %.3f ms" % t(lambda: x_p.copy_(plan.solve(A_p, b_p), non_blocking=True)))
print("run+D2H             %.3f ms" % t(lambda: (plan.run(), x_p.copy_(plan.x, non_blocking=True))))
