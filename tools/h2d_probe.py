"""H2D bandwidth and host-plan timing probe: python tools/h2d_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_08375_b200 as mdls  # noqa: E402
from paper_2110_08375_b200 import inputs  # noqa: E402

h = torch.empty(16793600 // 8, dtype=torch.float64).pin_memory()
d = torch.empty_like(h, device="cuda")
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    d.copy_(h, non_blocking=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"H2D 16.8 MB: {ms:.3f} ms = {16.79 / ms:.1f} GB/s")
A, b = inputs.lstsq_problem(1024, 1024, "dd", 0)
hp = mdls.HostLstsqPlan("dd", 1024, 1024, 128)
hp.A.copy_(torch.from_numpy(A))
hp.b.copy_(torch.from_numpy(b))
dp = mdls.LstsqPlan("dd", 1024, 1024, 128)
dp.A.copy_(torch.from_numpy(A).cuda())
dp.b.copy_(torch.from_numpy(b).cuda())
for name, p in (("device plan", dp), ("host plan", hp), ("device plan", dp), ("host plan", hp)):
    for _ in range(3):
        p.run()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        p.run()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / 10:.3f} ms per replay", flush=True)
# direct calls (no graph): host-input call vs device call
Ap, bp = torch.from_numpy(A).pin_memory(), torch.from_numpy(b).pin_memory()
Ad, bd = torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda()
for name, f in (("direct device", lambda: mdls.lstsq("dd", Ad, bd, 128, form_q=True)),
                ("direct host", lambda: mdls.lstsq_host("dd", Ap, bp, 128, form_q=True))):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        f()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / 5:.3f} ms per call", flush=True)
print("MDLS_HOST_ZC =", os.environ.get("MDLS_HOST_ZC", "1 (default)"))
