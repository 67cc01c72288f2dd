"""BASELINE config 5a on one B200: octo double QR of an 8,192 x 8,192 matrix (tile 128) through mdls_qr (Q formed),
timed with CUDA events, then sampled invariants evaluated by the oracle (test infrastructure):
  E1 on column pairs of Q: |Q_c^T Q_d - delta_cd|;  E2 on columns j: |A_j - sum_{i<=j} Q_i R_ij| / |A|_max,
both against the north_star bound 1e3 * M * u (u = 2^-416).  usage: python tools/cfg5a_od8192.py [M] [prec]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (checker only)
import paper_2110_08375_b200 as mdls  # noqa: E402
from paper_2110_08375_b200 import inputs  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
prec = sys.argv[2] if len(sys.argv) > 2 else "od"
nb = 128
U = {"dd": 2.0 ** -104, "qd": 2.0 ** -208, "od": 2.0 ** -416}[prec]
oracle.build()
t0 = time.time()
A = inputs.random_matrix_torch(M, M, prec, seed=5)
torch.cuda.synchronize()
print(f"{prec} {M}x{M}: input generated on the device in {time.time() - t0:.1f} s", flush=True)
A0 = A.clone()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
F, Q, W, info = mdls.qr(prec, A, nb, form_q=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
c = mdls.counts(prec, 0, M, M, nb)
flops = c["total_flops"]
print(f"QR with Q: {ms / 1e3:.2f} s, info {int(info.item())}, {flops / (ms * 1e-3) / 1e12:.2f} TFLOP/s "
      f"(Table-1 tally, {flops / (ms * 1e-3) / 1e12 / 37.22:.3f} of 37.2 TF)", flush=True)
del W
cols = [0, 1, M // 2, M - 1]
Qs = Q[:, cols, :].cpu().numpy()  # (m, 4, M)
worst1 = 0.0
for a in range(len(cols)):
    for b in range(a, len(cols)):
        d = oracle.dot(prec, np.ascontiguousarray(Qs[:, a, :]), np.ascontiguousarray(Qs[:, b, :]))
        if a == b:
            one = np.zeros((Qs.shape[0], 1))
            one[0] = 1.0
            d = oracle.md_op("sub", prec, d[:, None], one)[:, 0]
        worst1 = max(worst1, abs(float(d[0])))
bound = 1e3 * M * U
print(f"E1 (Q columns {cols}): max |Q_c^T Q_d - delta| = {worst1:.3e}, bound {bound:.3e}", flush=True)
worst2 = 0.0
amax = float(A0[0].abs().max().item())
for j in (0, 7, 200):
    Qj = Q[:, : j + 1, :].cpu().numpy()  # (m, j+1, M)
    Rj = F[:, j, : j + 1].cpu().numpy()  # (m, j+1): R(0..j, j)
    acc = np.zeros((Qj.shape[0], M))
    for i in range(j + 1):
        r = np.repeat(Rj[:, i:i + 1], M, axis=1)
        acc = oracle.md_op("add", prec, acc, oracle.md_op("mul", prec, np.ascontiguousarray(Qj[:, i, :]), r))
    d = oracle.md_op("sub", prec, A0[:, j, :].cpu().numpy(), acc)
    worst2 = max(worst2, float(np.max(np.abs(d[0]))) / amax)
print(f"E2 (columns 0, 7, 200): max |A_j - (QR)_j| / |A|_max = {worst2:.3e}, bound {bound:.3e}", flush=True)
assert int(info.item()) == 0 and worst1 <= bound and worst2 <= bound
print("config 5a single-GPU: OK")
