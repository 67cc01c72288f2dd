import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle, paper_2110_08375_b200 as mdls
from paper_2110_08375_b200 import inputs
dev = torch.device("cuda:0")
for (M, K, nb) in [(64, 64, 8), (64, 64, 16), (128, 128, 16), (32, 32, 4), (64, 32, 8), (64, 16, 8), (16, 16, 8), (24, 16, 8), (64,64,32), (72, 64, 16)]:
    A = inputs.random_matrix(M, K, "dd", seed=1)
    F, Q, W, info = mdls.qr("dd", torch.from_numpy(A).to(dev), nb, form_q=True, want_w=True)
    torch.cuda.synchronize()
    Fo, beta = oracle.qr("dd", A)
    Qo = oracle.form_q("dd", Fo, beta)
    Qg = Q.cpu().numpy()
    dq = np.abs(Qg[0] - Qo[0])  # (cols, rows)
    bad = np.nonzero(dq.max(axis=1) > 1e-10)[0]
    print(M, K, nb, "Q bad cols", bad[:10], len(bad), "max", dq.max())
    # W check: P_WY of panel 0 applied: compare W from GPU vs recurrence in numpy fp64
    Wg = W.cpu().numpy()[0].T  # (M, K)
    Y = np.tril(Fo[0].T, -1)[:, :K] + np.eye(M)[:, :K]
    b0 = beta[0]
    for k in range(K // nb):
        j0 = k * nb
        Wk = np.zeros((M, nb))
        for l in range(nb):
            v = Y[:, j0 + l].copy(); v[:j0 + l] = 0
            z = -b0[j0 + l] * (v + Wk[:, :l] @ (Y[:, j0:j0 + l].T @ v)) if l else -b0[j0 + l] * v
            Wk[:, l] = z
        Wk[:j0] = 0
        e = np.abs(Wk - Wg[:, j0:j0 + nb]).max()
        if e > 1e-8: print("   panel", k, "W err", e)
