import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import oracle, paper_2110_08375_b200 as mdls
from paper_2110_08375_b200 import inputs
from tests._parity import vec_ok, mat_cols_ok
for seed in range(3):
    prec = 'od'; M = K = 64
    A, b = inputs.lstsq_problem(M, K, prec, seed)
    r = mdls.lstsq(prec, torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda(), 8, form_q=True, want_R=True, want_y=True)
    torch.cuda.synchronize()
    xo, Ro, yo = oracle.lstsq(prec, A, b)
    Rg = r.R.cpu().numpy()
    print('seed', seed, 'info', int(r.info.item()), 'R ratio', mat_cols_ok(oracle, prec, Rg, Ro, K), 'y err', vec_ok(oracle, prec, r.y.cpu().numpy()[:, :K].copy(), yo[:, :K].copy(), K), 'x err', vec_ok(oracle, prec, r.x.cpu().numpy(), xo, K))
    # backsub alone on the oracle's R and y
    x2, info2 = mdls.backsub(prec, torch.from_numpy(Ro).cuda(), torch.from_numpy(yo).cuda(), 8, n=K)
    print('   BS on oracle R: x err', vec_ok(oracle, prec, x2.cpu().numpy(), xo, K))
    d = np.abs(Rg[0] - Ro[0]); bad = np.nonzero(d.max(axis=1) > 1e-12)[0]; print('   bad R cols', bad[:10])
