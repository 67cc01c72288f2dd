"""GPU outputs at BASELINE's full sizes against the oracle's (pinned, tests/test_oracle_invariants.py)
invariants, north_star: "GPU and oracle must each also meet the same invariant bounds"
E1 = max|Q^T Q - I|, E2 = max|A - QR| / max|A|, E3 = normal-equation residual, all <= 1e3 M u.

At n = 1024 the full Q^T Q costs M^3 md pairs, so E1 and E2 are evaluated on sampled columns
(the first, last, panel edges and random ones; the oracle's ``cols`` argument) -- every entry of
those columns of Q^T Q - I and of A - QR.  E3 is evaluated in full.  The oracle's own outputs
meet the same bounds (same functions, same sampled columns)."""
import numpy as np
import pytest
import torch

from paper_2110_08375_b200 import inputs

from ._parity import U_OF

pytestmark = pytest.mark.gpu


def _cols(K, nb, n_rand=4, seed=0):
    rng = np.random.default_rng(seed)
    c = {0, 1, nb - 1, nb, K // 2, K - nb, K - 2, K - 1} | set(int(v) for v in rng.integers(0, K, n_rand))
    return sorted(v for v in c if 0 <= v < K)


@pytest.mark.parametrize("prec", ["d", "dd", "qd", "od"])
def test_invariants_config2_full(orc, mdls, dev, prec):
    M = K = 1024
    nb = 128
    A, b = inputs.lstsq_problem(M, K, prec, seed=1)
    r = mdls.lstsq(prec, torch.from_numpy(A).to(dev), torch.from_numpy(b).to(dev), nb, form_q=True, want_R=True,
                   want_Q=True)
    torch.cuda.synchronize()
    assert int(r.info.item()) == 0
    Q = r.Q.cpu().numpy()
    R = r.R.cpu().numpy()
    x = r.x.cpu().numpy()
    bound = 1e3 * M * U_OF[prec]
    cols = _cols(K, nb)
    e1 = orc.inv_orth(prec, Q, cols=cols)
    e2 = orc.inv_recon(prec, A, Q, R, cols=cols)
    e3 = orc.inv_normal(prec, A, x, b)
    print(f"{prec} 1024: E1 {e1:.3e}  E2 {e2:.3e}  E3 {e3:.3e}  bound {bound:.3e}")
    assert e1 <= bound and e2 <= bound and e3 <= bound
    # the strictly-lower part of R is exactly zero
    low = np.tril_indices(M, -1)
    assert np.all(R[:, low[1], low[0]] == 0.0)
