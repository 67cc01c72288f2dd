"""The opt-in factorisation and back-substitution variants stay correct:
the GEMM-chained panel path (MDLS_CHAIN=0), the shared-memory leaf (MDLS_LEAF=smem), backward Q for dd
(MDLS_QFORM=backward), split-K instead of stream-K (MDLS_STREAMK=0), per-leaf updates of every column
(MDLS_DEFER=0) and 8-CTA leaf clusters (MDLS_LEAF_C=8).  The
switches are read once per process, so each runs in a fresh interpreter; x and R
are compared with the oracle at the north_star tolerance."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2110_08375_b200 import inputs

from ._parity import mat_cols_ok, vec_ok

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, {root!r})
import paper_2110_08375_b200 as mdls
from paper_2110_08375_b200 import inputs
prec, M, nb = {prec!r}, {M}, {nb}
A, b = inputs.lstsq_problem(M, M, prec, 7)
r = mdls.lstsq(prec, torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda(), nb, form_q=True, want_R=True)
torch.cuda.synchronize()
np.save({xout!r}, r.x.cpu().numpy())
np.save({rout!r}, r.R.cpu().numpy())
print(json.dumps({{"info": int(r.info.item())}}))
"""


@pytest.mark.parametrize("env", [{"MDLS_CHAIN": "0"}, {"MDLS_LEAF": "smem", "MDLS_CHAIN": "0"}, {"MDLS_QFORM": "backward"},
                                 {"MDLS_STREAMK": "0"}, {"MDLS_DEFER": "0"}, {"MDLS_LEAF_C": "8"}])
@pytest.mark.parametrize("prec,M,nb", [("dd", 256, 32), ("qd", 128, 16)])
def test_variant_parity(orc, tmp_path, env, prec, M, nb):
    xout, rout = str(tmp_path / "x.npy"), str(tmp_path / "R.npy")
    code = SCRIPT.format(root=ROOT, prec=prec, M=M, nb=nb, xout=xout, rout=rout)
    p = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True,
                       timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    assert json.loads(p.stdout.strip().splitlines()[-1])["info"] == 0
    A, b = inputs.lstsq_problem(M, M, prec, 7)
    xo, Ro, _ = orc.lstsq(prec, A, b)
    err, tol = vec_ok(orc, prec, np.load(xout), xo, M)
    assert err <= tol, (env, err, tol)
    assert mat_cols_ok(orc, prec, np.load(rout), Ro, M) <= 1.0


@pytest.mark.parametrize("env", [{"MDLS_BS_FLOW": "0"}, {"MDLS_BS_TMA": "0"}, {"MDLS_PDL": "0"}, {"MDLS_BSU": "1"},
                                 {"MDLS_BSU": "2"}, {"MDLS_BSU": "3"}])
@pytest.mark.parametrize("prec,M,nb", [("dd", 256, 32), ("qd", 256, 64)])
def test_chain_variant_parity(orc, tmp_path, env, prec, M, nb):
    """launch-ordered back substitution, LDGSTS staging, no programmatic dependent launch, the update-kernel
    shapes of MDLS_BSU: x and R at the north_star tolerance"""
    test_variant_parity(orc, tmp_path, env, prec, M, nb)
