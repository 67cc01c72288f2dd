import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import oracle, paper_2110_08375_b200 as mdls
from paper_2110_08375_b200 import inputs
sys.path.insert(0, '/root/repo/tests')
from tests.test_gpu_arith import _operands
for prec in ['qd', 'od']:
    m = inputs.limbs(prec)
    a, _ = _operands(prec, 4000, 23)
    a = np.where(a[0] < 0, -a, a)
    z = a[0] == 0
    a[:, z] = 0.0
    a[0, z] = 1.0
    a = np.ascontiguousarray(a)
    ga = torch.from_numpy(a).cuda()
    one = np.zeros_like(a); one[0] = 1.0
    for op, ref in (('sqrt_fast', oracle.md_op('sqrt', prec, a)), ('recip_fast', oracle.md_op('div', prec, one, a))):
        got = mdls.md_op(op, prec, ga).cpu().numpy()
        d = oracle.md_op('sub', prec, got, ref)
        rel = np.abs(d[0]) / np.abs(ref[0])
        i = int(np.argmax(rel))
        print(prec, op, 'max rel', rel[i], 'at', i, 'nbad', int(np.sum(rel > 2.0**(-53*m+8))))
        print('  a  ', a[:, i]); print('  got', got[:, i]); print('  ref', ref[:, i])
