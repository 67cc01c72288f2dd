"""Config 4 timing (qd BS n = 17920, nb 128) through bench.bench_backsub: python tools/time_bs.py [prec n nb]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "qd"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 17920
nb = int(sys.argv[3]) if len(sys.argv) > 3 else 128
r = bench.bench_backsub(torch.device("cuda"), prec, n, nb, 5, 2, False)
print(os.environ.get("MDLS_INV_CHUNK", "default"), json.dumps({k: r[k] for k in ("ms_per_solve", "fp64_peak_frac", "stages_ms", "update_hbm_gbs")}))
