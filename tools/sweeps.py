"""f3: dimension and tile sweeps on the paper's shapes, one B200, CUDA events, L2 flushed between
solves; prints one JSON object (profiles/r02_sweeps.json) and a markdown summary (profiles/r02_sweeps.md).

  T5  real dd QR/lstsq at n = 512 over tilings 32x16, 16x32, 8x64, 4x128, 2x256 (the complex half
      of T5 is row f2, not built);
  T6  QR + BS (lstsq with Q) vs dimension n = 512, 1024, 1536, 2048 (4..16 x 128) in dd/qd/od;
  T7  back substitution in dd/qd/od at n = 5120, 10240, 20480 (64/128/256 x 80; od also 128 x 160);
  T8  qd back substitution at n = 20480 tiled 320x64, 160x128, 80x256;
  T9  qd back substitution 80 x nb, nb = 32..256 (n = 2560..20480), with the roofline of the
      update stage (T10): pairs x 8 m bytes per U entry read once -> GB/s vs the measured HBM
      peak, and FP64-pipe ops/s vs 18.6 T.
Flops are the ledger's Table-1 tallies (mdls_count), as in bench.py.  usage: python tools/sweeps.py [quick]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_08375_b200 as mdls  # noqa: E402
from paper_2110_08375_b200 import inputs  # noqa: E402

PEAK_TF = 37.22
PIPE_T = 18.61
OPS_PER_PAIR = {"dd": 12, "qd": 116, "od": 970}
quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
dev = torch.device("cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / reps


def lstsq_point(prec, n, nb, reps):
    A, b = inputs.lstsq_problem(n, n, prec, seed=n + nb)
    plan = mdls.LstsqPlan(prec, n, n, nb, form_q=True)
    plan.A.copy_(torch.from_numpy(A))
    plan.b.copy_(torch.from_numpy(b))
    ms = timed(plan.run, reps)
    assert int(plan.info.item()) == 0
    c = mdls.counts(prec, 2, n, n, nb)
    f = c["total_flops"]
    qr = sum(c["stages"][s]["flops"] for s in ("house", "panel", "wy", "trailing", "form_q"))
    return {"prec": prec, "n": n, "nb": nb, "tiles": n // nb, "ms": round(ms, 4), "tflops": round(f / ms / 1e9, 3),
            "peak_frac": round(f / ms / 1e9 / PEAK_TF, 4), "qr_share_flops": round(qr / f, 4)}


def backsub_point(prec, n, nb, reps):
    U = inputs.lu_upper_torch(n, prec, seed=n + nb, device=dev)
    y = inputs.random_vector_torch(n, prec, seed=n, device=dev)
    mdls.trace_enable(False)

    def run():
        return mdls.backsub(prec, U, y, nb)

    ms = timed(run, reps)
    x, info = run()
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    mdls.trace_enable(True)
    run()
    torch.cuda.synchronize()
    mdls.trace_enable(False)
    tr = mdls.trace_collect()
    c = mdls.counts(prec, 1, n, n, nb)
    f = c["total_flops"]
    pu = c["stages"]["bsupdate"]["mul"]
    upd = tr["stages_ms"]["bsupdate"]
    m = inputs.limbs(prec)
    del U
    torch.cuda.empty_cache()
    return {"prec": prec, "n": n, "nb": nb, "tiles": n // nb, "ms": round(ms, 4), "tflops": round(f / ms / 1e9, 3),
            "peak_frac": round(f / ms / 1e9 / PEAK_TF, 4),
            "stages_ms": {k: round(tr["stages_ms"][k], 4) for k in ("invert", "mulinv", "bsupdate")},
            "update_gbs": round(pu * 8 * m / (upd * 1e-3) / 1e9, 1) if upd > 0 else None,
            "update_intensity_pairs_per_byte": round(1.0 / (8 * m), 4),
            "update_pipe_frac": round(pu * OPS_PER_PAIR[prec] / (upd * 1e-3) / 1e12 / PIPE_T, 4) if upd > 0 else None}


out = {"device": torch.cuda.get_device_name(), "T5": [], "T6": [], "T7": [], "T8": [], "T9": []}
_lstsq_point, _backsub_point = lstsq_point, backsub_point


def lstsq_point(prec, n, nb, reps):  # noqa: F811
    try:
        return _lstsq_point(prec, n, nb, reps)
    except Exception as e:  # a shape the library refuses is recorded, not fatal
        return {"prec": prec, "n": n, "nb": nb, "error": str(e)[:200]}


def backsub_point(prec, n, nb, reps):  # noqa: F811
    try:
        return _backsub_point(prec, n, nb, reps)
    except Exception as e:
        torch.cuda.empty_cache()
        return {"prec": prec, "n": n, "nb": nb, "error": str(e)[:200]}

reps = 2 if quick else 3
for nb in (16, 32, 64, 128, 256):
    out["T5"].append(lstsq_point("dd", 512, nb, reps))
    print(json.dumps(out["T5"][-1]), flush=True)
for prec in ("dd", "qd", "od"):
    for n in ((512, 1024) if quick else (512, 1024, 1536, 2048)):
        if prec == "od" and n > 1536 and quick:
            continue
        out["T6"].append(lstsq_point(prec, n, 128, 1 if prec == "od" else reps))
        print(json.dumps(out["T6"][-1]), flush=True)
for prec in ("dd", "qd", "od"):
    for nb in (64, 128, 256):
        out["T7"].append(backsub_point(prec, 80 * nb, nb, reps))
        print(json.dumps(out["T7"][-1]), flush=True)
out["T7"].append(backsub_point("od", 128 * 160, 160, reps))
for nt, nb in ((320, 64), (160, 128), (80, 256)):
    out["T8"].append(backsub_point("qd", nt * nb, nb, reps))
    print(json.dumps(out["T8"][-1]), flush=True)
for nb in (32, 64, 96, 128, 160, 192, 224, 256):
    out["T9"].append(backsub_point("qd", 80 * nb, nb, reps))
    print(json.dumps(out["T9"][-1]), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/sweeps.json", "w") as f:
    json.dump(out, f, indent=1)
lines = ["# f3 sweeps (tools/sweeps.py), " + out["device"], ""]
for key, cols in (("T5", ["prec", "n", "nb", "tiles", "ms", "tflops", "peak_frac"]),
                  ("T6", ["prec", "n", "nb", "ms", "tflops", "peak_frac", "qr_share_flops"]),
                  ("T7", ["prec", "n", "nb", "tiles", "ms", "tflops", "peak_frac", "update_gbs", "update_pipe_frac"]),
                  ("T8", ["prec", "n", "nb", "tiles", "ms", "tflops", "peak_frac", "update_gbs", "update_pipe_frac"]),
                  ("T9", ["prec", "n", "nb", "tiles", "ms", "tflops", "peak_frac", "update_gbs", "update_pipe_frac"])):
    lines += [f"## {key}", "", "| " + " | ".join(cols) + " |", "|" + "---|" * len(cols)]
    for r in out[key]:
        lines.append("| " + " | ".join(str(r.get(c)) for c in cols) + " |")
    lines.append("")
with open("gpurun_out/sweeps.md", "w") as f:
    f.write("\n".join(lines))
print("\n".join(lines))
