#!/usr/bin/env python
"""Benchmark: multiple-double least squares (arXiv 2110.08375) on B200.

One "step" = one least-squares solve through the whole hot path (all SURVEY
8(a) rows): blocked Householder QR with W/Y accumulation and the trailing
update, backward Q formation, Q^T b with the explicit Q, tiled back
substitution (tile inversion + the multiply/update chain) -- the paper's
Table 11 pipeline.  Default workload = BASELINE config 2:
double double, 1,024 x 1,024, tile 128.

Metric (BASELINE.json): md QR+backsub double flops/s, i.e. canonical md-op
counts (mdls_count) weighted with the paper's Table 1 sums
(P:102-136), divided by device time; reported in GFLOP/s with the fraction of
the B200 FP64 peak (37.2 TFLOP/s = 148 SMs x 64 DFMA/clk x 2 x 1.965 GHz).

Launch: python bench.py [--gpus N --steps K --warmup W] [--impl reference].
N > 1 runs under torchrun, one rank per GPU, each rank solving its own
problem (batch sharding, no collective): weak scaling, max time over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (precision, M, K, nb)
    "cfg1": ("dd", 64, 64, 8),
    "cfg2": ("dd", 1024, 1024, 128),
    "cfg3qd": ("qd", 1024, 1024, 128),
    "cfg3od": ("od", 1024, 1024, 128),
    "cfg5b": ("dd", 1024, 1024, 128),  # + BATCH_5B independent problems sharded over the ranks
    "cfg5a": ("od", 8192, 8192, 128),  # block-column sharded QR + lstsq (sharded.py), --size overrides M = K
}
BATCH_5B = 256
BATCH_CHUNK = 32  # problems per captured CUDA graph (one mdls_lstsq_batched call each)
METRIC = "md QR+backsub double-flops/s & % FP64 peak at n=1024 dd/qd/od, 1/2/4/8 B200"
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12      # 37.2 (FMA = 2 flops)
FP64_PIPE_TOPS = 148 * 64 * 1.965e9 / 1e12            # 18.6 FP64-pipe lane ops/s (DADD/DMUL/DFMA each 1)
# FP64 pipe instructions per md pair (one md mul + one md add) as the GEMM kernels implement them
# (md.cuh Acc: dd unnormalised FMA pair accumulation 12; qd/od level-bin accumulation: 2M-1 FMAs +
# sum_{n<=M-2} (n+1) [two_prod + exact deposits] = 115 / 967, + the per-k-tile bin renormalisation)
OPS_PER_PAIR = {"d": 1, "dd": 12, "qd": 116, "od": 970}
# dram traffic per launch of the roofline GEMM (1024 x 1024 x 128, C += X Y^T) from one ncu --set full
# capture (tools/prof_gemm.py; dd: profiles/r02_ncu_final_c.txt, 64 x 32 tiles, split-K 4 -- the write is the
# split-K partials; qd/od: profiles/r01_ncu_gemm_roofline.txt)
GEMM_NCU_TRAFFIC = {"dd": 4259840 + 9678336, "qd": 42001664 + 119040, "od": 84171776 + 14920192}
# paper's V100 times for the same least-squares workload (T11): QR + BS kernel ms
PAPER_V100_MS = {"dd": 451.1 + 4.0, "qd": 3020.6 + 28.0, "od": 11924.5 + 114.5}
L2_FLUSH_BYTES = 512 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="cfg2")
    ap.add_argument("--no-extra", action="store_true", help="skip the qd/od side measurements")
    ap.add_argument("--no-cpu", action="store_true", help="skip the oracle cpu_baseline")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--groups", type=int, default=8, help="stream groups of the batched solves (cfg5b)")
    ap.add_argument("--batch", type=int, default=BATCH_5B, help="problems of the cfg5b batch (all ranks)")
    ap.add_argument("--size", type=int, default=0, help="cfg5a: M = K (default 8192)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.out = None

    def __enter__(self):
        try:
            self.out = open(f"/tmp/mdls_clocks_{os.getpid()}.csv", "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.out, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.out:
            self.out.close()

    def summary(self):
        try:
            rows = [l.strip().split(",") for l in open(self.out.name) if l.strip()]
        except Exception:
            rows = []
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = sorted(float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit())
        mx = max(float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for k, name in enumerate(names):
                if len(r) > 5 + k and "Active" in r[5 + k] and "Not" not in r[5 + k]:
                    reasons.add(name)
        loaded = [v for v in sm if v > 0.5 * mx] or sm
        return {"sm_mhz": loaded[len(loaded) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(rows)}


def make_problem(prec, M, K, seed):
    from paper_2110_08375_b200 import inputs

    return inputs.lstsq_problem(M, K, prec, seed)


def ledger_flops(prec, M, K, nb, form_q=True):
    import paper_2110_08375_b200 as mdls

    c = mdls.counts(prec, 2 if form_q else 4, M, K, nb)
    return c


def gemm_pairs(ledger):
    """md pairs computed by the md GEMM kernels (WY build, trailing update, Q formation, Q^T b)."""
    st = ledger["stages"]
    return sum(st[s]["mul"] for s in ("wy", "trailing", "form_q", "qtb"))


def step_fp64_ops(led, prec):
    """FP64-pipe instructions of all md pairs of the step (every stage, GEMM-rate per pair), for the GEMM share"""
    return float(sum(v["mul"] for v in led["stages"].values())) * OPS_PER_PAIR[prec]


def gemm_roofline(dev, prec, M, nb, reps=20, warmup=3):
    """Roofline of the dominant kernel: the md GEMM at the solve's largest launch shape (M x M x nb,
    C += X Y^T), timed alone with CUDA events on the current stream."""
    import torch

    import paper_2110_08375_b200 as mdls
    from paper_2110_08375_b200 import inputs

    m_l = {"d": 1, "dd": 2, "qd": 4, "od": 8}[prec]
    X = torch.from_numpy(inputs.random_matrix(M, nb, prec, seed=11)).to(dev)
    Y = torch.from_numpy(inputs.random_matrix(M, nb, prec, seed=12)).to(dev)
    C = torch.from_numpy(inputs.random_matrix(M, M, prec, seed=13)).to(dev)
    work = torch.empty(8 * m_l * 8 * M * M, dtype=torch.uint8, device=dev)
    for _ in range(warmup):
        mdls.gemm(prec, X, Y, C=C, trans_b=True, mode=1, work=work)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        mdls.gemm(prec, X, Y, C=C, trans_b=True, mode=1, work=work)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    pairs = M * M * nb
    ops = pairs * OPS_PER_PAIR[prec]
    achieved = ops / (ms * 1e-3) / 1e12
    return {"ms": round(ms, 5), "ops": ops, "achieved": round(achieved, 3), "frac": round(achieved / FP64_PIPE_TOPS, 4),
            "bytes": 8 * m_l * (2 * M * nb + 2 * M * M)}


def run_ours(args, ws, rank, local):
    import numpy as np
    import torch

    import paper_2110_08375_b200 as mdls

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if ws > 1:
            import torch.distributed as dist

            dist.barrier()

    def max_over_ranks(v):
        if ws == 1:
            return v
        import torch.distributed as dist

        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    prec, M, K, nb = WORKLOADS[args.workload]
    if args.workload == "cfg5b":
        return run_batch_workload(args, ws, rank, dev, barrier, max_over_ranks)
    if args.workload == "cfg5a":
        return run_sharded_workload(args, ws, rank, dev, barrier, max_over_ranks)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    def measure(prec, M, K, nb, steps, warmup, seed, with_e2e, with_trace, sampler=None):
        A_h, b_h = make_problem(prec, M, K, seed)
        A = torch.from_numpy(A_h).to(dev)
        b = torch.from_numpy(b_h).to(dev)
        stream = torch.cuda.current_stream()
        # the solve as a library plan (mdls_lstsq_plan: the whole launch sequence captured once into a
        # library-owned CUDA graph, replayed by one mdls_plan_launch per step); --no-graph: direct calls
        plan = None
        if not args.no_graph:
            plan = mdls.LstsqPlan(prec, M, K, nb, form_q=True, device=dev)
            plan.A.copy_(A)
            plan.b.copy_(b)
            work = plan.work
        else:
            work = torch.empty(mdls.workspace_bytes(prec, 2, M, K, nb), dtype=torch.uint8, device=dev)

        def step():
            if plan is not None:
                plan.run()
                return plan.info
            return mdls.lstsq(prec, A, b, nb, form_q=True, work=work).info

        for _ in range(warmup):
            info = step()
        torch.cuda.synchronize()
        assert int(info.item()) == 0, f"dev_info={int(info.item())}"
        n0 = mdls.launch_count()
        step()
        torch.cuda.synchronize()
        per_step_launches = mdls.launch_count() - n0
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        barrier()
        torch.cuda.synchronize()
        ctx = sampler if sampler is not None else _Null()
        with ctx:
            for i in range(steps):
                flush.fill_(float(i))  # L2 flush between timed steps (untimed)
                ev[i][0].record(stream)
                step()
                ev[i][1].record(stream)
            torch.cuda.synchronize()
        barrier()
        ms = [a.elapsed_time(bb) for a, bb in ev]
        ms_step = max_over_ranks(sum(ms) / steps)
        out = {"ms_per_step": ms_step, "ms_min": min(ms), "launches_per_step": per_step_launches}
        if with_e2e:  # through the public API from pinned host buffers (mdls_lstsq_host plan), copies timed
            A_p = torch.from_numpy(A_h).pin_memory()
            b_p = torch.from_numpy(b_h).pin_memory()
            x_p = torch.empty((A_h.shape[0], K), dtype=torch.float64).pin_memory()
            if plan is None:
                A_d, b_d = torch.empty_like(A), torch.empty_like(b)
            else:  # mdls_lstsq_host_plan: the copies are inside the library graph, A's panels overlap the QR
                hplan = mdls.HostLstsqPlan(prec, M, K, nb, form_q=True, device=dev, A=A_p, b=b_p, x=x_p)

            def e2e_step():
                if plan is not None:
                    hplan.run()
                    return hplan.info
                A_d.copy_(A_p, non_blocking=True)
                b_d.copy_(b_p, non_blocking=True)
                rr = mdls.lstsq(prec, A_d, b_d, nb, form_q=True, work=work)
                x_p.copy_(rr.x, non_blocking=True)
                return rr.info

            for _ in range(2):
                e2e_step()
            torch.cuda.synchronize()
            barrier()
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            for _ in range(steps):
                info = e2e_step()
            t1.record(stream)
            torch.cuda.synchronize()
            barrier()
            out["e2e_ms"] = max_over_ranks(t0.elapsed_time(t1) / steps)
            out["h2d"] = A_h.nbytes + b_h.nbytes
            out["d2h"] = x_p.numel() * 8
            # parity guard on the e2e result (cheap invariant: finite, dev_info 0)
            assert int(info.item()) == 0 and bool(np.isfinite(x_p.numpy()).all())
        if with_trace:  # second pass, traced launch by launch (per-stage and per-family kernel times)
            mdls.trace_enable(True)
            for i in range(steps):
                flush.fill_(float(i))
                mdls.lstsq(prec, A, b, nb, form_q=True, work=work)
            torch.cuda.synchronize()
            mdls.trace_enable(False)
            tr = mdls.trace_collect()
            out["trace"] = {k: ({s: v / steps for s, v in d.items()} if isinstance(d, dict) else d / steps)
                            for k, d in tr.items()}
        del plan
        return out

    sampler = ClockSampler(local)
    main = measure(prec, M, K, nb, args.steps, args.warmup, seed=rank, with_e2e=True, with_trace=True,
                   sampler=sampler)
    led = ledger_flops(prec, M, K, nb)
    flops = led["total_flops"]
    value = ws * flops / (main["ms_per_step"] * 1e-3) / 1e9  # GFLOP/s, whole job
    e2e_val = ws * flops / (main["e2e_ms"] * 1e-3) / 1e9
    tr = main["trace"]
    gemm_ms = tr["family_ms"]["gemm"]
    pairs = gemm_pairs(led)
    roof = gemm_roofline(dev, prec, M, nb)
    res = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "GFLOP/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(main["ms_per_step"], 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {
            "workload": f"{prec} least squares {M}x{K}, tile {nb} (QR + W/Y + trailing + Q + Q^T b + tiled BS)",
            "precision": prec, "M": M, "K": K, "nb": nb,
            "parallelism": f"batch{ws}" if ws > 1 else "single",
            "l2": f"flushed between timed steps ({L2_FLUSH_BYTES >> 20} MiB write, untimed)",
            "graph": "library plan (mdls_lstsq_plan: one CUDA graph replay per step)" if not args.no_graph else False,
            "flops_per_solve": flops,
        },
        "fp64_peak_frac": round(value / ws / (FP64_PEAK_TFLOPS * 1e3), 4),
        "fp64_peak_tflops": round(FP64_PEAK_TFLOPS, 2),
        # the same step measured in FP64-pipe instructions executed (every stage's md pairs at the GEMM kernels'
        # cost per pair, a lower bound: the panel's scalar chain and reductions execute more) against the
        # 18.6 T/s issue peak -- utilisation, as opposed to the Table-1 tally of "value"
        "fp64_pipe_frac_executed_lower_bound": round(step_fp64_ops(led, prec) / (main["ms_per_step"] * 1e-3)
                                                     / (FP64_PIPE_TOPS * 1e12), 4),
        "clocks": sampler.summary(),
        "e2e": {"value": round(e2e_val, 2), "unit": "GFLOP/s", "h2d_bytes_per_step": main["h2d"],
                "d2h_bytes_per_step": main["d2h"], "ms_per_step": round(main["e2e_ms"], 4)},
        "gpu_launches": int(main["launches_per_step"] * args.steps),
        "roofline": {
            "kernel": "gemm_kernel (md GEMM) at the solve's largest launch: Q(:, 0:) += X Y_1^T, "
                      f"{M} x {M} x {nb} (\"Q + QWY\", P:551-554; trailing update has the same form)",
            "bound": "alu",
            "achieved": roof["achieved"],
            "peak": round(FP64_PIPE_TOPS, 2),
            "unit": "TFLOP/s",
            "unit_note": "FP64-pipe lane operations (DADD/DMUL/DFMA each 1) per second; algorithmic ops = md pairs x "
                         f"{OPS_PER_PAIR[prec]} FP64 instructions per pair (md.cuh Acc); peak = 148 SMs x 64 lanes x "
                         "1.965 GHz (measured DADD 18.56 T/s, profiles/r01_fp64_peak.txt)",
            "frac": roof["frac"],
            "traffic": GEMM_NCU_TRAFFIC.get(prec),
            "algorithmic_ops_per_launch": roof["ops"],
            "algorithmic_bytes_per_launch": roof["bytes"],
            "launch_ms": roof["ms"],
            "measured": "CUDA events on the launching (current torch) stream around 20 back-to-back launches "
                        "through mdls_gemm after 3 warm-ups, inside bench.py",
            "gemm_ops_share_of_step": round(pairs * OPS_PER_PAIR[prec] / step_fp64_ops(led, prec), 4),
            "gemm_family_ms_traced": round(gemm_ms, 4),
            "note": "in the solve the GEMMs run on 3 streams concurrently with the leaf chain, so traced per-launch "
                    "times overlap; the roofline launch is timed alone",
        },
        "stages_ms": {k: round(v, 4) for k, v in tr["stages_ms"].items()},
        "family_ms": {k: round(v, 4) for k, v in tr["family_ms"].items()},
        "paper_context": {
            "V100_kernel_ms_T11": PAPER_V100_MS[prec],
            "speedup_vs_V100_kernel_time": round(PAPER_V100_MS[prec] / main["ms_per_step"], 1),
            "note": "paper GF rates use its own (~14x larger) tallies; compare time per solve",
        },
    }
    if not args.no_extra and args.workload == "cfg2":
        extra = {"dd": {"ms_per_solve": round(main["ms_per_step"], 4), "gflops": round(value / ws, 2)}}
        for p, steps in (("qd", max(2, min(args.steps, 5))), ("od", max(2, min(args.steps, 3)))):
            r = measure(p, M, K, nb, steps, 1, seed=rank, with_e2e=False, with_trace=False)
            f = ledger_flops(p, M, K, nb)["total_flops"]
            extra[p] = {"ms_per_solve": round(r["ms_per_step"], 3),
                        "gflops": round(f / (r["ms_per_step"] * 1e-3) / 1e9, 2),
                        "fp64_peak_frac": round(f / (r["ms_per_step"] * 1e-3) / 1e12 / FP64_PEAK_TFLOPS, 4),
                        "speedup_vs_V100_kernel_time": round(PAPER_V100_MS[p] / r["ms_per_step"], 1)}
        # plain double ("1d"): the paper lists its timings beside the md runs but does not compare them
        # (P:599-604); flops = the same ledger counts at one flop per operation
        r = measure("d", M, K, nb, max(3, min(args.steps, 10)), 1, seed=rank, with_e2e=False, with_trace=False)
        f = ledger_flops("d", M, K, nb)["total_flops"]
        extra["d"] = {"ms_per_solve": round(r["ms_per_step"], 4),
                      "gflops": round(f / (r["ms_per_step"] * 1e-3) / 1e9, 2),
                      "note": "plain double, same kernels with one limb; listed, not compared (P:599-604)"}
        res["precisions"] = extra
        res["overhead"] = {
            "dd_to_qd": round(extra["qd"]["ms_per_solve"] / extra["dd"]["ms_per_solve"], 2),
            "qd_to_od": round(extra["od"]["ms_per_solve"] / extra["qd"]["ms_per_solve"], 2),
            "predicted_T1": {"dd_to_qd": 11.7, "qd_to_od": 5.4},
        }
    if not args.no_extra and args.workload == "cfg2" and ws == 1:
        rb = bench_batch(dev, prec, M, K, nb, BATCH_CHUNK, args.groups, max(2, min(args.steps, 5)), 1, 0, 1,
                         lambda: None, lambda v: v, args.no_graph)
        fb = ledger_flops(prec, M, K, nb)["total_flops"] * BATCH_CHUNK
        vb = fb / (rb["ms_per_step"] * 1e-3) / 1e9
        res["batch_cfg5b_1gpu"] = {
            "workload": f"{BATCH_CHUNK} independent {prec} {M}x{K} solves, one mdls_lstsq_batched call, "
                        f"{rb['groups']} stream groups (config 5b's per-GPU unit)",
            "ms_per_batch": round(rb["ms_per_step"], 3), "ms_per_solve": round(rb["ms_per_solve_per_gpu"], 4),
            "gflops": round(vb, 2), "fp64_peak_frac": round(vb / (FP64_PEAK_TFLOPS * 1e3), 4)}
    if not args.no_extra and args.workload == "cfg2" and ws == 1:
        res["complex_t5"] = bench_complex(dev, "dd", 512, 64, max(3, min(args.steps, 10)))
    if not args.no_extra and args.workload == "cfg2":
        res["backsub_cfg4"] = bench_backsub(dev, "qd", 17920, 128, max(3, min(args.steps, 10)), 2, args.no_graph)
    if rank == 0 and ws == 1 and not args.no_cpu:
        res["cpu_baseline"] = cpu_baseline(prec, M, K, nb)
        # the oracle's rate counts the no-Q pipeline (it never forms Q): compare time per solve, not rates
        res["cpu_baseline"]["gpu_speedup_time_per_solve"] = round(
            res["cpu_baseline"]["seconds_per_solve"] / (main["ms_per_step"] * 1e-3), 1)
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(res), flush=True)


def run_batch_workload(args, ws, rank, dev, barrier, max_over_ranks):
    """--workload cfg5b: BASELINE config 5b, a batch of args.batch independent dd 1024 x 1024 solves sharded
    over the ranks (fixed total: strong scaling), no data-path collective."""
    prec, M, K, nb = WORKLOADS["cfg5b"]
    sampler = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    r = bench_batch(dev, prec, M, K, nb, args.batch, args.groups, args.steps, args.warmup, rank, ws, barrier,
                    max_over_ranks, args.no_graph, sampler=sampler, with_e2e=True)
    flops = ledger_flops(prec, M, K, nb)["total_flops"] * args.batch
    value = flops / (r["ms_per_step"] * 1e-3) / 1e9
    res = {
        "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(r["ms_per_step"], 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"batch of {args.batch} independent {prec} least squares {M}x{K}, tile {nb}, "
                               f"sharded over {ws} GPU(s) (mdls_lstsq_batched, {r['groups']} stream groups)",
                   "precision": prec, "M": M, "K": K, "nb": nb, "batch": args.batch,
                   "parallelism": f"batch-shard{ws}", "l2": "inputs exceed L2 (no flush)", "graph": not args.no_graph,
                   "flops_per_solve": flops / args.batch},
        "fp64_peak_frac": round(value / ws / (FP64_PEAK_TFLOPS * 1e3), 4),
        "fp64_peak_tflops": round(FP64_PEAK_TFLOPS, 2),
        "ms_per_solve_per_gpu": round(r["ms_per_solve_per_gpu"], 4),
        "clocks": sampler.summary(),
        "e2e": {"value": round(flops / (r["e2e_ms"] * 1e-3) / 1e9, 2), "unit": "GFLOP/s",
                "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": r["d2h"], "ms_per_step": round(r["e2e_ms"], 3)},
        "gpu_launches": int(r["launches_per_step"] * args.steps),
    }
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(res), flush=True)


def run_sharded_workload(args, ws, rank, dev, barrier, max_over_ranks):
    """--workload cfg5a: BASELINE config 5a, the block-column sharded QR + least squares (sharded.py) of an od
    M x M matrix (default 8192) over the ranks: panel k on rank k mod N, W_k / Y_k NCCL-broadcast from the owner
    (row-trimmed), look-ahead panel on a high-priority stream; fixed total work (strong scaling)."""
    import torch

    import paper_2110_08375_b200 as mdls
    from paper_2110_08375_b200 import inputs, sharded

    prec, M, K, nb = WORKLOADS["cfg5a"]
    if args.size:
        M = K = args.size
    st = sharded.plan(prec, M, K, nb, ws)
    A = inputs.random_matrix_torch(M, K, prec, seed=5, device=dev)  # every rank generates the same A ...
    b = inputs.random_vector_torch(M, prec, seed=5, device=dev)
    A_src = {rank: A[:, sharded.local_columns(st, rank), :].contiguous()}  # ... and keeps its own panels
    del A
    torch.cuda.empty_cache()
    comm = sharded.Comm() if ws > 1 else None
    ops = sharded.GpuOps()
    new = lambda shape: torch.zeros(shape, dtype=torch.float64, device=dev)  # noqa: E731

    def step():
        A_loc = {r: t.clone() for r, t in A_src.items()}
        return sharded.sharded_lstsq(prec, A_loc, b, M, K, nb, ws, ops, comm, new, sharded.Streams(dev))

    for _ in range(max(1, args.warmup)):
        x, F, y, info = step()
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    sampler = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    n0 = mdls.launch_count()
    with sampler:
        for i in range(args.steps):
            ev[i][0].record()
            x, F, y, info = step()
            ev[i][1].record()
        torch.cuda.synchronize()
    launches = mdls.launch_count() - n0
    barrier()
    ms = max_over_ranks(sum(a.elapsed_time(bb) for a, bb in ev) / args.steps)
    flops = ledger_flops(prec, M, K, nb)["total_flops"]
    value = flops / (ms * 1e-3) / 1e9
    res = {
        "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{prec} least squares {M}x{K}, tile {nb}, block-column sharded over {ws} GPU(s) "
                               "(sharded.py: panel k on rank k mod N, W/Y NCCL broadcast, look-ahead)",
                   "precision": prec, "M": M, "K": K, "nb": nb, "parallelism": f"colshard{ws}",
                   "l2": "operands exceed L2", "graph": False, "flops_per_solve": flops},
        "fp64_peak_frac": round(value / ws / (FP64_PEAK_TFLOPS * 1e3), 4),
        "clocks": sampler.summary(), "gpu_launches": int(launches),
    }
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(res), flush=True)


def bench_complex(dev, prec, n, nb, steps):
    """Row f2 / T5's complex shape: complex least squares n x n (mdls_zlstsq, the real embedding solved by the
    real pipeline), time per solve with CUDA events; flops = the ledger of the embedded 2n x 2n real solve."""
    import torch

    import paper_2110_08375_b200 as mdls
    from paper_2110_08375_b200 import inputs

    Are, bre = inputs.lstsq_problem(n, n, prec, 51)
    Aim, bim = inputs.lstsq_problem(n, n, prec, 52)
    t = [torch.from_numpy(a).to(dev) for a in (Are, Aim, bre, bim)]
    work = torch.empty(mdls.workspace_bytes(prec, 5, n, n, nb), dtype=torch.uint8, device=dev)
    for _ in range(2):
        mdls.zlstsq(prec, *t, nb, work=work)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        _, _, info = mdls.zlstsq(prec, *t, nb, work=work)
    e1.record()
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    ms = e0.elapsed_time(e1) / steps
    f = ledger_flops(prec, 2 * n, 2 * n, nb)["total_flops"]
    return {"workload": f"complex {prec} least squares {n}x{n}, tile {nb} (real embedding 2n x 2n, mdls_zlstsq)",
            "ms_per_solve": round(ms, 4), "embedded_gflops": round(f / (ms * 1e-3) / 1e9, 2),
            "paper_V100_complex_dd_512_ms_T5": "see BASELINE.md T5"}


def bench_backsub(dev, prec, n, nb, steps, warmup, no_graph):
    """BASELINE config 4: tiled back substitution alone (Algorithm 1), U from an LU (device generated)."""
    import torch

    import paper_2110_08375_b200 as mdls
    from paper_2110_08375_b200 import inputs

    U = inputs.lu_upper_torch(n, prec, seed=4, device=dev)
    y = inputs.random_vector_torch(n, prec, seed=4, device=dev)
    work = torch.empty(mdls.workspace_bytes(prec, 1, n, n, nb), dtype=torch.uint8, device=dev)
    x = torch.empty((U.shape[0], n), dtype=torch.float64, device=dev)
    info = torch.zeros(1, dtype=torch.int32, device=dev)
    import ctypes

    from paper_2110_08375_b200 import _lib

    fn = _lib.fn("mdls_backsub_", prec)

    def step():
        st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        rc = fn(n, nb, ctypes.c_void_p(U.data_ptr()), n, n * n, ctypes.c_void_p(y.data_ptr()), n,
                ctypes.c_void_p(x.data_ptr()), n, ctypes.c_void_p(work.data_ptr()), work.numel(),
                ctypes.c_void_p(info.data_ptr()), st)
        assert rc == 0

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    g = None
    if not no_graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in ev:  # U (n^2/2 x 32 B = 5.1 GB for qd 17,920) exceeds L2: no flush needed
        a.record()
        g.replay() if g is not None else step()
        b.record()
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev) / steps
    mdls.trace_enable(True)
    step()
    torch.cuda.synchronize()
    mdls.trace_enable(False)
    tr = mdls.trace_collect()
    c = mdls.counts(prec, 1, n, n, nb)
    flops = c["total_flops"]
    pairs_upd = c["stages"]["bsupdate"]["mul"]
    upd_ms = tr["stages_ms"]["bsupdate"]
    bytes_upd = pairs_upd * 8 * U.shape[0]  # each strictly-upper tile entry read once
    del U
    return {
        "workload": f"{prec} tiled back substitution, n={n}, {n // nb} tiles of {nb}",
        "ms_per_solve": round(ms, 4),
        "gflops": round(flops / (ms * 1e-3) / 1e9, 2),
        "fp64_peak_frac": round(flops / (ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS, 4),
        "stages_ms": {k: round(tr["stages_ms"][k], 4) for k in ("invert", "mulinv", "bsupdate")},
        "update_hbm_gbs": round(bytes_upd / (upd_ms * 1e-3) / 1e9, 1) if upd_ms > 0 else None,
        "update_fp64_tops": round(pairs_upd * OPS_PER_PAIR[prec] / (upd_ms * 1e-3) / 1e12, 3) if upd_ms else None,
        "paper_V100_kernel_ms": 237.1,
        "paper_V100_tiling": "80 x 224",
        "speedup_vs_V100_kernel_time": round(237.1 / ms, 1),
    }


def bench_batch(dev, prec, M, K, nb, total, groups, steps, warmup, rank, ws, barrier, max_over_ranks, no_graph,
                sampler=None, with_e2e=False):
    """Independent problems p = 0..total-1 (seed p), rank r solving its shard_range block with
    mdls_lstsq_batched plans (chunks of BATCH_CHUNK problems, one plan each)."""
    import numpy as np
    import torch

    import paper_2110_08375_b200 as mdls
    from paper_2110_08375_b200 import batch

    lo, hi = batch.shard_range(total, rank, ws)
    nloc = hi - lo
    G = max(1, min(groups, 16))
    chunks = [(c, min(nloc, c + BATCH_CHUNK)) for c in range(0, nloc, BATCH_CHUNK)]
    # one plan per chunk (mdls_lstsq_batched_plan: the chunk's solves captured into a library-owned CUDA graph);
    # each plan owns its chunk's A, b, x; problem p generated from seed p
    plans, A_h, b_h = [], [], []
    for c0, c1 in chunks:
        probs = [make_problem(prec, M, K, lo + p) for p in range(c0, c1)]
        ah = np.stack([a for a, _ in probs])
        bh = np.stack([bb for _, bb in probs])
        del probs
        pl = mdls.BatchedLstsqPlan(prec, c1 - c0, M, K, nb, form_q=True, groups=G, device=dev)
        pl.A.copy_(torch.from_numpy(ah))
        pl.b.copy_(torch.from_numpy(bh))
        plans.append(pl)
        if with_e2e:
            A_h.append(torch.from_numpy(ah).pin_memory())
            b_h.append(torch.from_numpy(bh).pin_memory())
    launches = sum(pl.launches for pl in plans)

    def step():
        for pl in plans:
            pl.run()

    for _ in range(max(1, warmup)):
        step()
    torch.cuda.synchronize()
    for pl in plans:
        assert int(pl.info.abs().sum()) == 0
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    barrier()
    torch.cuda.synchronize()
    with (sampler if sampler is not None else _Null()):
        for i in range(steps):
            ev[i][0].record(stream)
            step()  # inputs (16.8 MB per problem x problems per rank) exceed L2: no flush needed
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = max_over_ranks(sum(a.elapsed_time(bb) for a, bb in ev) / steps)
    out = {"ms_per_step": ms, "problems_total": total, "problems_per_rank_max": -(-total // ws), "groups": G,
           "launches_per_step": launches, "ms_per_solve_per_gpu": ms / max(1, -(-total // ws))}
    if with_e2e:  # public API from pinned host buffers: inputs copied in, plan replayed, solutions copied out
        x_p = [torch.empty(tuple(pl.x.shape), dtype=torch.float64).pin_memory() for pl in plans]

        def e2e_step():
            for pl, ah, bh, xp in zip(plans, A_h, b_h, x_p):
                xp.copy_(pl.solve(ah, bh), non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(steps):
            e2e_step()
        t1.record(stream)
        torch.cuda.synchronize()
        barrier()
        out["e2e_ms"] = max_over_ranks(t0.elapsed_time(t1) / steps)
        out["h2d"] = sum(t.numel() * 8 for t in A_h + b_h)
        out["d2h"] = sum(t.numel() * 8 for t in x_p)
        assert all(bool(torch.isfinite(t).all()) for t in x_p)
    del plans
    torch.cuda.empty_cache()
    return out


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def cpu_baseline(prec, M, K, nb, repeats=1):
    """The oracle (plain C, threads over independent columns) on the host cores."""
    import oracle

    oracle.build()
    cores = oracle.default_threads()
    A, b = make_problem(prec, M, K, 0)
    t0 = time.perf_counter()
    for _ in range(repeats):
        oracle.lstsq(prec, A, b, nthreads=cores)
    dt = (time.perf_counter() - t0) / repeats
    flops = ledger_flops(prec, M, K, nb, form_q=False)["total_flops"]
    return {"value": round(flops / dt / 1e9, 4), "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
            "sample": f"{repeats} full {prec} {M}x{K} least-squares solve(s) (unblocked Householder QR, "
                      f"Q^T b by reflectors, back substitution); flops = ledger count of the no-Q pipeline",
            "seconds_per_solve": round(dt, 3)}


def run_reference(args, ws, rank, local):
    """--impl reference: the oracle as it stands, on the host cores (rank 0 only)."""
    if rank != 0:
        return
    import oracle

    prec, M, K, nb = WORKLOADS[args.workload]
    oracle.build()
    cores = oracle.default_threads()
    A, b = make_problem(prec, M, K, 0)
    for _ in range(args.warmup):
        oracle.lstsq(prec, A, b, nthreads=cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.lstsq(prec, A, b, nthreads=cores)
    dt = (time.perf_counter() - t0) / args.steps
    flops = ledger_flops(prec, M, K, nb, form_q=False)["total_flops"]
    v = round(flops / dt / 1e9, 4)
    res = {
        "metric": METRIC, "value": v, "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{prec} least squares {M}x{K}, tile {nb} (oracle: unblocked QR + Q^T b + BS)",
                   "precision": prec, "M": M, "K": K, "nb": nb},
        "impl": "reference",
        "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
                         "sample": f"each step one full {prec} {M}x{K} solve"},
        "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(res), flush=True)


def main():
    args = parse()
    ws, rank, local = dist_env()
    if args.gpus != ws and ws > 1:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {ws}", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, ws, rank, local)
    else:
        run_ours(args, ws, rank, local)


if __name__ == "__main__":
    main()
