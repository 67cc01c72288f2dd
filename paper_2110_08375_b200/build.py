"""Build libmdls.so in-tree for sm_100a (nvcc, no torch extension machinery).

Each precision is its own translation unit (api_dd.cu, api_qd.cu, api_od.cu)
so the three compile in parallel; ledger.cu holds the host-only ledger.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libmdls.so")
SOURCES = [f"{k}_{p}.cu" for p in ("od", "qd", "dd", "d") for k in ("panel", "leafsm", "gemm", "bs", "api")] + ["ledger.cu"]
HEADERS = ["md.cuh", "md_warp.cuh", "types.cuh", "launch.cuh", "kern_misc.cuh", "kern_gemm.cuh", "kern_leaf.cuh", "kern_bs.cuh",
           "solver.cuh", "api.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--fmad=false",            # no contraction anywhere: EFTs are written with explicit intrinsics
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-warn-spills",
]


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found")
    return cand


def _deps(path: str, seen: set | None = None) -> set:
    """the file and every quoted #include it reaches (recursively)"""
    seen = set() if seen is None else seen
    path = os.path.normpath(path)
    if path in seen or not os.path.exists(path):
        return seen
    seen.add(path)
    with open(path) as f:
        for line in f:
            line = line.strip()
            if line.startswith("#include \""):
                inc = line.split('"')[1]
                _deps(os.path.join(os.path.dirname(path), inc), seen)
    return seen


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in _deps(src))


def build(force: bool = False, verbose: bool = False, extra: list[str] | None = None) -> str:
    os.makedirs(BUILD, exist_ok=True)
    nvcc = _nvcc()
    jobs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, s.replace(".cu", ".o"))
        only = os.environ.get("MDLS_BUILD_ONLY")  # dev iteration: recompile one precision, link the rest as built
        if only and os.path.exists(obj) and not (s.endswith(f"_{only}.cu") or s == "ledger.cu"):
            continue
        if force or _stale(obj, src):
            cmd = [nvcc, *NVCC_FLAGS, *(extra or []), "-c", src, "-o", obj]
            if verbose:
                cmd += ["-Xptxas", "-v"]
            jobs.append((s, cmd))
    objs_all = [os.path.join(BUILD, s.replace(".cu", ".o")) for s in SOURCES]
    relink = bool(jobs) or not os.path.exists(LIB) or any(
        not os.path.exists(o) or os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs_all)

    def run(job):
        name, cmd = job
        p = subprocess.run(cmd, capture_output=True, text=True)
        return name, p.returncode, p.stdout + p.stderr

    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        for name, rc, out in ex.map(run, jobs):
            if rc != 0:
                raise RuntimeError(f"nvcc failed on {name}:\n{out}")
            if verbose and out.strip():
                print(out, file=sys.stderr)
    if relink:
        objs = [os.path.join(BUILD, s.replace(".cu", ".o")) for s in SOURCES]
        tmp = LIB + ".tmp"
        cmd = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp, *objs]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError("link failed:\n" + p.stdout + p.stderr)
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
