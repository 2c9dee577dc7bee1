"""Build libperks_stencil.so (sm_100a) in-tree with nvcc.

Each csrc/*.cu is compiled separately (in parallel) with
``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xptxas -v`` and linked into one
shared library next to this file.  ptxas spill reports are collected into
``build/ptxas_report.txt``; any spill fails the build (P:859-860 register discipline).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import re
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "libperks_stencil.so")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr",
         "-I", os.path.join(ROOT, "include")]


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)
            if f.endswith((".cuh", ".h"))] + [os.path.join(ROOT, "include", "perks", "perks_stencil.h")]


def _compile(src: str) -> tuple[str, str]:
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    dep_mtime = max(os.path.getmtime(d) for d in _deps() + [src])
    if os.path.exists(obj) and os.path.getmtime(obj) >= dep_mtime:
        log = obj + ".log"
        return obj, open(log).read() if os.path.exists(log) else ""
    cmd = [NVCC, *FLAGS, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    with open(obj + ".log", "w") as f:
        f.write(r.stderr)
    return obj, r.stderr


def _func_spill_report(report: str) -> dict:
    """{mangled function name: spill bytes} from the ptxas -v report."""
    out, cur = {}, None
    for ln in report.splitlines():
        m = re.search(r"Function properties for (\S+)", ln)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", ln)
        if m and cur and (int(m.group(1)) or int(m.group(2))):
            out[cur] = int(m.group(1)) + int(m.group(2))
    return out


def spills_in_plane_loops(obj: str, func: str) -> list:
    """Local-memory accesses (LDL/STL) of `func` that lie inside a hot loop: an innermost
    backward-branch range (of >= 32 instructions) of the main body (before the final EXIT; the
    mbarrier retry stubs follow it) that contains an mbarrier wait.  Spills of loop-invariant state in a prologue or
    in the per-step outer loop cost one access per unit/step and are tolerated; spills in the
    per-plane loop are not (P:859-860 register discipline).  Kernels without such a loop (the 2D
    kernels): every spill inside the time loop (a backward branch over >= 256 instructions)."""
    r = subprocess.run(["cuobjdump", "-sass", "-fun", func, obj], capture_output=True, text=True)
    ins = []
    for ln in r.stdout.splitlines():
        m = re.match(r"\s*/\*([0-9a-f]+)\*/\s+(.*?);", ln)
        if m:
            ins.append((int(m.group(1), 16), m.group(2)))
    if not ins:
        return ["<no SASS>"]
    end = max((a for a, t in ins if re.fullmatch(r"\s*EXIT\s*", t)), default=ins[-1][0])
    waits = [a for a, t in ins if "TRYWAIT" in t and a <= end]
    loops = []
    for a, t in ins:
        m = re.search(r"\bBRA(?:\.\S+)?\s+(?:\S+,\s*)?0x([0-9a-f]+)", t)
        if m and a <= end and int(m.group(1), 16) <= a:
            loops.append((int(m.group(1), 16), a))
    # (a wait's own spin loop — try_wait, timer read, compare — is a loop too: ignore tiny ones)
    hot = [lp for lp in loops if any(lp[0] <= w <= lp[1] for w in waits)
           and sum(1 for a, _ in ins if lp[0] <= a <= lp[1]) >= 32]
    spills = [hex(a) for a, t in ins if re.search(r"\b(LDL|STL)\b", t)]
    if not hot:  # no mbarrier-paced loop (2D kernels): any spill inside the time loop (a loop of
        # >= 256 instructions) counts; prologue / epilogue spills run once per launch
        big = [lp for lp in loops if sum(1 for a, _ in ins if lp[0] <= a <= lp[1]) >= 256]
        return [a for a in spills if any(lo <= int(a, 16) <= hi for lo, hi in big)]
    inner = [lp for lp in hot if not any(o != lp and lp[0] <= o[0] and o[1] <= lp[1] for o in hot)]
    return [a for a in spills if any(lo <= int(a, 16) <= hi for lo, hi in inner)]


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(_compile, srcs))
    objs = [o for o, _ in results]
    report = "".join(log for _, log in results)
    with open(os.path.join(BUILD, "ptxas_report.txt"), "w") as f:
        f.write(report)
    bad = []
    for (obj, log) in results:
        for fn, nbytes in _func_spill_report(log).items():
            hot = spills_in_plane_loops(obj, fn)
            if hot:
                bad.append(f"{fn}: {nbytes} spill bytes, {len(hot)} in the plane loop at {hot[:4]}")
    if bad and not os.environ.get("PERKS_ALLOW_SPILLS"):
        raise RuntimeError("register spills in a plane loop (P:860 discipline):\n" + "\n".join(bad[:20]))
    newest = max(os.path.getmtime(o) for o in objs)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp, *objs,
               "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)
    if verbose:
        print(report)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
