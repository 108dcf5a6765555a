"""Build the in-tree CUDA library `lib/libqcldpc_b200.so` for sm_100a.

    python -m paper_1204_0334_b200.build          # or __graft_entry__.build()

Each csrc/*.cu is compiled to an object in parallel, then linked with nvcc.
`-fmad=false` pins the floating-point operation sequence (no implicit FMA
contraction), so every lane runs the same instruction stream regardless of
gamma or kernel variant; the fused multiply-adds that are wanted are written
explicitly (fmaf).
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "lib")
LIB = os.path.join(OUT_DIR, "libqcldpc_b200.so")
SOURCES = ["plan.cu", "block.cu", "vnu.cu", "cnu_dc4.cu", "cnu_dc8.cu", "cnu_dc16.cu", "cnu_dc24.cu",
           "cnu_dc32.cu", "recycle.cu", "block64.cu", "channel.cu", "stream.cu",
           "host_pipe.cu", "agg.cu", "es_compact.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-fvisibility=hidden"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build the CUDA library")


def _stale(obj: str, deps) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, defines=(), lib: str = LIB) -> str:
    """Compile into `lib`; `defines` (e.g. ["-DAGG_VAR_MINB=1"]) build an A/B
    variant into its own object directory."""
    nvcc = _nvcc()
    tag = "".join(d.strip("-D").replace("=", "") for d in defines)
    obj_dir = os.path.join(OUT_DIR, "obj" + (("_" + tag) if tag else ""))
    os.makedirs(obj_dir, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(os.path.dirname(HERE), "include", "qcldpc_b200.h"))
    jobs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(obj_dir, src.replace(".cu", ".o"))
        if force or _stale(o, [s] + headers):
            jobs.append([nvcc, *ARCH, *FLAGS, *defines, "-c", s, "-o", o])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)

    with cf.ThreadPoolExecutor(max_workers=max(1, len(jobs))) as ex:
        list(ex.map(run, jobs))
    objs = [os.path.join(obj_dir, s.replace(".cu", ".o")) for s in SOURCES]
    if force or jobs or _stale(lib, objs):
        os.makedirs(os.path.dirname(lib), exist_ok=True)
        tmp = lib + ".tmp"
        run([nvcc, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"])
        os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
