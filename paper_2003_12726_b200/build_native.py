"""Build libpxst_b200.so in-tree with nvcc for sm_100a.

Each ``csrc/*.cu`` compiles to an object in ``build/`` in parallel, then
links into ``paper_2003_12726_b200/libpxst_b200.so``.  Re-running only
rebuilds objects whose sources (or shared headers) changed.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.environ.get("PXST_BUILD_DIR", os.path.join(ROOT, "build", "pxst"))
LIB = os.environ.get("PXST_LIB_OUT", os.path.join(HERE, "libpxst_b200.so"))

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", INCLUDE, "-I", CSRC]
FLAGS += os.environ.get("PXST_NVCC_EXTRA", "").split()
# Per-file flags.  PXST_NVCC_FILE_FLAGS="a.cu=<flags>;b.cu=<flags>" replaces the
# table (variant builds, tools/variant.sh).
FILE_FLAGS = {
    # ptxas's register-usage level (default 5) at 0-3 gives the K3 kernels a
    # better allocation under their 128-register cap: config 3 K3 31.15 -> 30.5
    # ms, config 4 282.9 -> 278.8 ms (measured side by side, tools/variant_bench.sh).
    # The same level costs K2 6-14 % and the fixed-point pass ~8 %, so it is set
    # for this file only; levels 8-10 help K2's 1 x 17 kernel (-2.4 %) but cost
    # 13 x 13 up to 1 %: not taken.
    "trans_search.cu": ["-Xptxas", "--register-usage-level=3"],
}
if "PXST_NVCC_FILE_FLAGS" in os.environ:
    FILE_FLAGS = {k.strip(): v.split() for k, v in
                  (kv.split("=", 1) for kv in os.environ["PXST_NVCC_FILE_FLAGS"].split(";") if kv)}


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _headers_mtime() -> float:
    ts = [os.path.getmtime(os.path.join(CSRC, f)) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    ts += [os.path.getmtime(os.path.join(INCLUDE, f)) for f in os.listdir(INCLUDE)]
    return max(ts) if ts else 0.0


def build(verbose: bool = False, force: bool = False, ptxas_verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    nv = nvcc()
    hdr = _headers_mtime()
    jobs = []
    objs = []
    for src in _sources():
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src[:-3] + ".o")
        objs.append(o)
        if force or not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(s), hdr):
            cmd = [nv, *ARCH, *FLAGS, *FILE_FLAGS.get(src, []), "-c", s, "-o", o]
            if ptxas_verbose:
                cmd += ["-Xptxas", "-v"]
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, r

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        for cmd, r in ex.map(run, jobs):
            if verbose or ptxas_verbose or r.returncode:
                sys.stderr.write(r.stdout + r.stderr)
            if r.returncode:
                raise RuntimeError(f"nvcc failed: {' '.join(cmd)}")
    if jobs or not os.path.exists(LIB) or force:
        cmd = [nv, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
    return LIB


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv, ptxas_verbose="-v" in sys.argv)
    print(LIB)
