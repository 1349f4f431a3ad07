"""Build librii_b200.so (sm_100a only) in-tree with nvcc.

    python -m paper_1808_03969_b200.build [--force] [--verbose] [--checked]

--checked builds librii_b200_checked.so (objects in build_obj_checked/) with
-DRII_BOUNDS_CHECK: device-side index and shared-memory layout assertions and a
device synchronisation after every launch (common.cuh RII_DCHECK), loaded by the
binding when RII_LIB=checked.  It stands in for compute-sanitizer, which the GPU
pool does not run.

Every translation unit is compiled with -gencode arch=compute_100a,code=sm_100a,
-lineinfo (ncu source view) and --fmad=false (the canonical fp32 arithmetic of
DESIGN.md CA1/CA2 must not be contracted into FMAs).  The CUDA runtime is linked
statically; NCCL is dlopen'ed at run time (csrc/comm.cpp).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build_obj")
LIB = os.path.join(HERE, "librii_b200.so")
OBJ_CHECKED = os.path.join(HERE, "build_obj_checked")
LIB_CHECKED = os.path.join(HERE, "librii_b200_checked.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--fmad=false", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include")]
# No -split-compile: it parallelises a unit's NVVM / ptxas work (k_scan.cu 198 s -> 59 s) but the code
# it produced for the headline u6 scan loop varied from build to build (a 17 % slower register
# allocation was observed).  Units compile in parallel with each other instead.
SPLIT = {"default": []}
# (source, extra defines, object): k_scan.cu is compiled once for its common code and once per M
# for the scan kernels of that M (its translation units then build in parallel)
SOURCES = [("capi.cu", [], "capi.cu.o"), ("k_scan.cu", [], "k_scan.cu.o")] + \
          [("k_scan.cu", [f"-DRII_SCAN_M={m}"], f"k_scan_m{m}.o") for m in (4, 8, 16, 32, 64)] + \
          [(f, [], f + ".o") for f in ("k_ivf.cu", "k_build.cu", "k_opq.cu", "k_large.cu", "k_large_u6.cu", "sort.cu", "comm.cpp",
                                        "opq.cpp")]


def _headers_mtime():
    return max(os.path.getmtime(os.path.join(CSRC, f)) for f in os.listdir(CSRC)
               if f.endswith((".cuh", ".hpp", ".h"))) if os.path.isdir(CSRC) else 0.0


def _compile(entry, force: bool, verbose: bool, checked: bool = False) -> str:
    src, defines, objname = entry
    path = os.path.join(CSRC, src)
    obj = os.path.join(OBJ_CHECKED if checked else OBJ, objname)
    if checked:
        defines = [*defines, "-DRII_BOUNDS_CHECK"]
    newest = max(os.path.getmtime(path), _headers_mtime(), os.path.getmtime(os.path.join(ROOT, "include", "rii.h")))
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= newest:
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, *SPLIT.get(src, SPLIT["default"]), *defines, "-c", path, "-o", obj]
    if verbose:
        cmd[1:1] = ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose:
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    LIB = LIB_CHECKED if checked else globals()["LIB"]
    os.makedirs(OBJ_CHECKED if checked else OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, verbose, checked), SOURCES))
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-cudart", "static", "-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--checked", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.verbose, a.checked))
