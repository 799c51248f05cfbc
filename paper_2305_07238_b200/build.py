"""Builds libmcg.so in-tree (paper_2305_07238_b200/_lib/) for sm_100a.

Host translation units are compiled like the reference (C++20, -O2,
-ffp-contract=off; proj/CMakeLists.txt:16). Device translation units use
nvcc with ``-gencode arch=compute_100a,code=sm_100a --fmad=false``: the
descriptor pipeline (footprint, mip level, texel indices) and every value the
cache stores must be bit-identical to the host's IEEE evaluation, so no
multiply-add contraction is allowed anywhere on the path. CUDA runtime is
linked statically so the library does not depend on torch's libcudart.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import site
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
OBJ_DIR = os.path.join(OUT_DIR, "obj")
LIB = os.path.join(OUT_DIR, "libmcg.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# The system compiler explicitly (not $CXX): its libstdc++ is the one the
# Python process has loaded.
CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; libmcg needs the CUDA 12.9 toolchain")


def json_include() -> str:
    """Directory holding nlohmann/json.hpp (3.11.3 ships in the image)."""
    cands = []
    for sp in site.getsitepackages() + [site.getusersitepackages()]:
        cands.append(os.path.join(sp, "include", "cudnn_frontend", "thirdparty"))
    cands += ["/usr/include", "/usr/local/include"]
    for c in cands:
        if os.path.exists(os.path.join(c, "nlohmann", "json.hpp")):
            return c
    raise RuntimeError("nlohmann/json.hpp not found")


def _sources():
    cpp = sorted(glob.glob(os.path.join(CSRC, "*.cpp")))
    cu = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    headers = sorted(glob.glob(os.path.join(CSRC, "*.h*")) + glob.glob(os.path.join(CSRC, "*.cuh")))
    headers.append(os.path.join(ROOT, "include", "mcg.h"))
    return cpp, cu, headers


def _stale(obj: str, deps: list[str]) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str]) -> str:
    p = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{p.stdout}")
    return p.stdout


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ_DIR, exist_ok=True)
    nvcc = _nvcc()
    jinc = json_include()
    cpp, cu, headers = _sources()
    jobs = []
    for src in cpp:
        obj = os.path.join(OBJ_DIR, os.path.basename(src) + ".o")
        cmd = [CXX, "-std=c++20", "-O2", "-ffp-contract=off", "-fPIC", "-g0", "-Wall",
               "-I" + jinc, "-I" + os.path.join(ROOT, "include"), "-c", src, "-o", obj]
        jobs.append((obj, [src] + headers, cmd))
    for src in cu:
        obj = os.path.join(OBJ_DIR, os.path.basename(src) + ".o")
        cmd = [nvcc, "-ccbin", CXX, *ARCH, "-std=c++17", "-O3", "-lineinfo", "--fmad=false",
               "-Xptxas", "-v", "-Xcompiler", "-fPIC,-ffp-contract=off",
               "-I" + os.path.join(ROOT, "include"), "-c", src, "-o", obj]
        jobs.append((obj, [src] + headers, cmd))
    todo = [(o, c) for o, d, c in jobs if force or _stale(o, d)]
    logs = {}
    if todo:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(todo))) as ex:
            futs = {ex.submit(_run, c): o for o, c in todo}
            for f in cf.as_completed(futs):
                logs[futs[f]] = f.result()
    objs = [o for o, _, _ in jobs]
    if force or todo or _stale(LIB, objs):
        _run([nvcc, "-ccbin", CXX, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs,
              "-Xcompiler", "-fPIC", "-lpthread", "-ldl"])
        with open(os.path.join(OUT_DIR, "ptxas.log"), "w") as f:
            for o in sorted(logs):
                f.write(f"==== {os.path.basename(o)}\n{logs[o]}\n")
    if verbose:
        for o in sorted(logs):
            print(logs[o])
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
