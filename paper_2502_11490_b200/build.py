"""Build libgmpgr.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels with the repo)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgmpgr.so")
# one translation unit per kernel family, compiled in parallel, then linked
SOURCES = ["gmpgr.cu", "inst_duo.cu", "inst_mq.cu", "inst_search.cu", "hnsw_build.cpp"]
OBJ = os.path.join(HERE, "_obj")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
    # host code (hnsw_build.cpp) must keep separately rounded mul/add like the reference's
    # compiled Cython and numpy loops: no FMA contraction
    "-Xcompiler", "-ffp-contract=off",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    import glob

    deps = [os.path.join(CSRC, f) for f in SOURCES] + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
    deps.append(os.path.join(os.path.dirname(HERE), "include", "gmpgr.h"))
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    nvcc = os.environ.get("NVCC", "nvcc")
    os.makedirs(OBJ, exist_ok=True)

    def obj_stale(obj):
        # the object is current when it is newer than every file its .d dependency list names
        dep = obj[:-2] + ".d"
        if force or not (os.path.exists(obj) and os.path.exists(dep)):
            return True
        t = os.path.getmtime(obj)
        files = open(dep).read().replace("\\\n", " ").split(":", 1)[-1].split()
        return any(not os.path.exists(f) or os.path.getmtime(f) > t for f in files)

    def compile_one(src):
        obj = os.path.join(OBJ, os.path.splitext(src)[0] + ".o")
        if not obj_stale(obj):
            return obj, subprocess.CompletedProcess([], 0, "", "")
        cmd = [nvcc, *NVCC_FLAGS, "-MD", "-MF", obj[:-2] + ".d", "-c", "-o", obj, os.path.join(CSRC, src)]
        return obj, subprocess.run(cmd, capture_output=True, text=True)

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    report = ""
    for obj, res in results:
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc failed building {os.path.basename(obj)}")
        log = obj[:-2] + ".log"
        if res.args:  # compiled now: keep its ptxas report beside the object
            with open(log, "w") as f:
                f.write(res.stderr)
        if os.path.exists(log):
            report += open(log).read()
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
           "-o", LIB + ".tmp", *[obj for obj, _ in results]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed linking libgmpgr.so")
    if verbose:
        sys.stderr.write(report)
    os.replace(LIB + ".tmp", LIB)
    with open(os.path.join(HERE, "ptxas_report.txt"), "w") as f:
        f.write(report)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
