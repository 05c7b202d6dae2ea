"""Build the sm_100a C-ABI library in-tree: paper_2501_01676_b200/_bddc_b200.so.

    python -m paper_2501_01676_b200.build

nvcc compiles every csrc/*.cu for -gencode arch=compute_100a,code=sm_100a with
-lineinfo (ncu source mapping) and links one shared object; no torch headers
are involved (the ABI is plain pointers + cudaStream_t).
"""

import fcntl
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_bddc_b200.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-I", INCLUDE]


def _fresh(target, deps):
    return os.path.exists(target) and os.path.getmtime(target) >= max(os.path.getmtime(d) for d in deps)


def build(force=False, verbose=False, defines=(), out=None):
    """Compile csrc/*.cu into OUT (or `out`), optionally with -D defines
    (tuning variants for tools/bench_tile.py).  Concurrent callers (one
    process per GPU) serialise on a file lock; the header the ctypes
    binding parses is a dependency too."""
    target = out or OUT
    sources = sorted(glob.glob(os.path.join(SRC, "*.cu")))
    deps = (sources + glob.glob(os.path.join(SRC, "*.cuh")) + glob.glob(os.path.join(SRC, "*.h"))
            + [os.path.join(INCLUDE, "bddc_b200.h")])
    if not force and not defines and _fresh(target, deps):
        return target
    with open(os.path.join(HERE, ".build.lock"), "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        if not force and not defines and _fresh(target, deps):
            return target  # another process built it while we waited
        return _compile(target, sources, verbose, defines)


def _compile(target, sources, verbose, defines):
    objdir = os.path.join(HERE, "build" if not defines else "build_" + "_".join(d.replace("=", "") for d in defines))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for s in sources:
        o = os.path.join(objdir, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        cmd = [NVCC, *FLAGS, *["-D" + d for d in defines], "-c", s, "-o", o]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((s, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for s, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {s}:\n{out.decode()}")
        if verbose and out:
            sys.stdout.write(out.decode())
    tmp = target + ".tmp"
    subprocess.check_call([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
                           *objs, "-o", tmp, "-lcudart"])
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
