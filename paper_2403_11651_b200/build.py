"""Build libccrd.so in-tree with nvcc for sm_100a (no JIT cache, no torch
extension machinery: a plain shared library with a C ABI)."""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libccrd.so")
SOURCES = ["arm_rate.cu", "arm_tc.cu", "arm_decode.cu", "pyramid.cu", "synth.cu", "train.cu", "analysis.cu", "analysis_tc.cu", "ccrd_api.cu"]
HEADERS = ["ccrd_common.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         f"-I{os.path.join(ROOT, 'include')}"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str = None) -> str:
    """Compile csrc/*.cu into libccrd.so.  ``defines``/``out`` build an
    experiment variant (extra -D flags) into another file (tools/ only)."""
    lib = out or LIB
    objdir = os.path.join(HERE, "build" if not defines else "build_" + "_".join(d.replace("=", "") for d in defines))
    os.makedirs(objdir, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "ccrd.h")]
    jobs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(objdir, s.replace(".cu", ".o"))
        if force or _stale(obj, [src] + hdrs):
            jobs.append((src, obj))

    def compile_one(j):
        src, obj = j
        cmd = [NVCC] + ARCH + FLAGS + [f"-D{d}" for d in defines] + ["-c", src, "-o", obj + ".tmp"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
        os.replace(obj + ".tmp", obj)
        log = os.path.join(objdir, os.path.basename(src) + ".ptxas.log")
        with open(log, "w") as f:
            f.write(r.stderr)
        return src

    with ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        for s in ex.map(compile_one, jobs):
            if verbose:
                print("compiled", s, file=sys.stderr)
    objs = [os.path.join(objdir, s.replace(".cu", ".o")) for s in SOURCES]
    if force or jobs or _stale(lib, objs):
        tmp = lib + f".{os.getpid()}.tmp"
        subprocess.check_call([NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-lcudart", "-lcublasLt"])
        os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose=True, defines=defs, out=outs[0] if outs else None))
