"""Build libvoxcap.so in-tree: nvcc for sm_100a, one object per .cu, linked shared.

    python -m paper_2004_02609_b200.build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
OUT = os.path.join(HERE, "libvoxcap.so")
BUILD = os.path.join(HERE, "_build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-std=c++17", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr", "-I", INCLUDE]


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _digest():
    h = hashlib.sha256()
    for f in sorted(os.listdir(CSRC)) + ["../../include/voxcap.h"]:
        p = os.path.join(CSRC, f)
        if os.path.isfile(p):
            h.update(f.encode())
            h.update(open(p, "rb").read())
    h.update(" ".join(FLAGS).encode())
    return h.hexdigest()


def build(force=False, verbose=False):
    """Compile every .cu for sm_100a and link libvoxcap.so (skipped if sources unchanged)."""
    os.makedirs(BUILD, exist_ok=True)
    stamp = os.path.join(BUILD, "digest")
    dig = _digest()
    if not force and os.path.exists(OUT) and os.path.exists(stamp) and open(stamp).read() == dig:
        return OUT

    # per-object digest: a .cu is recompiled when it, any header or the flags changed
    hdr = hashlib.sha256()
    for f in sorted(os.listdir(CSRC)) + ["../../include/voxcap.h"]:
        if not f.endswith(".cu") and os.path.isfile(os.path.join(CSRC, f)):
            hdr.update(f.encode())
            hdr.update(open(os.path.join(CSRC, f), "rb").read())
    hdr.update(" ".join(FLAGS).encode())

    def comp(src):
        obj = os.path.join(BUILD, src[:-3] + ".o")
        od = hashlib.sha256(hdr.digest() + open(os.path.join(CSRC, src), "rb").read()).hexdigest()
        ostamp = obj + ".digest"
        if not force and os.path.exists(obj) and os.path.exists(ostamp) and open(ostamp).read() == od:
            return obj
        cmd = [NVCC, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-6000:]}")
        with open(os.path.join(BUILD, src[:-3] + ".ptxas.log"), "w") as fh:
            fh.write(r.stderr)
        with open(ostamp, "w") as fh:
            fh.write(od)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(comp, _sources()))
    tmp = OUT + f".{os.getpid()}.tmp"
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp, *objs,
           "-lcudart", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    os.replace(tmp, OUT)
    with open(stamp, "w") as fh:
        fh.write(dig)
    if verbose:
        print("built", OUT)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
