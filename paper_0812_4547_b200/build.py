"""Build the in-tree C-ABI library ``libsrht.so`` for sm_100a with nvcc.

``python -m paper_0812_4547_b200.build`` (or ``__graft_entry__.build()``).
Objects go to ``build/``; the shared library lands next to this file so it
travels with the repo snapshot to the GPU box.
"""

import concurrent.futures
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libsrht.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v",
         "-I" + os.path.join(ROOT, "include")]
SOURCES = ["plan.cu", "sketch.cu", "sketch_ws.cu", "sketch_tma.cu", "sketch_f64.cu", "sketch_tma64.cu", "gram.cu", "nnls.cu", "subspace.cu", "api.cu"]


def _compile(src, verbose):
    out = os.path.join(OBJ, os.path.splitext(src)[0] + ".o")
    dep_mtime = max(os.path.getmtime(os.path.join(CSRC, f)) for f in os.listdir(CSRC))
    dep_mtime = max(dep_mtime, os.path.getmtime(os.path.join(ROOT, "include", "srht.h")))
    if os.path.exists(out) and os.path.getmtime(out) >= dep_mtime:
        return out, ""
    cmd = [NVCC] + ARCH + FLAGS + ["-c", os.path.join(CSRC, src), "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed for %s:\n%s\n%s" % (src, r.stdout, r.stderr))
    return out, r.stderr if verbose else ""


def build_debug():
    """Experiment build (scripts/ws_experiments.py): libsrht_dbg.so with kernel knock-outs."""
    os.makedirs(OBJ, exist_ok=True)
    out = os.path.join(PKG, "libsrht_dbg.so")
    objs = []
    for src in SOURCES:
        o = os.path.join(OBJ, "dbg_" + os.path.splitext(src)[0] + ".o")
        cmd = [NVCC] + ARCH + FLAGS + ["-DSRHT_WS_DEBUG", "-c", os.path.join(CSRC, src), "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(r.stderr)
        objs.append(o)
    r = subprocess.run([NVCC] + ARCH + ["-shared", "-o", out] + objs + ["-lcudart_static", "-lrt", "-ldl", "-lpthread"],
                       capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(r.stderr)
    return out


def build_variant(name, defines):
    """Experiment build: lib<name>.so with extra -D defines (A/B runs via SRHT_LIB=lib<name>.so)."""
    os.makedirs(OBJ, exist_ok=True)
    out = os.path.join(PKG, "lib%s.so" % name)
    objs = []
    for src in SOURCES:
        o = os.path.join(OBJ, "%s_%s.o" % (name, os.path.splitext(src)[0]))
        cmd = [NVCC] + ARCH + FLAGS + ["-D" + d for d in defines] + ["-c", os.path.join(CSRC, src), "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(r.stderr)
        objs.append(o)
    r = subprocess.run([NVCC] + ARCH + ["-shared", "-o", out] + objs + ["-lcudart_static", "-lrt", "-ldl", "-lpthread"],
                       capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(r.stderr)
    return out


def build(verbose=False, force=False):
    os.makedirs(OBJ, exist_ok=True)
    if force:
        for f in os.listdir(OBJ):
            os.remove(os.path.join(OBJ, f))
    with concurrent.futures.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log:
                sys.stderr.write(log)
    if not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("link failed:\n%s\n%s" % (r.stdout, r.stderr))
    return LIB


if __name__ == "__main__":
    if "--debug" in sys.argv:
        print(build_debug())
    else:
        print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
