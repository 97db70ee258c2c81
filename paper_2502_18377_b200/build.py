"""Build libmpde.so (sm_100a) in-tree with nvcc.  Used by __graft_entry__.build()."""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = [os.path.join(HERE, "csrc", f) for f in ("kernels.cu", "schur.cu", "dense.cu", "template.cu", "fgmres.cu", "march.cu", "slab.cu", "mpde.cu")]
DEPS = SRC + [os.path.join(HERE, "csrc", f) for f in ("common.cuh", "internal.h")] + [
    os.path.join(os.path.dirname(HERE), "include", "mpde.h")]
OUT = os.path.join(HERE, "libmpde.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"]


def stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(f) > t for f in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        # one translation unit per nvcc process (no cross-file device symbols), then link;
        # an object is rebuilt when its source or a shared header is newer (or force)
        hdr = max(os.path.getmtime(f) for f in DEPS if f not in SRC)
        objs = [os.path.join(HERE, "csrc", os.path.basename(f)[:-3] + ".o") for f in SRC]
        cmds = [[NVCC] + FLAGS + ["-c", f, "-o", o] for f, o in zip(SRC, objs)
                if force or not os.path.exists(o)
                or os.path.getmtime(o) < max(hdr, os.path.getmtime(f))]
        if verbose:
            for c in cmds:
                print(" ".join(c), file=sys.stderr)
        if cmds:
            with ThreadPoolExecutor(len(cmds)) as ex:
                for r in ex.map(lambda c: subprocess.run(c), cmds):
                    if r.returncode:
                        raise subprocess.CalledProcessError(r.returncode, r.args)
        subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared"] + objs
                       + ["-o", OUT + ".tmp"], check=True)
        os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
