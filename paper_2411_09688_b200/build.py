"""Build libsqz.so (sm_100a) in-tree with nvcc.  Used by __graft_entry__.build()."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libsqz.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-v", "-I", os.path.join(ROOT, "include")]
FLAGS += os.environ.get("SQZ_NVCC_EXTRA", "").split()  # tuning experiments only


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stamp() -> str:
    """Hash of every source, header and flag that goes into libsqz.so."""
    import hashlib

    h = hashlib.sha256()
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
    deps += glob.glob(os.path.join(ROOT, "include", "*.h"))
    for f in sorted(deps):
        h.update(os.path.relpath(f, ROOT).encode())
        h.update(open(f, "rb").read())
    h.update(" ".join([NVCC, *ARCH, *FLAGS]).encode())
    return h.hexdigest()


STAMP = OUT + ".sha256"


def needs_build() -> bool:
    """Rebuild unless libsqz.so exists AND was built from exactly these sources
    and flags (content hash, not modification times: a copied-in or stale
    binary is never reused)."""
    if not os.path.exists(OUT) or not os.path.exists(STAMP):
        return True
    return open(STAMP).read().strip() != _stamp()


def build(force: bool = False, verbose: bool = False, jobs: int = 8) -> str:
    if not force and not needs_build():
        return OUT
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    procs = []
    objs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
        log = open(obj + ".log", "w")
        procs.append((subprocess.Popen(cmd, stdout=log, stderr=subprocess.STDOUT), obj, cmd))
    bad = []
    for p, obj, cmd in procs:
        if p.wait() != 0:
            bad.append(obj)
    if bad:
        msg = "".join(open(o + ".log").read() for o in bad)
        raise RuntimeError("nvcc failed:\n" + msg[-6000:])
    if verbose:
        for o in objs:
            sys.stdout.write(open(o + ".log").read())
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", OUT, *objs])
    with open(STAMP, "w") as f:
        f.write(_stamp())
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
