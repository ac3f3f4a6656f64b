"""Build libquapi.so in-tree with nvcc for sm_100a (host setup + kernels + C ABI).

Safe to call from several processes at once (e.g. every torchrun rank): the build takes an exclusive
file lock, compiles into a private temporary directory and installs the library with an atomic rename.
"""
from __future__ import annotations

import fcntl
import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
SO = os.path.join(LIBDIR, "libquapi.so")
SOURCES = [os.path.join(CSRC, f) for f in ("host.cpp", "slide4.cu", "slide3.cu", "slide2.cu", "slide2t.cu", "slide_r.cu", "persist.cu", "grow.cu", "ofpf.cu", "batch.cu", "eta.cu")]
DEPS = SOURCES + [os.path.join(CSRC, "qp_internal.h"), os.path.join(CSRC, "common.cuh"), os.path.join(CSRC, "tmem.cuh"), os.path.join(ROOT, "include", "quapi.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
         "-I", os.path.join(ROOT, "include")]


def _fresh() -> bool:
    return os.path.exists(SO) and os.path.getmtime(SO) >= max(os.path.getmtime(d) for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    if not force and _fresh():
        return SO
    with open(os.path.join(LIBDIR, ".build.lock"), "w") as lock:
        fcntl.flock(lock, fcntl.LOCK_EX)  # another process may be building: wait, then re-check
        if not force and _fresh():
            return SO
        tmp = tempfile.mkdtemp(prefix="quapi_build_", dir=LIBDIR)
        procs = []
        try:
            # one nvcc process per translation unit (in parallel), then one link step
            objs = []
            for src in SOURCES:
                obj = os.path.join(tmp, os.path.basename(src) + ".o")
                cmd = [NVCC, *ARCH, *FLAGS, "-c", "-o", obj, src]
                if verbose:
                    cmd.insert(1, "-Xptxas=-v")
                    print(" ".join(cmd), file=sys.stderr)
                procs.append((subprocess.Popen(cmd), cmd))
                objs.append(obj)
            for pr, cmd in procs:
                if pr.wait() != 0:
                    raise subprocess.CalledProcessError(pr.returncode, cmd)
            out = os.path.join(tmp, "libquapi.so")
            subprocess.check_call([NVCC, *ARCH, "-shared", "-o", out, *objs, "-lpthread"])
            os.replace(out, SO)  # atomic: a concurrent loader sees the old or the new library, never a partial one
        finally:
            for pr, _ in procs:
                if pr.poll() is None:
                    pr.kill()
                    pr.wait()
            shutil.rmtree(tmp, ignore_errors=True)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
