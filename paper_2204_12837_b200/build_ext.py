"""Build the sm_100a shared library ``_build/libb200pic.so`` (in-tree, so it
travels to the GPU box with the repo snapshot).

-fmad=false keeps the reference's IEEE op order (numba emits no FMA); the
deposit adds no explicit FMA either, so every per-particle value is the
reference's bit for bit and only the J summation order differs.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_build")
LIB = os.path.join(OUT_DIR, "libb200pic.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
    "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr",
    "-Xptxas", "-warn-spills",
]


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(HERE, "..", "include", "b200pic.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(verbose=False, force=False):
    if not force and not needs_build():
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    extra = []
    if os.environ.get("B200PIC_K1_THREADS"):  # tuning experiments only
        extra.append(f"-DK1_THREADS={int(os.environ['B200PIC_K1_THREADS'])}")
    extra += os.environ.get("B200PIC_EXTRA_DEFS", "").split()  # tuning experiments only (-DNAME=V ...)
    out = os.environ.get("B200PIC_BUILD_OUT", LIB)
    cmd = [_nvcc()] + NVCC_FLAGS + extra + ["-o", out + ".tmp"] + sources()
    if verbose:
        print(" ".join(cmd))
    env = dict(os.environ)
    env.pop("CC", None)  # the image's CC points at a gcc without libgomp; nvcc uses PATH gcc
    r = subprocess.run(cmd, capture_output=True, text=True, env=env)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libb200pic.so")
    if verbose and (r.stdout or r.stderr):
        sys.stderr.write(r.stdout + r.stderr)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
    print(LIB)
