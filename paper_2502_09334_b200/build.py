"""Builds the in-tree CUDA extension ``_kvx.so`` for sm_100a (nvcc, no JIT cache).

The .so is git-ignored but travels to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(HERE, "_kvx.so")
SOURCES = [os.path.join(HERE, "csrc", "kvx.cu")]
DEPS = SOURCES + [
    os.path.join(HERE, "csrc", "kvx_kernels.cuh"),
    os.path.join(HERE, "csrc", "kvx_kivi.cuh"),
    os.path.join(os.path.dirname(HERE), "include", "kvx.h"),
]
NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(SO_PATH):
        return True
    t = os.path.getmtime(SO_PATH)
    return any(os.path.getmtime(d) > t for d in DEPS if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, variant: str | None = None,
          defines: tuple = ()) -> str:
    """Build _kvx.so (or _kvx_<variant>.so with extra -D defines, for A/B runs
    selected at run time with KVX_LIB=<path>)."""
    out = SO_PATH if variant is None else os.path.join(HERE, f"_kvx_{variant}.so")
    if variant is None and not force and not stale():
        return SO_PATH
    cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-o", out, *SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed ({r.returncode}): {' '.join(cmd)}")
    if verbose:
        sys.stderr.write(r.stderr)
    return out


FAST_SRC = os.path.join(HERE, "csrc", "kvx_fast.c")


def fast_path() -> str:
    import sysconfig
    return os.path.join(HERE, "_kvx_fast" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_fast(force: bool = False) -> str:
    """The CPython fast-call shims for kvx_pair_send/recv (csrc/kvx_fast.c)."""
    import sysconfig
    out = fast_path()
    if not force and os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(FAST_SRC):
        return out
    cmd = [os.environ.get("CC", "gcc"), "-O2", "-shared", "-fPIC", "-Wall",
           f"-I{sysconfig.get_paths()['include']}", "-o", out, FAST_SRC]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"cc failed ({r.returncode}): {' '.join(cmd)}")
    return out


if __name__ == "__main__":
    if "--variant" in sys.argv:
        i = sys.argv.index("--variant")
        name, defs = sys.argv[i + 1], tuple(sys.argv[i + 2:])
        print(build(variant=name, defines=defs))
    else:
        print(build(force="--force" in sys.argv, verbose=True))
        print(build_fast(force="--force" in sys.argv))
