"""Build the sm_100a shared library in-tree (``libcommtrace_b200.so``).

nvcc cross-compiles here without a GPU; the .so travels to the GPU box with the
repo snapshot.  ``python -m paper_2110_10401_b200.build`` or __graft_entry__.build().
"""

from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
OUT = os.environ.get("CT_BUILD_OUT", "")  # variant builds: alternate output directory
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(OUT or PKG, "libcommtrace_b200.so")
SOURCES = ["ct_api.cu", "ct_fast.cu", "ct_exact.cu", "ct_canon.cu", "ct_emit.cu", "ct_gen.cu", "ct_jsonl.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
    "-I", os.path.join(ROOT, "include"), "-Xcompiler", "-fopenmp",
] + os.environ.get("CT_NVCC_EXTRA", "").split()


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "commtrace_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps)


SHIM = os.path.join(OUT or PKG, "libcomscribe_shim.so")


def build_shim(force: bool = False) -> str:
    """LD_PRELOAD NCCL interposer (host C, no CUDA): csrc/comscribe_shim.c."""
    src = os.path.join(CSRC, "comscribe_shim.c")
    if force or not os.path.exists(SHIM) or os.path.getmtime(src) > os.path.getmtime(SHIM):
        subprocess.run(["gcc", "-O2", "-shared", "-fPIC", "-fvisibility=hidden", "-Wall", "-o", SHIM, src,
                        "-ldl", "-lpthread"], check=True)
    return SHIM


def build_pack(force: bool = False) -> str:
    """Native TraceEvent packer (CPython C API, gcc): csrc/ct_pack.c -> _ctpack extension."""
    import sysconfig

    out = os.path.join(OUT or PKG, "_ctpack" + sysconfig.get_config_var("EXT_SUFFIX"))
    src = os.path.join(CSRC, "ct_pack.c")
    if force or not os.path.exists(out) or os.path.getmtime(src) > os.path.getmtime(out):
        subprocess.run(["gcc", "-O2", "-shared", "-fPIC", "-Wall", "-I", sysconfig.get_paths()["include"], "-o", out,
                        src], check=True)
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    build_shim(force)
    build_pack(force)
    if not force and not _stale():
        return LIB
    objs = []
    obj_dir = os.path.join(OUT or PKG, "_obj")
    os.makedirs(obj_dir, exist_ok=True)
    cmds = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        if not os.path.exists(path):
            continue
        obj = os.path.join(obj_dir, src.replace(".cu", ".o"))
        cmds.append([NVCC, *FLAGS, "-c", path, "-o", obj])
        objs.append(obj)
    # translation units compile independently: one nvcc per source, in parallel
    from concurrent.futures import ThreadPoolExecutor

    def _cc(cmd):
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)

    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        list(ex.map(_cc, cmds))
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB, *objs,
           "-lcudart", "-lgomp"]
    subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
