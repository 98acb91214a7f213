"""In-tree build of the native library (CUDA kernels for sm_100a + host code).

    python -m paper_2101_10463_b200.build

produces paper_2101_10463_b200/librtgpu.so.  Nothing is JIT-compiled at
import time; the package refuses to run without this library.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "librtgpu.so")
SOURCES = ["rtgpu_engine.cu", "rtgpu_k_f64.cu", "rtgpu_k_i64.cu", "rtgpu_k_i128.cu", "rtgpu_k_lat.cu",
           "taskgen.cpp", "executor.cu", "simulator.cu"]
HEADERS = ["engine_core.cuh", "kernel.cuh", "lattice.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "-I", os.path.join(ROOT, "include")]
OBJDIR = os.path.join(HERE, "build")


def _inputs():
    out = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    out += [os.path.join(ROOT, "include", h) for h in ("rtgpu.h", "rtgpu_gen.h", "rtgpu_exec.h", "rtgpu_sim.h")]
    return out


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in _inputs())


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    lib = out or LIB
    if not force and out is None and up_to_date():
        return LIB
    os.makedirs(OBJDIR, exist_ok=True)
    procs, objs = [], []
    tag = "" if out is None else "." + os.path.basename(out)
    for src in SOURCES:  # one translation unit per arithmetic: compile in parallel
        obj = os.path.join(OBJDIR, src + tag + ".o")
        objs.append(obj)
        cmd = [NVCC, *ARCH, *FLAGS, *["-D" + d for d in defines], "-c",
               os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((cmd, subprocess.Popen(cmd, cwd=CSRC)))
    for cmd, pr in procs:
        if pr.wait() != 0:
            raise RuntimeError("build failed: " + " ".join(cmd))
    link = [NVCC, *ARCH, "-shared", "-o", lib + ".tmp", *objs]
    subprocess.run(link, check=True, cwd=CSRC)
    os.replace(lib + ".tmp", lib)
    return lib


def build_packer(force: bool = False) -> str:
    """The CPython extension paper_2101_10463_b200._packer (csrc/packer.cpp):
    TaskSet objects -> blobs without Python-level field walking."""
    import sysconfig
    out = os.path.join(HERE, "_packer" + sysconfig.get_config_var("EXT_SUFFIX"))
    src = os.path.join(CSRC, "packer.cpp")
    if not force and os.path.exists(out) and os.path.getmtime(src) <= os.path.getmtime(out):
        return out
    cmd = [os.environ.get("CXX", "g++"), "-O2", "-std=c++17", "-fPIC", "-shared",
           "-I", sysconfig.get_paths()["include"], src, "-o", out + ".tmp"]
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    return out


TORCH_OP = os.path.join(HERE, "rtgpu_torch.so")


def build_torch_op(force: bool = False, verbose: bool = False) -> str:
    """The PyTorch operator torch.ops.rtgpu.analyze_out (csrc/torch_ops.cpp),
    an in-tree shared library linked against librtgpu.so."""
    src = os.path.join(CSRC, "torch_ops.cpp")
    if not force and os.path.exists(TORCH_OP) and all(
            os.path.getmtime(p) <= os.path.getmtime(TORCH_OP)
            for p in (src, LIB, os.path.join(ROOT, "include", "rtgpu.h"))):
        return TORCH_OP
    from torch.utils import cpp_extension
    bdir = os.path.join(HERE, "build", "torch_op")
    os.makedirs(bdir, exist_ok=True)
    cpp_extension.load(name="rtgpu_torch", sources=[src], build_directory=bdir,
                       extra_include_paths=[os.path.join(ROOT, "include")],
                       extra_cflags=["-O2"], extra_ldflags=[f"-L{HERE}", "-lrtgpu", "-Wl,-rpath,$ORIGIN", f"-Wl,-rpath,{HERE}"],
                       with_cuda=True, is_python_module=False, verbose=verbose)
    built = os.path.join(bdir, "rtgpu_torch.so")
    os.replace(built, TORCH_OP)
    return TORCH_OP


if __name__ == "__main__":
    # python -m paper_2101_10463_b200.build [--force] [--out PATH -DNAME=VAL ...]
    argv = sys.argv[1:]
    out = argv[argv.index("--out") + 1] if "--out" in argv else None
    defs = [a[2:] for a in argv if a.startswith("-D")]
    print(build(force="--force" in argv or out is not None, verbose=True, out=out, defines=defs))
    if out is None and "--no-torch-op" not in argv:
        print(build_torch_op(force="--force" in argv))
    if out is None:
        print(build_packer(force="--force" in argv))
