"""Build libfc.so in-tree: nvcc for sm_100a (-gencode arch=compute_100a,code=sm_100a).

The shared library links the CUDA runtime statically and NCCL dynamically
against the same libnccl.so.2 that torch loads (nvidia-nccl wheel), so one
NCCL is in the process.  Host code that computes weights / tables is built
with -ffp-contract=off (R2/R4/R5 need IEEE rounding exactly as written).
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libfc.so")
SOURCES = ["fc_plan.cpp", "fc_kernels.cu", "fc_inst_ks1.cu", "fc_inst_ks2.cu", "fc_inst_ks3.cu", "fc_inst_ks4.cu",
           "fc_expand.cu", "fc_gather.cpp", "fc_tc.cu", "fc_pages.cu", "fc_jpeg.cpp", "fc_sched.cpp"]
HEADERS = ["fc_internal.h", "fc_device.cuh", "fc_fused.cuh", "fc_tc.cuh", "fc_launch.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs() -> tuple[str, str]:
    site = sysconfig.get_paths()["purelib"]
    base = os.path.join(site, "nvidia", "nccl")
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [os.path.join(INCLUDE, "fc.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    inc, libdir = nccl_dirs()
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    common = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
              *os.environ.get("FC_NVCC_DEFS", "").split(),  # extra -D flags for A/B experiment builds only
              "-I", INCLUDE, "-I", CSRC, "-I", inc]
    cmds, objs = [], []
    for src in SOURCES:
        obj = os.path.join(objdir, src + ".o")
        cmd = [NVCC, *ARCH, *common, "-lineinfo", "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v", "--fmad=false"] if verbose else ["--fmad=false"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        cmds.append(cmd)
        objs.append(obj)
    # the translation units are independent: compile them concurrently
    procs = [subprocess.Popen(c) for c in cmds]
    bad = [c for c, p in zip(cmds, procs) if p.wait() != 0]
    if bad:
        raise subprocess.CalledProcessError(1, bad[0])
    tmp = LIB + ".tmp"
    cuda_lib = os.path.join(os.path.dirname(os.path.dirname(NVCC)), "lib64")  # libnvjpeg (JPEG images, NEXT-4)
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-L", libdir, "-l:libnccl.so.2", "-L", cuda_lib, "-lnvjpeg",
           "-Xlinker", "-rpath," + libdir, "-Xlinker", "-rpath," + cuda_lib, "-cudart", "static"]
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
