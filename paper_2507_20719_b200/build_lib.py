"""Build libpic.so (sm_100a) in-tree with nvcc.  No torch types cross the ABI."""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpic.so")
SOURCES = ["api.cu", "control.cu", "kernels_basic.cu", "exchange.cu", "gmm.cu", "inject.cu", "order.cu", "peer.cu", "sources.cu", "tiled.cu"]


def _nccl_dirs():
    site = sysconfig.get_paths()["purelib"]
    base = os.path.join(site, "nvidia", "nccl")
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
        return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def nvcc_flags(debug: bool = False):
    inc, _ = _nccl_dirs()
    return ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
            "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
            "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc,
            "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"] + (["-G"] if debug else [])


def build(force: bool = False, verbose: bool = False, defines=(), out: str = None) -> str:
    srcs = [os.path.join(CSRC, f) for f in SOURCES]
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    deps.append(os.path.join(ROOT, "include", "pic.h"))
    lib = out or LIB
    if not force and os.path.exists(lib) and all(os.path.getmtime(lib) >= os.path.getmtime(d) for d in deps):
        return lib
    _, nccl_lib = _nccl_dirs()
    objdir = os.path.join(HERE, "build" + ("_" + "_".join(d.replace("=", "") for d in defines) if defines else ""))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in srcs:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = ["nvcc", "-c", src, "-o", obj] + nvcc_flags() + ["-D" + d for d in defines]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT), src))
        objs.append(obj)
    for p, src in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{out.decode()}")
        if verbose and out:
            print(out.decode(), file=sys.stderr)
    tmp = lib + f".tmp{os.getpid()}"
    cmd = ["nvcc", "-shared", "-o", tmp] + objs + ["-gencode", "arch=compute_100a,code=sm_100a",
                                                   "-L", nccl_lib, "-l:libnccl.so.2",
                                                   "-Xlinker", "-rpath=" + nccl_lib]
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    return lib


CHECKED_LIB = os.path.join(HERE, "libpic_checked.so")


def build_checked(force: bool = False) -> str:
    """libpic with the device bounds checks compiled in (-DPIC_CHECKED: every
    violated index invariant is counted and pic_sync returns PIC_ECUDA) -- the
    stand-in for compute-sanitizer, which is closed on this pool."""
    return build(force=force, defines=("PIC_CHECKED",), out=CHECKED_LIB)


FP64PEAK_SRC = os.path.join(ROOT, "tools", "microbench", "fp64peak.cu")
FP64PEAK_LIB = os.path.join(ROOT, "tools", "microbench", "libfp64peak.so")


def build_fp64peak(force: bool = False) -> str:
    """The sustained-DFMA microbenchmark bench.py reports roofline_fp64 against
    (measurement infrastructure, not part of libpic)."""
    if force or not os.path.exists(FP64PEAK_LIB) or os.path.getmtime(FP64PEAK_LIB) < os.path.getmtime(FP64PEAK_SRC):
        tmp = FP64PEAK_LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["nvcc", "-shared", "-o", tmp, FP64PEAK_SRC, "-gencode", "arch=compute_100a,code=sm_100a",
                               "-O3", "-Xcompiler", "-fPIC"])
        os.replace(tmp, FP64PEAK_LIB)
    return FP64PEAK_LIB


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose=True, defines=defs, out=outs[0] if outs else None))
