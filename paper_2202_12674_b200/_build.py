"""Build the C-ABI shared library libplssvm_b200.so IN-TREE with nvcc for sm_100a.

    python -m paper_2202_12674_b200._build          (or __graft_entry__.build())
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libplssvm_b200.so")
# experiment build (-DPLSSVM_OZ_EXPERIMENTS: the PLSSVM_OZ_DEBUG / PLSSVM_OZ_GROUP switches of the Ozaki
# kernel, which make results WRONG); only tools/ load it, through PLSSVM_EXPERIMENT_LIB=1
LIB_EXP = os.path.join(LIBDIR, "libplssvm_b200_exp.so")
BINDIR = os.path.join(PKG, "bin")
CLI = os.path.join(BINDIR, "plssvm")
SOURCES = ["capi.cu", "driver.cu", "comm.cu", "multi.cu", "io.cpp"]
HEADERS = ["common.cuh", "tile_engine.cuh", "kernels.cuh", "tc_engine.cuh", "ozaki_engine.cuh", "driver.h", "io.h",
           "comm.h"]


def nccl_dirs():
    import nvidia.nccl  # torch-bundled NCCL 2.28 (header + libnccl.so.2)

    base = list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "plssvm.h"), __file__]
    return any(os.path.getmtime(p) > t for p in deps)


def build_cli(force: bool = False) -> str:
    """The LIBSVM-style CLI (csrc/cli.cpp, host C++ over the C ABI) -> bin/plssvm and the
    plssvm-train / plssvm-predict / plssvm-scale links."""
    src = os.path.join(CSRC, "cli.cpp")
    if force or not os.path.exists(CLI) or os.path.getmtime(CLI) < max(os.path.getmtime(src), os.path.getmtime(LIB)):
        os.makedirs(BINDIR, exist_ok=True)
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-Wall", "-o", CLI, src, "-I", os.path.join(ROOT, "include"),
                               "-L", LIBDIR, "-l:libplssvm_b200.so", "-Wl,-rpath,$ORIGIN/../lib"])
    for name in ("plssvm-train", "plssvm-predict", "plssvm-scale"):
        link = os.path.join(BINDIR, name)
        if not os.path.islink(link):
            if os.path.exists(link):
                os.remove(link)
            os.symlink("plssvm", link)
    return CLI


def build(force: bool = False, verbose: bool = False, variant: str = "product", out: str | None = None,
          defines: tuple = ()) -> str:
    """variant "product" (LIB), "exp" (LIB_EXP), or an A/B build of the current sources with extra
    -D defines written to `out` (tools/ only, loaded through PLSSVM_LIB_PATH)."""
    lib = out if out else (LIB if variant == "product" else LIB_EXP)
    if not force and not _stale(lib):
        if variant == "product":
            build_cli()
        return lib
    os.makedirs(LIBDIR, exist_ok=True)
    inc, libd = nccl_dirs()
    tmp = f"{lib}.{os.getpid()}.tmp"
    cmd = [
        "nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
        "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC,-fvisibility=hidden", "-shared", "--threads", "4",
        "-I", os.path.join(ROOT, "include"), "-I", inc,
        *(["-DPLSSVM_OZ_EXPERIMENTS"] if variant == "exp" else []), *[f"-D{x}" for x in defines],
        "-o", tmp, *[os.path.join(CSRC, f) for f in SOURCES],
        "-L", libd, "-l:libnccl.so.2", f"-Xlinker=-rpath,{libd}", "-lcudart",
    ]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    if variant == "product" and not out:
        build_cli(force=True)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv,
                variant="exp" if "--exp" in sys.argv else "product"))
