"""Build libragged.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2604_15408_b200.build [--verbose]

The library is a plain C-ABI shared object (include/ragged.h); CUDA runtime is
linked statically so it does not depend on which libcudart torch loads.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libragged.so")
SOURCES = ["kernels.cu", "prune.cu", "block.cu", "attn_general.cu", "attn_fa.cu", "dist_nccl.cu", "api.cu"]
HEADERS = ["device.cuh", "launch.h", "tcgen05.cuh", "attn_tc.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-fvisibility=hidden", "-I", os.path.join(ROOT, "include")]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


VARIANTS = {"": [], "tl": ["-DRAGGED_TIMELINE"],
            # timing experiments only: ablations of the mma.sync engine
            "tlz": ["-DRAGGED_TIMELINE", "-DRAGGED_ABLATE_QK", "-DRAGGED_ABLATE_PV", "-DRAGGED_ABLATE_EXP",
                    "-DRAGGED_ABLATE_ZERO"],
            "abz": ["-DRAGGED_ABLATE_ZERO"],
            "tlnz": ["-DRAGGED_TIMELINE", "-DRAGGED_ABLATE_ZERO"],
            "abc": ["-DRAGGED_ABLATE_QK", "-DRAGGED_ABLATE_PV", "-DRAGGED_ABLATE_EXP"],
            "aball": ["-DRAGGED_ABLATE_QK", "-DRAGGED_ABLATE_PV", "-DRAGGED_ABLATE_EXP",
                      "-DRAGGED_ABLATE_ZERO"],
            # A/B of the fused kernel's pre-wait prefetch: none / keep row only (default: keep row
            # read + kept q/k/v rows prefetched)
            "nopf": ["-DRAGGED_NO_KEEP_PREFETCH"],
            "keeppf": ["-DRAGGED_KEEP_PREFETCH_ONLY"],
            # ablations of the warp-specialised engine (timing experiments only)
            "fansm": ["-DRAGGED_FA_ABLATE_SOFTMAX"], "fanpv": ["-DRAGGED_FA_ABLATE_PV"],
            "fanone": ["-DRAGGED_FA_ABLATE_SOFTMAX", "-DRAGGED_FA_ABLATE_PV"]}


def lib_path(variant: str = "") -> str:
    return LIB if not variant else os.path.join(PKG, f"libragged_{variant}.so")


def _stale(variant: str = "") -> bool:
    lib = lib_path(variant)
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    for h in ("ragged.h", "ragged_debug.h", "ragged_dist.h", "ragged_block.h"):
        deps.append(os.path.join(ROOT, "include", h))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, variant: str = "") -> str:
    lib = lib_path(variant)
    if not force and not _stale(variant):
        return lib
    objdir = os.path.join(PKG, "build" + (f"_{variant}" if variant else ""))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [nvcc(), *ARCH, *FLAGS, *VARIANTS[variant], "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stderr.write(out.decode(errors="replace"))
        if p.returncode != 0:
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
    tmp = lib + ".tmp"
    cmd = [nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", tmp, *objs, "-ldl"]
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    if r.returncode != 0:
        sys.stderr.write(r.stdout.decode(errors="replace"))
        raise RuntimeError("link failed")
    os.replace(tmp, lib)
    return lib


TOOL_SRC = os.path.join(ROOT, "tools", "ragged_bench.cu")
TOOL_BIN = os.path.join(ROOT, "tools", "ragged_bench")


def build_tool(verbose: bool = False) -> str:
    """tools/ragged_bench: the native timing driver (links libragged.so)."""
    build(verbose=verbose)
    cmd = [nvcc(), *ARCH, "-O2", "-std=c++17", "-I", os.path.join(ROOT, "include"), TOOL_SRC, "-o", TOOL_BIN,
           "-L", PKG, "-lragged", "-Xlinker", "-rpath", "-Xlinker", "$ORIGIN/../paper_2604_15408_b200"]
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    if r.returncode != 0:
        sys.stderr.write(r.stdout.decode(errors="replace"))
        raise RuntimeError("ragged_bench build failed")
    return TOOL_BIN


if __name__ == "__main__":
    print(build(force=True, verbose="--verbose" in sys.argv))
    if "--tl" in sys.argv:
        print(build(force=True, variant="tl"))
    if "--tlz" in sys.argv:
        print(build(force=True, variant="tlz"))
    for v in VARIANTS:
        if v and f"--{v}" in sys.argv and v not in ("tl", "tlz"):  # noqa: E501
            print(build(force=True, variant=v))
    if "--tool" in sys.argv:
        print(build_tool())
