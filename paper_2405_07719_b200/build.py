"""Builds libusp_b200.so in-tree: every CUDA/C++ source under csrc/ compiled
for sm_100a only (nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo).

The library exports the C ABI declared in include/usp_attn.h. It links the
CUDA runtime statically and resolves libcuda (tensor-map encoding) and
libnccl (transport) at run time, so it loads on hosts without a GPU.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# Development A/B builds: USPB_VARIANT=name builds libusp_b200_<name>.so from
# objects in build_<name>/ (with USPB_NVCC_EXTRA flags and, optionally, the
# forward kernel taken from USPB_FA_FWD_SRC); load it with USPB_LIB_PATH.
_VARIANT = os.environ.get("USPB_VARIANT", "")
OUT = os.path.join(HERE, f"libusp_b200_{_VARIANT}.so" if _VARIANT else "libusp_b200.so")
OBJ = os.path.join(HERE, f"build_{_VARIANT}" if _VARIANT else "build")
SOURCES = ["fa_fwd_sm100.cu", "fa_bwd_sm100.cu", "reshard.cu", "engine.cu", "plan.cpp", "transport.cpp",
           "simulate.cu", "check_fp64.cu", "transport_p2p.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _flags() -> list[str]:
    extra = ["-DUSPB_TRACE", "-DUSPB_DEV"] if os.environ.get("USPB_TRACE_BUILD") else []
    if _VARIANT:
        extra.append("-DUSPB_DEV")  # development knobs (environment) only in variant builds
    extra += os.environ.get("USPB_NVCC_EXTRA", "").split()  # development experiments only
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
                   "-I", os.path.join(ROOT, "include"), "-I", CSRC, "--expt-relaxed-constexpr"] + extra


def _compile(src: str) -> str:
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    path = os.path.join(CSRC, src)
    if _VARIANT and src == "fa_fwd_sm100.cu" and os.environ.get("USPB_FA_FWD_SRC"):
        path = os.environ["USPB_FA_FWD_SRC"]
    deps = [path] + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".hpp", ".cuh", ".h"))]
    deps += [os.path.join(ROOT, "include", h) for h in ("usp_attn.h", "usp_sim.h")]
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj
    lang = [] if src.endswith(".cu") else ["-x", "cu"]
    cmd = [nvcc()] + _flags() + lang + ["-c", path, "-o", obj]
    subprocess.run(cmd, check=True)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(_compile, SOURCES))
    if os.path.exists(OUT) and os.path.getmtime(OUT) >= max(os.path.getmtime(o) for o in objs):
        return OUT
    tmp = OUT + ".tmp"
    cmd = [nvcc()] + ARCH + ["-shared", "-Xcompiler", "-fPIC", "-o", tmp] + objs + ["-ldl", "-lpthread"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, OUT)
    if verbose:
        print("built", OUT)
    return OUT


if __name__ == "__main__":
    build(verbose=True)
    sys.exit(0)
