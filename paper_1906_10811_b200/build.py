"""Build libaw.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_1906_10811_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libaw.so")
# AW_DEV_BUILD=1: development build -- adds the measurement variants of the streaming kernel
# (aw_stream_r{4,6,8}v.cu, AW_STREAM_VARIANT) and makes libaw read the development knobs
# (aw_internal.h dev_knob).  The product library (default) has neither.
DEV = os.environ.get("AW_DEV_BUILD", "0") == "1"
SOURCES = (["aw_api.cu", "aw_kernels.cu", "aw_stream.cu", "aw_diffusion.cu", "aw_fwi.cu", "aw_stencil2d.cu"]
           + [f"aw_stream_r{r}.cu" for r in range(1, 9)]
           + (["aw_stream_r4v.cu", "aw_stream_r6v.cu", "aw_stream_r8v.cu"] if DEV else []))
HEADERS = ["aw_internal.h", "aw_stream.cuh", os.path.join("..", "..", "include", "aw.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2,-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-Xptxas", "-v", "-I" + os.path.join(HERE, "..", "include")]
if DEV:
    FLAGS += ["-DAW_DEV_KNOBS", "-DAW_DEV_VARIANTS"]
STAMP = os.path.join(CSRC, ".build_kind")  # "dev" / "product": a switch forces a rebuild


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    kind = "dev" if DEV else "product"
    if not os.path.exists(STAMP) or open(STAMP).read().strip() != kind:
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [__file__]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    # the translation units compile in parallel (aw_stream.cu dominates: one kernel per R and mode)
    procs = []
    for src in SOURCES:
        obj = os.path.join(CSRC, src.replace(".cu", ".o"))
        cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((src, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    objs, logs, errors = [], [], []
    for src, obj, p in procs:
        out, _ = p.communicate()
        logs.append(out)
        if p.returncode != 0:
            errors.append(f"nvcc failed for {src}:\n{out}")
        objs.append(obj)
    if errors:
        raise RuntimeError("\n".join(errors))
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-cudart", "static", "-Xcompiler", "-fPIC"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    with open(STAMP, "w") as f:
        f.write("dev" if DEV else "product")
    with open(os.path.join(CSRC, "ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
