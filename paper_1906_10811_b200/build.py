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
SOURCES = (["aw_api.cu", "aw_kernels.cu", "aw_stream.cu", "aw_diffusion.cu", "aw_fwi.cu", "aw_stencil2d.cu", "aw_resident2d.cu"]
           + [f"aw_stream_r{r}.cu" for r in range(1, 9)]
           + (["aw_stream_r2v.cu", "aw_stream_r4v.cu", "aw_stream_r6v.cu", "aw_stream_r8v.cu"] if DEV else []))
HEADERS = ["aw_internal.h", "aw_stream.cuh", "aw_hstream.cuh", os.path.join("..", "..", "include", "aw.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O2,-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-Xptxas", "-v", "-I" + os.path.join(HERE, "..", "include")]
if DEV:
    FLAGS += ["-DAW_DEV_KNOBS", "-DAW_DEV_VARIANTS"]
STAMP = os.path.join(CSRC, ".build_kind")  # "dev" / "product": a switch forces a rebuild


OBJDIR = os.path.join(CSRC, "obj-dev" if DEV else "obj")  # per build kind: flags differ


def _deps(path: str, seen=None) -> set:
    """path plus the local headers it includes (recursively)."""
    seen = set() if seen is None else seen
    if path in seen or not os.path.exists(path):
        return seen
    seen.add(path)
    for line in open(path, errors="replace"):
        line = line.strip()
        if line.startswith("#include \""):
            inc = os.path.normpath(os.path.join(os.path.dirname(path), line.split('"')[1]))
            _deps(inc, seen)
    return seen


def _obj(src: str) -> str:
    return os.path.join(OBJDIR, src.replace(".cu", ".o"))


def _obj_stale(src: str) -> bool:
    obj = _obj(src)
    if not os.path.exists(obj) or not os.path.exists(obj + ".log"):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in _deps(os.path.join(CSRC, src)) | {__file__})


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    kind = "dev" if DEV else "product"
    if not os.path.exists(STAMP) or open(STAMP).read().strip() != kind:
        return True
    t = os.path.getmtime(LIB)
    return any(_obj_stale(s) or os.path.getmtime(_obj(s)) > t for s in SOURCES)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(OBJDIR, exist_ok=True)
    # the translation units compile in parallel (one streaming-kernel unit per R); only stale objects
    procs = []
    for src in SOURCES:
        if not force and not _obj_stale(src):
            continue
        obj = _obj(src)
        cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((src, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    errors = []
    for src, obj, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            errors.append(f"nvcc failed for {src}:\n{out}")
            if os.path.exists(obj):
                os.remove(obj)
            continue
        with open(obj + ".log", "w") as f:
            f.write(out)
    if errors:
        raise RuntimeError("\n".join(errors))
    objs = [_obj(s) for s in SOURCES]
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-cudart", "static", "-Xcompiler", "-fPIC"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    with open(STAMP, "w") as f:
        f.write("dev" if DEV else "product")
    logs = [open(o + ".log").read() for o in objs]
    with open(os.path.join(CSRC, "ptxas.log" if not DEV else "ptxas-dev.log"), "w") as f:
        f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
