"""In-tree build of libeinplan_b200.so (sm_100a CUDA kernels + C++20 host).

Invoked by ``__graft_entry__.build()`` and ``python -m paper_2206_08301_b200.build``.
nvcc cross-compiles for sm_100a without a GPU.  Objects are rebuilt only
when a source or header is newer than the object.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# EB_BUILD_TAG=t + EB_BUILD_DEFS="-DX ..." build an A/B variant of the
# library (build/obj_t, lib/t/libeinplan_b200.so; load it with EB_LIB_PATH).
_TAG = os.environ.get("EB_BUILD_TAG", "")
_DEFS = os.environ.get("EB_BUILD_DEFS", "").split()
OBJ = os.path.join(PKG, "build", "obj" + (f"_{_TAG}" if _TAG else ""))
LIB = os.path.join(PKG, "lib", *([_TAG] if _TAG else []), "libeinplan_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NCCL_ROOT = None


def _nccl_root():
    try:
        import nvidia.nccl  # the NCCL torch itself loads (2.28.x)
        root = list(nvidia.nccl.__path__)[0]
        if os.path.exists(os.path.join(root, "include", "nccl.h")):
            return root
    except Exception:
        pass
    return None


def _nlohmann():
    """nlohmann/json 3.11.3 as shipped inside cudnn_frontend in this image (the
    same library the reference uses for its einplan/v1 reports)."""
    import sysconfig
    base = os.path.join(sysconfig.get_paths()["purelib"], "include", "cudnn_frontend",
                        "thirdparty")
    if not os.path.exists(os.path.join(base, "nlohmann", "json.hpp")):
        raise RuntimeError("nlohmann/json.hpp not found under " + base)
    return base


def _headers():
    hs = glob.glob(os.path.join(CSRC, "**", "*.h*"), recursive=True)
    hs += glob.glob(os.path.join(CSRC, "**", "*.cuh"), recursive=True)
    hs += glob.glob(os.path.join(ROOT, "include", "**", "*.h"), recursive=True)
    return max((os.path.getmtime(h) for h in hs), default=0.0)


def _compile(src: str, hdr_time: float, nccl: str | None) -> str:
    rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
    obj = os.path.join(OBJ, rel + ".o")
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_time):
        return obj
    inc = ["-I" + os.path.join(ROOT, "include"), "-I" + CSRC, "-isystem", _nlohmann()]
    defs = list(_DEFS)
    if nccl:
        inc.append("-I" + os.path.join(nccl, "include"))
        defs.append("-DEB_HAVE_NCCL=1")
    if src.endswith(".cu"):
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-Xcompiler", "-ffp-contract=off", *defs, *inc, "-c", src, "-o", obj]
    else:
        # Host planner: plain -O2 x86-64, no FMA contraction, no fast-math — the
        # tile solver must reproduce the reference's FP results bit for bit.
        cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-ffp-contract=off", "-fno-fast-math",
               "-I/usr/local/cuda/include", *defs, *inc, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    nccl = _nccl_root()
    srcs = sorted(glob.glob(os.path.join(CSRC, "**", "*.cu"), recursive=True)
                  + glob.glob(os.path.join(CSRC, "**", "*.cpp"), recursive=True))
    ht = _headers()
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(lambda s: _compile(s, ht, nccl), srcs))
    newest = max(os.path.getmtime(o) for o in objs)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        link = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB + ".tmp", *objs,
                "-ldl", "-lpthread", "-lrt"]
        if nccl:
            link += ["-L" + os.path.join(nccl, "lib"), "-l:libnccl.so.2",
                     "-Xlinker", "-rpath=" + os.path.join(nccl, "lib")]
        r = subprocess.run(link, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(link)}\n{r.stdout}\n{r.stderr}")
        os.replace(LIB + ".tmp", LIB)
    if verbose:
        print(LIB)
    return LIB


if __name__ == "__main__":
    build(verbose=True)
