"""Build the in-tree C-ABI library libcgx.so for sm_100a with nvcc (no torch extension machinery).

Each .cu under csrc/ compiles to an object in build/ (in parallel, rebuilt when the source or any
header is newer), then everything links into paper_2503_19779_b200/libcgx.so against the NCCL that
ships with torch (the same libnccl.so.2 the process loads).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "cgx")
LIB = os.path.join(PKG, "libcgx.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for d in spec.submodule_search_locations:
            cands.append(os.path.join(d, "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    raise RuntimeError("NCCL headers (torch-bundled nvidia/nccl) not found")


def _flags():
    inc, _ = _nccl_dirs()
    return ARCH + ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-ffp-contract=off",
                   "-Xptxas", "-warn-spills", "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc]


def _newest_header():
    hs = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))
    return max((os.path.getmtime(h) for h in hs), default=0)


RDC = {"k_prelude.cu"}   # translation units calling the device runtime (device graph API)


def _compile(src, verbose):
    obj = os.path.join(BUILD, os.path.basename(src).replace(".cu", ".o"))
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), _newest_header()):
        return obj, None
    extra = ["-rdc=true"] if os.path.basename(src) in RDC else []
    cmd = [NVCC, *_flags(), *extra, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        return obj, f"{' '.join(cmd)}\n{r.stdout}\n{r.stderr}"
    if verbose and (r.stderr.strip() or r.stdout.strip()):
        print(r.stderr, r.stdout, file=sys.stderr)
    return obj, None


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    if force:
        for o in glob.glob(os.path.join(BUILD, "*.o")):
            os.remove(o)
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        res = list(ex.map(lambda s: _compile(s, verbose), srcs))
    errs = [e for _, e in res if e]
    if errs:
        raise RuntimeError("nvcc failed:\n" + "\n\n".join(errs))
    objs = [o for o, _ in res]
    if os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(o) for o in objs):
        return LIB
    # device link of the relocatable objects (device runtime: cudadevrt)
    rdc_objs = [o for o in objs if os.path.basename(o).replace(".o", ".cu") in RDC]
    dlink = os.path.join(BUILD, "dlink.o")
    if rdc_objs:
        cmd = [NVCC, *ARCH, "-Xcompiler", "-fPIC", "-dlink", *rdc_objs, "-lcudadevrt", "-o", dlink]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"device link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        objs = objs + [dlink]
    _, nccl_lib = _nccl_dirs()
    cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudadevrt", "-L", nccl_lib, "-l:libnccl.so.2",
           "-Xlinker", "-rpath," + nccl_lib]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
