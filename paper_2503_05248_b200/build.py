"""Build libdbk.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with gpurun)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libdbk.so")
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
    if os.path.exists("/usr/include/nccl.h"):
        return "/usr/include", "/usr/lib/x86_64-linux-gnu"
    raise RuntimeError("nccl.h not found")


def _common_flags(nccl_inc):
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-Wall",
                   "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", nccl_inc]


SAN = ["-fsanitize=address", "-fsanitize=undefined", "-fno-omit-frame-pointer", "-fno-sanitize-recover=undefined"]


def _compile(src, flags, verbose, suffix=""):
    obj = os.path.join(OBJ, os.path.basename(src) + suffix + ".o")
    deps = [src] + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "dbk.h")]
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj
    extra = ["-Xptxas", "-v"] if (verbose and src.endswith(".cu")) else []
    cmd = [NVCC] + flags + extra + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = False, sanitize: bool = False) -> str:
    """libdbk.so; sanitize=True: libdbk_asan.so, the host C++ (allocator, scheduler, engine,
    exchange) under AddressSanitizer + UndefinedBehaviorSanitizer."""
    os.makedirs(OBJ, exist_ok=True)
    if force:
        for f in glob.glob(os.path.join(OBJ, "*.o")):
            os.remove(f)
    nccl_inc, nccl_lib = _nccl_dirs()
    flags = _common_flags(nccl_inc)
    lib = LIB.replace("libdbk.so", "libdbk_asan.so") if sanitize else LIB
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))

    def one(src):
        if sanitize and src.endswith(".cpp"):
            return _compile(src, flags + [x for f in SAN for x in ("-Xcompiler", f)], verbose, ".asan")
        return _compile(src, flags, verbose)
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(one, srcs))
    if (not force and os.path.exists(lib)
            and os.path.getmtime(lib) >= max(os.path.getmtime(o) for o in objs)):
        return lib
    link = [NVCC] + ARCH + ["-shared", "-o", lib] + objs + (["-Xlinker", "-lasan", "-Xlinker", "-lubsan"] if sanitize else []) + [
        "-L", nccl_lib, "-Xlinker", "-l:libnccl.so.2", "-Xlinker", f"-rpath,{nccl_lib}",
        "-lpthread"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, sanitize="--sanitize" in sys.argv))
