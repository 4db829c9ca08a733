"""Build libtiletune.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery).

    python -m paper_1909_10616_b200.build [--force]

Every translation unit is compiled in parallel to build/*.o, then linked into
``paper_1909_10616_b200/libtiletune.so`` (static cudart; the CUDA driver is reached through
cudaGetDriverEntryPoint, so no -lcuda).  Flags: -gencode arch=compute_100a,code=sm_100a
-lineinfo -O3.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "..", "build", "tiletune")
LIB = os.path.join(HERE, "libtiletune.so")
INCLUDE = os.path.join(HERE, "..", "include")
SOURCES = ["space.cpp", "search.cpp", "abi.cpp", "ctx.cu", "gemm_simt.cu", "gemm_umma.cu", "conv.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _deps_mtime() -> float:
    files = [os.path.join(SRC, f) for f in os.listdir(SRC)] + [os.path.join(INCLUDE, "tiletune.h"), __file__]
    return max(os.path.getmtime(f) for f in files)


def _compile(src: str, obj_dir: str = OBJ, defines=()) -> str:
    obj = os.path.join(obj_dir, src + ".o")
    cmd = [nvcc(), "-c", os.path.join(SRC, src), "-o", obj, "-O3", "-std=c++17", "-lineinfo",
           "-Xcompiler", "-fPIC", "-I", INCLUDE] + ARCH + [f"-D{d}" for d in defines]
    if src.endswith(".cu"):
        cmd += ["-Xptxas", "-v"] if os.environ.get("TT_PTXAS_VERBOSE") else []
    else:   # host search code: no mul-add contraction, so the N-A2C MLP sums exactly as written (Z24)
        cmd += ["-Xcompiler", "-ffp-contract=off"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    if r.stderr.strip():
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _deps_mtime():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(_compile, SOURCES))
    tmp = LIB + ".tmp"
    r = subprocess.run([nvcc(), "-shared", "-o", tmp] + objs + ARCH + ["-lpthread"], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


def build_variant(name: str, defines) -> str:
    """Experiment build: the same sources with extra -D defines -> build/variants/<name>/libtiletune.so
    (load it with TT_LIB_PATH)."""
    obj_dir = os.path.join(HERE, "..", "build", "variants", name)
    os.makedirs(obj_dir, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, obj_dir, defines), SOURCES))
    lib = os.path.join(obj_dir, "libtiletune.so")
    r = subprocess.run([nvcc(), "-shared", "-o", lib] + objs + ARCH + ["-lpthread"], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    return lib


if __name__ == "__main__":
    if "--variant" in sys.argv:
        i = sys.argv.index("--variant")
        print(build_variant(sys.argv[i + 1], sys.argv[i + 2:]))
    else:
        print(build(force="--force" in sys.argv))
