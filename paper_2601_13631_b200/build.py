"""Build libckv.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python -m paper_2601_13631_b200.build [--force] [--tuning]

Each csrc/*.cu is compiled to an object in parallel, then linked with the static
CUDA runtime (no libcuda link dependency: the driver API is reached through
cudaGetDriverEntryPoint), so the library loads on a machine without a GPU.

--variant NAME builds the current sources into libckv_NAME.so (A/B of source variants:
CKV_LIBRARY=variant:NAME in scripts/).
--tuning builds libckv_tuning.so with -DCKV_TUNING: the same kernels plus the environment
knobs the A/B scripts use (CKV_PDL, CKV_SCORE_POLY, CKV_ATTN_SPLITS, traces ...).  The
product libckv.so reads no environment variable.  Scripts select the tuning library with
CKV_LIBRARY=tuning; tests, smoke() and bench.py always load libckv.so.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libckv.so")
BUILD_TUNING = os.path.join(HERE, "_build_tuning")
LIB_TUNING = os.path.join(HERE, "libckv_tuning.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
         "-Xptxas", "-v", "-I", os.path.join(ROOT, "include")]


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    return hs + [os.path.join(ROOT, "include", "ckv.h")]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, build_dir=BUILD, extra=()):
    obj = os.path.join(build_dir, os.path.basename(src)[:-3] + ".o")
    if not _stale(obj, [src] + _headers()):
        return obj, ""
    cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    with open(obj[:-2] + ".ptxas.log", "w") as f:  # register / spill report of this object
        f.write(r.stderr)
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False, tuning: bool = False, variant: str = "") -> str:
    build_dir, lib_path = (BUILD_TUNING, LIB_TUNING) if tuning else (BUILD, LIB)
    if variant:  # A/B: the current sources as libckv_<variant>.so (CKV_LIBRARY=variant:<variant>)
        build_dir = os.path.join(HERE, "_build_var_" + variant)
        lib_path = os.path.join(HERE, "libckv_" + variant + ".so")
    extra = ("-DCKV_TUNING",) if tuning else ()
    os.makedirs(build_dir, exist_ok=True)
    srcs = _sources()
    if force:
        for f in os.listdir(build_dir):
            os.remove(os.path.join(build_dir, f))
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        results = list(ex.map(lambda s_: _compile(s_, build_dir, extra), srcs))
    objs = [o for o, _ in results]
    log = "".join(e for _, e in results)
    if verbose and log:
        print(log)
    if force or _stale(lib_path, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", lib_path, *objs, "-cudart", "static", "-Xlinker", "--no-undefined"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return lib_path


if __name__ == "__main__":
    var = sys.argv[sys.argv.index("--variant") + 1] if "--variant" in sys.argv else ""
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, tuning="--tuning" in sys.argv, variant=var))
