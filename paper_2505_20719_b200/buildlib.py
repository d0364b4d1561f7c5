"""Builds paper_2505_20719_b200/lib/libf3rg.so (sm_100a CUDA kernels + C++ host
engine + C ABI) in-tree, and the CPU checkers under oracle/ (test infrastructure).

    python -m paper_2505_20719_b200.buildlib [--force] [-j N]

nvcc cross-compiles for sm_100a without a GPU. Flags that matter:
  -gencode arch=compute_100a,code=sm_100a   Blackwell-only (TMA bulk copies, mbarrier)
  -fmad=false                               never contract a*b+c (reference is no-FMA)
  -lineinfo                                 ncu source view
Host C++ is built with -ffp-contract=off for the same reason. libstdc++ is linked
dynamically on purpose (the image's gcc wrapper would otherwise embed a static
copy, which breaks iostreams inside a dlopen'ed library).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
OBJDIR = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(LIBDIR, "libf3rg.so")

CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
CXX = "g++"

CU_SRCS = ["launch_level.cu", "launch_rich.cu", "launch_blas.cu", "launch_krylov.cu", "launch_precond.cu",
           "launch_setup.cu"]
# launch_tile_inst.cu is compiled once per (matrix precision, kernel family): 18 units
TILE_INST = [(pa, fam) for pa in range(3) for fam in range(6)]
CPP_SRCS = ["engine.cpp", "spec.cpp", "capi.cpp", "problems.cpp", "partition.cpp", "exchange.cpp", "precond.cpp", "mmio.cpp"]


def _gomp_flags():
    specs = glob.glob("/usr/lib/gcc/x86_64-linux-gnu/*/libgomp.spec")
    return ["-fopenmp"] + ([f"-B{os.path.dirname(specs[0])}/"] if specs else [])


def _stdcxx_flags():
    if os.path.exists("/usr/lib/x86_64-linux-gnu/libstdc++.so.6"):
        return ["-L/usr/lib/x86_64-linux-gnu", "-l:libstdc++.so.6"]
    return ["-lstdc++"]


NVCC_FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-fmad=false", "-gencode", "arch=compute_100a,code=sm_100a",
              "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr"]
CXX_FLAGS = ["-std=c++17", "-O2", "-fPIC", "-ffp-contract=off", f"-I{CUDA_HOME}/include", "-Wall", "-Wno-unused"]


def _newest(paths):
    return max((os.path.getmtime(p) for p in paths if os.path.exists(p)), default=0.0)


def _run(cmd, log=None):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if log:
        with open(log, "w") as f:
            f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"command failed ({r.returncode}): {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r


def build_lib(force: bool = False, jobs: int = 8, verbose: bool = False, defines=(), name: str = "") -> str:
    """Builds lib/libf3rg.so, or (tuning sweeps) lib/variants/libf3rg_<name>.so with
    extra -D defines (F3RG_TILE_SCALE, F3RG_STAGES, F3RG_CHUNK)."""
    global OBJDIR, LIB
    saved = (OBJDIR, LIB)
    if name:
        OBJDIR = os.path.join(ROOT, "build", "obj_" + name)
        LIB = os.path.join(LIBDIR, "variants", f"libf3rg_{name}.so")
        os.makedirs(os.path.dirname(LIB), exist_ok=True)
    try:
        return _build_lib(force, jobs, verbose, [f"-D{d}" for d in defines], name)
    finally:
        OBJDIR, LIB = saved


def _build_lib(force, jobs, verbose, dflags, name=""):
    os.makedirs(LIBDIR, exist_ok=True)
    os.makedirs(OBJDIR, exist_ok=True)
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.hpp")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))
    hdr_time = _newest(headers)
    jobs_list = []
    units = [(src, src + ".o", []) for src in CU_SRCS + CPP_SRCS]
    units += [("launch_tile_inst.cu", f"launch_tile_inst_p{pa}_f{fam}.cu.o",
               [f"-DF3RG_INST_PA={pa}", f"-DF3RG_INST_FAMILY={fam}"]) for pa, fam in TILE_INST]
    for src, oname, udefs in units:
        path = os.path.join(CSRC, src)
        obj = os.path.join(OBJDIR, oname)
        if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(path), hdr_time):
            continue
        if src.endswith(".cu"):
            cmd = [NVCC] + NVCC_FLAGS + dflags + udefs + ["-c", path, "-o", obj]
        else:
            cmd = [CXX] + CXX_FLAGS + dflags + _gomp_flags() + ["-c", path, "-o", obj]
        jobs_list.append((cmd, obj + ".log"))
    # the heaviest units first, so the pool's tail is short
    jobs_list.sort(key=lambda j: 0 if "launch_tile_inst" in j[1] else 1)
    if jobs_list:
        with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
            futs = [ex.submit(_run, c, log) for c, log in jobs_list]
            for f in futs:
                f.result()
    objs = [os.path.join(OBJDIR, o) for _, o, _ in units]
    if force or jobs_list or not os.path.exists(LIB) or os.path.getmtime(LIB) < _newest(objs):
        cmd = [CXX, "-shared", "-o", LIB] + objs + [f"-L{CUDA_HOME}/lib64", "-lcudart_static", "-ldl", "-lrt",
                                                     "-lpthread"] + _gomp_flags() + _stdcxx_flags() + \
            ["-Wl,-soname,libf3rg.so", "-Wl,--no-undefined"]
        _run(cmd, os.path.join(OBJDIR, "link.log"))
    # standalone binary-CSR cache writer (host code only, no CUDA): csr_cache.py
    gen = os.path.join(LIBDIR, "f3rg_gen")
    gsrc = [os.path.join(CSRC, "problem_gen.cpp"), os.path.join(CSRC, "problems.cpp")]
    if not name and (force or not os.path.exists(gen) or os.path.getmtime(gen) < max(_newest(gsrc), hdr_time)):
        _run([CXX] + CXX_FLAGS + _gomp_flags() + gsrc + ["-o", gen] + _stdcxx_flags(),
             os.path.join(OBJDIR, "f3rg_gen.log"))
    if verbose:
        print(f"built {LIB}")
    return LIB


def build_oracle(verbose: bool = False) -> None:
    """Compiles the CPU checkers (test infrastructure only): our C restatement
    always, the reference library only where /root/reference exists."""
    odir = os.path.join(ROOT, "oracle")
    _run(["make", "-C", odir, "liboracle"])
    if os.path.isdir("/root/reference/proj/src"):
        _run(["make", "-C", odir, "ref"])
        _run(["make", "-C", odir, "dropin"])  # after build_lib(): links libf3rg.so
    elif verbose:
        print("reference sources absent: using prebuilt oracle/_ref if present")


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=8)
    ap.add_argument("--no-oracle", action="store_true")
    a = ap.parse_args(argv)
    if not shutil.which(NVCC) and not os.path.exists(NVCC):
        sys.exit("nvcc not found")
    build_lib(a.force, a.j, verbose=True)
    if not a.no_oracle:
        build_oracle(verbose=True)


if __name__ == "__main__":
    main()
