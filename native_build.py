"""Build the native libraries in-tree with nvcc / g++.

Product: paper_1904_11201_b200/libgjoin.so (sm_100a).

Each csrc/*.cu is compiled to an object in parallel, then linked into
paper_1904_11201_b200/libgjoin.so (static cudart; NCCL linked from the venv's
nvidia-nccl wheel when present).  Rebuilds only when a source is newer.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess

ROOT = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.join(ROOT, "paper_1904_11201_b200")
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libgjoin.so")
OBJDIR = os.path.join(PKG, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "--expt-relaxed-constexpr", "-I", INCLUDE, "-I", CSRC]
FLAGS += os.environ.get("GJ_NVCC_EXTRA", "").split()  # extra nvcc flags, e.g. -DNDEBUG


def nccl_paths():
    try:
        import nvidia.nccl as nn  # type: ignore
        base = os.path.dirname(nn.__file__) if nn.__file__ else list(nn.__path__)[0]
    except Exception:
        return None, None
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if os.path.exists(os.path.join(inc, "nccl.h")) and glob.glob(os.path.join(lib, "libnccl.so*")):
        return inc, lib
    return None, None


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _headers():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(INCLUDE, "*.h"))


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJDIR, exist_ok=True)
    srcs = _sources()
    hdrs = _headers()
    inc, libdir = nccl_paths()
    extra = ["-DGJ_HAVE_NCCL=1", "-I", inc] if inc else []
    objs = []
    jobs = []
    for s in srcs:
        o = os.path.join(OBJDIR, os.path.basename(s) + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            jobs.append([NVCC, *ARCH, *FLAGS, *extra, "-c", s, "-o", o])
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            futs = [ex.submit(subprocess.run, j, capture_output=True, text=True) for j in jobs]
            for j, f in zip(jobs, futs):
                r = f.result()
                if verbose or r.returncode != 0:
                    print(" ".join(j))
                    print(r.stdout + r.stderr)
                if r.returncode != 0:
                    raise RuntimeError(f"nvcc failed for {j[-3]}")
    if force or jobs or _stale(LIB, objs):
        link = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart_static"]
        if libdir:
            link += ["-L", libdir, "-l:libnccl.so.2", "-Xlinker", f"-rpath={libdir}"]
        r = subprocess.run(link, capture_output=True, text=True)
        if r.returncode != 0:
            print(" ".join(link))
            print(r.stdout + r.stderr)
            raise RuntimeError("link failed")
    return LIB


GEN_SRC = os.path.join(ROOT, "gen", "gen_device.cu")
GEN_LIB = os.path.join(ROOT, "gen", "libgjgen.so")


def build_gen(force: bool = False) -> str:
    """Test/bench infrastructure: the CUDA twin of the numpy generator."""
    if force or _stale(GEN_LIB, [GEN_SRC]):
        cmd = [NVCC, *ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-o", GEN_LIB, GEN_SRC]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            print(" ".join(cmd))
            print(r.stdout + r.stderr)
            raise RuntimeError("gen build failed")
    return GEN_LIB


def build_all(force: bool = False, verbose: bool = False):
    """Product library, generator twin and the CPU oracle (building the checker is not using it)."""
    import importlib.util
    out = [build(force, verbose), build_gen(force)]
    spec = importlib.util.spec_from_file_location("_oracle_build", os.path.join(ROOT, "oracle", "__init__.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    out.append(mod.build(force))
    return out


if __name__ == "__main__":
    import sys
    print(build_all(force="--force" in sys.argv, verbose="-v" in sys.argv))
