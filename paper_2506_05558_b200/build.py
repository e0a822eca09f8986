"""Build libminiba.so in-tree for sm_100a with nvcc (no JIT cache, so the
shared object travels to the GPU box with the repository snapshot)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libminiba.so")
LIB_PROF = os.path.join(HERE, "libminiba_prof.so")
# (source, extra defines, object): the cluster kernel is built once per arithmetic type
SOURCES = [("mba_solve.cu", [], "mba_solve.o"), ("mba_v4.cu", [], "mba_v4_f64.o"),
           ("mba_v4.cu", ["-DMBA_V4_F32"], "mba_v4_f32.o"), ("mba_stages.cu", [], "mba_stages.o"),
           ("mba_pose.cu", [], "mba_pose.o"), ("mba_tri.cu", [], "mba_tri.o"),
           ("mba_match.cu", [], "mba_match.o"),
           ("mba_pack.cu", [], "mba_pack.o"), ("mba_bootstrap.cu", [], "mba_bootstrap.o")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "miniba.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, prof: bool = False) -> str:
    """Compile libminiba.so (or libminiba_prof.so with per-phase cycle counters)."""
    lib = LIB_PROF if prof else LIB
    if not prof:
        build_host(force)
    if not force and not prof and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    def compile_one(job):
        src, defs, obj = job
        obj = os.path.join(CSRC, obj)
        cmd = [NVCC, *FLAGS, *defs, *(["-DMBA_PHASE_PROF"] if prof else []), "-c",
               os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        return obj, r.stderr

    # one nvcc per translation unit, in parallel (the big units dominate)
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        res = list(ex.map(compile_one, SOURCES))
    objs = [o for o, _ in res]
    log = [e for _, e in res]
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", lib, *objs,
           "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    for o in objs:
        os.remove(o)
    if not prof:
        with open(os.path.join(HERE, "build_ptxas.log"), "w") as fh:
            fh.write("\n".join(log))
    if verbose:
        print("\n".join(log))
    return lib


HOST_SRC = os.path.join(CSRC, "host", "mba_host.cpp")


def host_ext_path():
    import sysconfig
    return os.path.join(HERE, "_mba_host" + sysconfig.get_config_var("EXT_SUFFIX"))


def _numpy_include():
    import numpy
    return numpy.get_include()


def build_host(force: bool = False) -> str:
    """Compile the native host extension (CPython C API, no torch) in-tree."""
    import sysconfig
    out = host_ext_path()
    if not force and os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(HOST_SRC):
        return out
    cmd = [os.environ.get("CXX", "g++"), "-O3", "-std=c++17", "-shared", "-fPIC", "-pthread",
           "-Wall", "-Wno-missing-field-initializers", "-I", sysconfig.get_paths()["include"],
           "-I", _numpy_include(),
           HOST_SRC, "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"host extension build failed:\n{r.stderr}")
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, prof="--prof" in sys.argv))
    print(build_host(force="--force" in sys.argv))
