"""Build libgpulsm.so in-tree for sm_100a (nvcc; no JIT, no torch extension).

    python -m paper_1707_05354_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libgpulsm.so")
BUILD = os.path.join(HERE, "_build")

SOURCES = ["sort.cu", "merge.cu", "query.cu", "scan.cu", "index.cu", "cleanup.cu", "shard.cu", "lsm.cu",
           "router.cu"]


def _nccl_dirs():
    """(include dir, lib dir) of the NCCL that torch loads (the nvidia-nccl
    wheel), else the system one. The native router links it by soname, so at
    run time it shares the library torch.distributed already loaded."""
    try:
        import nvidia.nccl
        base = list(nvidia.nccl.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    except ImportError:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


NCCL_INC, NCCL_LIB = _nccl_dirs()
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-I", INCLUDE, "-I", CSRC, "-I", NCCL_INC,
]


def _deps():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    files.append(os.path.join(INCLUDE, "gpulsm.h"))
    files.append(os.path.abspath(__file__))
    return files


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in _deps())


def build(force: bool = False, verbose: bool = False, defines=(), lib: str = LIB,
          build_dir: str = BUILD) -> str:
    """Compile every source and link `lib`. `defines` (e.g. ["GPULSM_L2HINT=0"])
    build an A/B variant into its own object directory."""
    if not force and not defines and up_to_date():
        return LIB
    os.makedirs(build_dir, exist_ok=True)
    procs = []
    objs = []
    for src in SOURCES:
        obj = os.path.join(build_dir, src.replace(".cu", ".o"))
        objs.append(obj)
        cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = []
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or (verbose and out):
            sys.stderr.write(out.decode())
        if p.returncode != 0:
            failed.append(src)
    if failed:
        raise RuntimeError(f"nvcc failed for {failed}")
    tmp = lib + ".tmp"
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                           "-Xcompiler", "-fPIC", "--cudart", "static", *objs,
                           "-L", NCCL_LIB, "-l:libnccl.so.2", "-Xlinker", f"-rpath={NCCL_LIB}",
                           "-o", tmp])
    os.replace(tmp, lib)
    return lib


def build_variant(name: str, defines) -> str:
    """A/B variant libgpulsm_<name>.so (selected at load time by GPULSM_LIB)."""
    return build(force=True, defines=list(defines), lib=os.path.join(HERE, f"libgpulsm_{name}.so"),
                 build_dir=os.path.join(BUILD, name))


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
