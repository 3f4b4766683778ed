"""Build the CUDA library libgr_b200.so in-tree with nvcc for sm_100a."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgr_b200.so")
SOURCES = ["abi.cu", "graph.cu", "bfs.cu", "sssp.cu", "bc.cu", "cc.cu", "pagerank.cu", "comm.cu", "pbfs.cu", "psssp.cu"]
HEADERS = ["gr_internal.cuh", "frontier.cuh", "pull.cuh", "part.cuh", os.path.join("..", "..", "include", "gr.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# NCCL: the library's own communicator (gr_comm_create) links the libnccl.so.2
# torch ships (nvidia-nccl wheel), found again at run time through the rpath
def _nccl_dir():
    d = os.environ.get("GR_NCCL_DIR", "")
    if d:
        return d
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    for loc in (spec.submodule_search_locations or []) if spec else []:
        if os.path.exists(os.path.join(loc, "include", "nccl.h")):
            return loc
    raise RuntimeError("nccl.h not found (set GR_NCCL_DIR to the nvidia/nccl directory)")


NCCL_DIR = _nccl_dir()
EXTRA = os.environ.get("GR_NVCC_EXTRA", "").split()
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-I" + os.path.join(NCCL_DIR, "include")]
LDFLAGS = ["-Xlinker", os.path.join(NCCL_DIR, "lib", "libnccl.so.2"), "-Xlinker", "-rpath=" + os.path.join(NCCL_DIR, "lib")]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, lib=None):
    global LIB
    if lib:
        LIB = lib
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in HEADERS] + [__file__]
    if not force and not _stale(LIB, deps):
        return LIB
    def compile_one(s):
        o = os.path.join(CSRC, os.path.basename(s) + ".o")
        cmd = [NVCC] + FLAGS + EXTRA + ["-c", s, "-o", o]
        return s, o, subprocess.run(cmd, capture_output=True, text=True)

    # one nvcc per translation unit, in parallel (the units are independent)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, srcs))
    objs = []
    logs = []
    for s, o, r in results:
        logs.append(r.stderr)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed on %s" % s)
        objs.append(o)
    tmp = LIB + ".tmp%d" % os.getpid()
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp] + objs + LDFLAGS
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, LIB)
    for o in objs:
        os.remove(o)
    with open(os.path.join(CSRC, "ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
