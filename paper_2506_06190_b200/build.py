"""Builds libnat.so in-tree with nvcc for sm_100a (no JIT, no PTX fallback).

    python -m paper_2506_06190_b200.build            # incremental
    python -m paper_2506_06190_b200.build --clean

The library links the NCCL shipped with torch's pip wheel (nvidia-nccl 2.28.x), not the
system copy, so it shares one libnccl.so.2 with torch.distributed.
"""
import concurrent.futures
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libnat.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dirs():
    try:
        import nvidia.nccl as m
        root = list(m.__path__)[0]
        return os.path.join(root, "include"), os.path.join(root, "lib")
    except Exception:  # pragma: no cover
        return None, None


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r.stdout + r.stderr


def build(verbose=False, clean=False):
    os.makedirs(BUILD, exist_ok=True)
    inc, libdir = _nccl_dirs()
    if inc is None:
        raise RuntimeError("nvidia-nccl (pip) headers not found")
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(HERE, "..", "include", "nat.h")]
    hdr_mtime = max(os.path.getmtime(h) for h in hdrs)
    objs = []
    flags = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
             "--expt-relaxed-constexpr", "-I", inc] + ARCH
    flags += os.environ.get("NAT_NVCC_EXTRA", "").split()   # tuning experiments only (-D...)
    todo = []
    for s in srcs:
        o = os.path.join(BUILD, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if not clean and os.path.exists(o) and os.path.getmtime(o) > max(os.path.getmtime(s), hdr_mtime):
            continue
        todo.append([NVCC] + flags + ["-c", s, "-o", o])
    # one nvcc per translation unit, in parallel (bem.cu dominates the serial build time)
    jobs = max(1, min(len(todo), int(os.environ.get("NAT_BUILD_JOBS", os.cpu_count() or 1))))
    with concurrent.futures.ThreadPoolExecutor(jobs) as ex:
        for out in ex.map(_run, todo):
            if verbose:
                print(out)
    lib_needs = clean or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs)
    if lib_needs:
        _run([NVCC] + ARCH + ["-shared", "-o", LIB + ".tmp"] + objs +
             ["-L", libdir, "-l:libnccl.so.2", "-Xlinker", "-rpath," + libdir])
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, clean="--clean" in sys.argv))
