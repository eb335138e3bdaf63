"""Build libtawpipe.so in-tree with nvcc for sm_100a (no torch extension machinery, no JIT cache).

    python -m paper_2511_09741_b200.build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libtawpipe.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def nccl_dir() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("nvidia-nccl wheel not found (needed for nccl.h / libnccl.so.2)")
    return list(spec.submodule_search_locations)[0]


def flags():
    nd = nccl_dir()
    return ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
            "-Xcompiler", "-fPIC", "-Xptxas", "-v" if os.environ.get("TAWPIPE_PTXAS_V") else "-O3",
            "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nd, "include")], nd


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs.append(os.path.join(ROOT, "include", "tawpipe.h"))
    return hs


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    fl, nd = flags()
    hdr_mtime = max(os.path.getmtime(h) for h in headers())
    jobs = []
    for src in sources():
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        if force or not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(src), hdr_mtime):
            jobs.append((src, obj))

    def compile_one(job):
        src, obj = job
        cmd = [NVCC, *fl, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        return src, r.stderr

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for src, err in ex.map(compile_one, jobs):
            if verbose and err:
                print(err, file=sys.stderr)
    objs = [os.path.join(BUILD, os.path.basename(s) + ".o") for s in sources()]
    if force or jobs or not os.path.exists(LIB):
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB, *objs,
               "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2",
               "-Xlinker", "-rpath=" + os.path.join(nd, "lib")]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
