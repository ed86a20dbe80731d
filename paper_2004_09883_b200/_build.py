"""Build libfb.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libfb.so")
CSRC = os.path.join(HERE, "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def nccl_dir() -> str:
    import nvidia.nccl  # torch-bundled NCCL 2.28 (same one torch.distributed uses)
    return os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps() -> list[str]:
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "fb.h"),
                                                               __file__]


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(d) > t for d in deps())


def build(force: bool = False, verbose: bool = False, out: str | None = None, extra: list[str] | None = None) -> str:
    """Compile libfb.so (or `out` with extra nvcc flags, for experiments).  Each .cu compiles
    in its own nvcc process (in parallel), then one link step."""
    from concurrent.futures import ThreadPoolExecutor
    so = out or SO
    if out is None and not force and not needs_build():
        return SO
    nd = nccl_dir()
    flags = ["-Xcompiler", "-fPIC", "-std=c++17", "-O3", "-lineinfo",
             "-gencode", "arch=compute_100a,code=sm_100a",
             "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nd, "include"),
             "-Xptxas", "-v" if verbose else "-O3", *(extra or [])]
    tag = os.path.basename(so).replace(".", "_")
    objdir = os.path.join(HERE, "build", tag)
    os.makedirs(objdir, exist_ok=True)
    objs = [os.path.join(objdir, os.path.basename(src)[:-3] + ".o") for src in sources()]
    cmds = [[NVCC, "-c", *flags, "-o", o, src] for src, o in zip(sources(), objs)]
    if verbose:
        for c in cmds:
            print(" ".join(c), file=sys.stderr)
    with ThreadPoolExecutor(max_workers=len(cmds)) as ex:
        procs = list(ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), cmds))
    for c, pr in zip(cmds, procs):
        sys.stderr.write(pr.stderr)
        if pr.returncode != 0:
            raise subprocess.CalledProcessError(pr.returncode, c)
    link = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", so + ".tmp", *objs,
            "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2",
            "-Xlinker", "-rpath=" + os.path.join(nd, "lib"), "-cudart", "static"]
    subprocess.check_call(link)
    os.replace(so + ".tmp", so)
    return so


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", action="store_true")
    ap.add_argument("--out", default=None)
    ap.add_argument("-D", action="append", default=[])
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.v, out=a.out, extra=["-D" + d for d in a.D]))
