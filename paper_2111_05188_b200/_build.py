"""Build libpod.so in-tree with nvcc for sm_100a (no JIT, no torch extension)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libpod.so")
SOURCES = [os.path.join(HERE, "csrc", f) for f in ("pod_api.cu", "pod_elite.cpp")]
DEPS = SOURCES + [os.path.join(HERE, "csrc", f) for f in os.listdir(os.path.join(HERE, "csrc"))] + [
    os.path.join(ROOT, "include", "pod.h")]


def _nccl_include() -> str:
    try:
        import nvidia.nccl  # type: ignore

        p = os.path.join(list(nvidia.nccl.__path__)[0], "include")
        if os.path.exists(os.path.join(p, "nccl.h")):
            return p
    except Exception:
        pass
    return "/usr/include"


def nvcc_cmd(out: str = LIB):
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    return [nvcc, "-std=c++17", "-O3", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
            "-Xcompiler", "-fPIC,-Wall", "-Xptxas", "-v", "-shared",
            "-I", os.path.join(ROOT, "include"), "-I", _nccl_include(),
            "-o", out] + SOURCES + ["-ldl"]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS if os.path.exists(p))


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile libpod.so if it is missing or older than its sources.  Several processes (one per GPU
    under torchrun) may call this at once: an exclusive file lock serialises them, the first one
    builds into a temporary file that is renamed into place, the others find it up to date."""
    import fcntl

    if not (force or needs_build()):
        return LIB
    with open(os.path.join(HERE, ".build.lock"), "w") as lock:
        fcntl.flock(lock, fcntl.LOCK_EX)
        try:
            if force or needs_build():
                tmp = LIB + ".%d.tmp" % os.getpid()
                cmd = nvcc_cmd(tmp)
                r = subprocess.run(cmd, capture_output=True, text=True)
                if verbose or r.returncode != 0:
                    sys.stderr.write(r.stdout + r.stderr)
                if r.returncode != 0:
                    if os.path.exists(tmp):
                        os.remove(tmp)
                    raise RuntimeError("nvcc failed building libpod.so")
                os.replace(tmp, LIB)
                with open(os.path.join(HERE, "build_ptxas.log"), "w") as f:
                    f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        finally:
            fcntl.flock(lock, fcntl.LOCK_UN)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
