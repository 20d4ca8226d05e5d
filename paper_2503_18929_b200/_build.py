"""Build the in-tree shared libraries with nvcc for sm_100a (B200).

libtba.so        — the product: paper_2503_18929_b200/csrc/tba.cu (C ABI in include/tba.h)
libtba_synth.so  — the seeded input generator's CUDA twin: tba_synth/csrc/synth.cu

Both link the CUDA runtime statically so that they dlopen on a machine without a GPU
(the CPU test suite checks the exported symbols) and depend only on the driver on the box.
"""
from __future__ import annotations

import os
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2503_18929_b200")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-O2", "-cudart", "static",
         "-Xptxas", "-warn-spills", "-diag-suppress", "177"]

TARGETS = {
    "tba": (os.path.join(PKG, "csrc", "tba.cu"), os.path.join(PKG, "libtba.so"),
            [os.path.join(ROOT, "include", "tba.h")]),
    "tba_synth": (os.path.join(ROOT, "tba_synth", "csrc", "synth.cu"),
                  os.path.join(ROOT, "tba_synth", "libtba_synth.so"), []),
}


def nvcc() -> str:
    for c in [os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"]:
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _stale(src: str, out: str, deps) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(p) > t for p in [src, *deps, __file__])


def build(force: bool = False, verbose: bool = False) -> dict:
    """Compile every extension that is missing or older than its sources. Returns {name: path}."""
    out = {}
    for name, (src, lib, deps) in TARGETS.items():
        if force or _stale(src, lib, deps):
            cmd = [nvcc(), *ARCH, *FLAGS, "-o", lib + ".tmp", src]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {name}:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
            if verbose and (r.stdout or r.stderr):
                print(r.stdout, r.stderr)
            os.replace(lib + ".tmp", lib)
        out[name] = lib
    return out


def build_c_example(out: str | None = None) -> str:
    """Compile examples/c_abi_example.c against include/tba.h and libtba.so (plain C + CUDA runtime)."""
    build()
    cuda = os.path.dirname(os.path.dirname(nvcc()))
    out = out or os.path.join(ROOT, "examples", "c_abi_example")
    cmd = ["gcc", "-O2", "-std=c11", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(cuda, "include"),
           os.path.join(ROOT, "examples", "c_abi_example.c"), "-L", PKG, "-ltba", f"-Wl,-rpath,{PKG}",
           "-L", os.path.join(cuda, "lib64"), "-lcudart", f"-Wl,-rpath,{os.path.join(cuda, 'lib64')}", "-lm",
           "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"gcc failed: {' '.join(cmd)}\n{r.stderr}")
    return out


if __name__ == "__main__":
    import sys
    print(build(force="--force" in sys.argv, verbose=True))
