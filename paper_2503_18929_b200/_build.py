"""Build the in-tree shared libraries with nvcc for sm_100a (B200).

libtba.so        — the product: paper_2503_18929_b200/csrc/*.cu (C ABI in include/tba.h), one
                   translation unit per kernel family, compiled in parallel and linked once
libtba_synth.so  — the seeded input generator's CUDA twin: tba_synth/csrc/synth.cu

Both link the CUDA runtime statically so that they dlopen on a machine without a GPU
(the CPU test suite checks the exported symbols) and depend only on the driver on the box.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2503_18929_b200")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-warn-spills",
          "-diag-suppress", "177"]
LDFLAGS = ["-shared", "-cudart", "static"]
CSRC = os.path.join(PKG, "csrc")

TARGETS = {
    # name: (translation units, output, extra dependencies)
    "tba": (sorted(glob.glob(os.path.join(CSRC, "*.cu"))), os.path.join(PKG, "libtba.so"),
            [os.path.join(ROOT, "include", "tba.h"), *glob.glob(os.path.join(CSRC, "*.cuh"))]),
    "tba_synth": ([os.path.join(ROOT, "tba_synth", "csrc", "synth.cu")],
                  os.path.join(ROOT, "tba_synth", "libtba_synth.so"), []),
}


def nvcc() -> str:
    for c in [os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"]:
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _stale(srcs, out: str, deps) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(p) > t for p in [*srcs, *deps, __file__])


def _run(cmd, what: str, verbose: bool) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {what}:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose and (r.stdout or r.stderr):
        print(r.stdout, r.stderr)


def build(force: bool = False, verbose: bool = False) -> dict:
    """Compile every extension that is missing or older than its sources. Returns {name: path}.

    Each translation unit compiles to an object in parallel (nvcc -c), then one nvcc link makes
    the shared library (CUDA runtime linked statically)."""
    out = {}
    for name, (srcs, lib, deps) in TARGETS.items():
        if force or _stale(srcs, lib, deps):
            objdir = os.path.join(os.path.dirname(lib), "build", name)
            os.makedirs(objdir, exist_ok=True)
            objs = [os.path.join(objdir, os.path.splitext(os.path.basename(s))[0] + ".o") for s in srcs]
            jobs = [([nvcc(), *ARCH, *CFLAGS, "-c", "-o", o, s], s) for s, o in zip(srcs, objs)]
            with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 1)) as ex:
                for f in [ex.submit(_run, c, w, verbose) for c, w in jobs]:
                    f.result()
            _run([nvcc(), *ARCH, *LDFLAGS, "-o", lib + ".tmp", *objs], name + " (link)", verbose)
            os.replace(lib + ".tmp", lib)
        out[name] = lib
    return out


def build_variant(name: str, defines, out_root: str = "/tmp/tba_variants", verbose: bool = False) -> str:
    """A/B builds (developer tool, never the product): libtba.so compiled with extra -D defines into
    out_root/name/; load one with TBA_LIBRARY=<path> (paper_2503_18929_b200._lib)."""
    srcs, _, _ = TARGETS["tba"]
    objdir = os.path.join(out_root, name, "obj")
    os.makedirs(objdir, exist_ok=True)
    lib = os.path.join(out_root, name, "libtba.so")
    flags = [f"-D{d}" for d in defines]
    objs = [os.path.join(objdir, os.path.splitext(os.path.basename(s_))[0] + ".o") for s_ in srcs]
    jobs = [([nvcc(), *ARCH, *CFLAGS, *flags, "-c", "-o", o, s_], s_) for s_, o in zip(srcs, objs)]
    with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 1)) as ex:
        for f in [ex.submit(_run, c, w, verbose) for c, w in jobs]:
            f.result()
    _run([nvcc(), *ARCH, *LDFLAGS, "-o", lib, *objs], name + " (link)", verbose)
    return lib


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
