"""Build libspanq.so in-tree for sm_100a (nvcc + g++, parallel, incremental).

    python -m paper_2511_02749_b200.build            # build if stale
    python -m paper_2511_02749_b200.build --force
    python -m paper_2511_02749_b200.build --profiling  # lib/libspanq_prof.so (tools/ only:
                                                       # CTA-0 timelines, timing variants)
    python -m paper_2511_02749_b200.build --variant NAME -D X=1   # lib/libspanq_NAME.so with extra
                                                       # defines (A/B builds for tools/kab.py only)

The library links the CUDA runtime statically and resolves the driver entry point for TMA
descriptors at run time (cudaGetDriverEntryPoint), so it loads on CPU-only hosts too (the
`-m "not gpu"` tests call its host-side planner).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libspanq.so")
BUILD = os.path.join(ROOT, "build", "spanq")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include")]


def sources():
    cu = sorted(glob.glob(os.path.join(CSRC, "kernels", "*.cu")))
    cpp = sorted(glob.glob(os.path.join(CSRC, "*.cpp")) + glob.glob(os.path.join(CSRC, "host", "*.cpp")))
    return cu, cpp


def headers():
    hs = glob.glob(os.path.join(CSRC, "**", "*.h"), recursive=True)
    hs += glob.glob(os.path.join(CSRC, "**", "*.cuh"), recursive=True)
    hs += glob.glob(os.path.join(ROOT, "include", "*.h"))
    return hs


def _tag(profiling=False, variant=None):
    return ("_prof" if profiling else "") + (f"_{variant}" if variant else "")


def _obj(src, profiling=False, variant=None):
    rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
    return os.path.join(BUILD + _tag(profiling, variant), rel + ".o")


def _compile(src, hdr_mtime, force, verbose_ptxas, profiling=False, variant=None, defines=()):
    obj = _obj(src, profiling, variant)
    if not force and os.path.exists(obj):
        m = os.path.getmtime(obj)
        if m >= os.path.getmtime(src) and m >= hdr_mtime:
            return obj, None
    cmd = [NVCC] + ARCH + COMMON + (["-DSPANQ_PROFILING"] if profiling else []) + [f"-D{d}" for d in defines]
    cmd += ["-c", src, "-o", obj]
    if src.endswith(".cu"):
        cmd += ["-Xptxas", "-v"] if verbose_ptxas else []
    else:
        cmd += ["-x", "c++"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return obj, (r.stderr if verbose_ptxas and src.endswith(".cu") else None)


def build(force: bool = False, verbose: bool = False, profiling: bool = False, variant: str = None,
          defines=()) -> str:
    """Build lib/libspanq.so (or, with profiling=True, lib/libspanq_prof.so: -DSPANQ_PROFILING
    compiles in the CTA-0 trace and the timing variants that spq_set_trace drives)."""
    os.makedirs(BUILD + _tag(profiling, variant), exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)
    lib_path = os.path.join(LIBDIR, f"libspanq{_tag(profiling, variant)}.so") if (profiling or variant) else LIB
    cu, cpp = sources()
    hdr_mtime = max(os.path.getmtime(h) for h in headers())
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        futs = [ex.submit(_compile, s, hdr_mtime, force, verbose, profiling, variant, tuple(defines)) for s in cu + cpp]
        results = [f.result() for f in futs]
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log:
                sys.stderr.write(log)
    if not force and os.path.exists(lib_path) and os.path.getmtime(lib_path) >= max(os.path.getmtime(o) for o in objs):
        return lib_path
    cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", lib_path] + objs + ["-lpthread", "-ldl", "-lrt"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return lib_path


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true", help="print ptxas resource usage")
    ap.add_argument("--profiling", action="store_true", help="build lib/libspanq_prof.so (tools only)")
    ap.add_argument("--variant", default=None, help="A/B build: lib/libspanq_<variant>.so (tools only)")
    ap.add_argument("-D", dest="defines", action="append", default=[], help="extra define for --variant")
    a = ap.parse_args()
    print(build(force=a.force or bool(a.defines), verbose=a.verbose, profiling=a.profiling, variant=a.variant,
                defines=a.defines))


if __name__ == "__main__":
    main()
