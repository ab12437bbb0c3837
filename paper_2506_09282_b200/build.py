"""In-tree build of libhdc.so (and the input generator's libhdcgen.so) for sm_100a.

The shared objects stay inside the repo so they travel to the GPU box with the
gpurun snapshot and are the ones the tests and bench load.
"""
import concurrent.futures
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# HDC_BUILD_TAG / HDC_NVCC_DEFS: side builds for A/B measurements (lib/libhdc_<tag>.so,
# loaded through HDC_LIB_PATH); the default build is the product.
_TAG = os.environ.get("HDC_BUILD_TAG", "")
OBJ = os.path.join(PKG, "build" + ("_" + _TAG if _TAG else ""))
LIB = os.path.join(PKG, "lib", "libhdc%s.so" % ("_" + _TAG if _TAG else ""))
DEFS = os.environ.get("HDC_NVCC_DEFS", "").split() if _TAG else []
GEN_SRC = os.path.join(ROOT, "hdc_inputs", "csrc", "hdcgen.cu")
GEN_LIB = os.path.join(ROOT, "hdc_inputs", "libhdcgen.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I", os.path.join(ROOT, "include")]


def _run(cmd):
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout)
        raise RuntimeError("nvcc failed: %s" % cmd[-1])
    return r.stdout


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False, ptxas_info=False):
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    headers = sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
                     + [os.path.join(ROOT, "include", "hdc.h")])
    extra = ["-Xptxas", "-v"] if ptxas_info else []
    jobs = []
    objs = []
    for s in sources:
        o = os.path.join(OBJ, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append([NVCC] + ARCH + FLAGS + DEFS + extra + ["-c", s, "-o", o])
    outs = []
    if jobs:
        with concurrent.futures.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
            outs = list(ex.map(_run, jobs))
    if force or jobs or _stale(LIB, objs):
        tmp = LIB + ".tmp%d" % os.getpid()
        _run([NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-lcuda"])
        os.replace(tmp, LIB)
    if not _TAG and (force or _stale(GEN_LIB, [GEN_SRC])):
        tmp = GEN_LIB + ".tmp%d" % os.getpid()
        _run([NVCC] + ARCH + FLAGS + ["-shared", GEN_SRC, "-o", tmp])
        os.replace(tmp, GEN_LIB)
    if verbose:
        for o in outs:
            sys.stdout.write(o)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, ptxas_info="--ptxas" in sys.argv)
    print(LIB)
