"""Build librollpacker.so in-tree with nvcc for sm_100a (no JIT cache: the
.so travels with the repo snapshot to the GPU box)."""
import glob
import os
import subprocess
import sys
import sysconfig
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
OUT = os.path.join(HERE, "librollpacker.so")
BUILD = os.path.join(ROOT, "build", "rollpacker")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def nccl_paths():
    site = sysconfig.get_paths()["purelib"]
    base = os.path.join(site, "nvidia", "nccl")
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if not os.path.exists(os.path.join(inc, "nccl.h")):
        inc = "/usr/include"
    return inc, lib


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("command failed: %s\n%s%s" % (" ".join(cmd), r.stdout, r.stderr))
    return r.stdout + r.stderr


def build(force=False, verbose=False):
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    deps = srcs + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "rollpacker.h"), __file__]
    if not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= max(os.path.getmtime(d) for d in deps):
        return OUT
    os.makedirs(BUILD, exist_ok=True)
    inc, lib = nccl_paths()
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I" + inc,
                    "-I" + os.path.join(ROOT, "include"), "-Xptxas", "-v", "--expt-relaxed-constexpr"]
    objs = []

    def comp(src):
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        log = _run([NVCC] + flags + ["-c", src, "-o", obj])
        return obj, log

    with ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        for obj, log in ex.map(comp, srcs):
            objs.append(obj)
            if verbose:
                sys.stdout.write(log)
    tmp = OUT + ".tmp"
    _run([NVCC] + ARCH + ["-shared", "-o", tmp] + objs +
         ["-L" + lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib, "-lcuda"])
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
