"""Build libfblts.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

python -m paper_2405_10505_b200.build
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "lib", "libfblts.so")
SOURCES = [os.path.join(HERE, "csrc", f) for f in ("host.cu", "kernels.cu")]
HEADERS = [os.path.join(ROOT, "include", "fblts.h"), os.path.join(HERE, "csrc", "fblts_internal.h")]

def nccl_root():
    """The NCCL torch loads (the nvidia-nccl wheel), so the library shares torch's libnccl.so.2."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        root = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(root, "include", "nccl.h")):
            return root
    raise RuntimeError("nccl.h not found in the nvidia-nccl wheel")


NVCC_FLAGS = [
    "-std=c++17", "-O3", "-lineinfo",
    "--fmad=false",                       # canonical arithmetic: no FMA contraction
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-shared",
]


def nvcc():
    for p in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if p and (os.path.isabs(p) and os.path.exists(p) or not os.path.isabs(p)):
            return p
    return "nvcc"


STAMP = LIB + ".flags"          # the nvcc flags of the library on disk (a rebuild is due when they change)


def _extra():
    return os.environ.get("FBLTS_NVCC_EXTRA", "").split()      # development knobs, e.g. -DFBLTS_MINB=8


def _flags_key(extra):
    return " ".join(NVCC_FLAGS + extra)


def up_to_date(extra=None):
    """The library exists, is newer than every source and header, and was built with the same flags
    (FBLTS_NVCC_EXTRA included): a development build (-DFBLTS_PROBE=1, ...) is never reused by a
    default build()."""
    extra = _extra() if extra is None else extra
    if not os.path.exists(LIB) or not os.path.exists(STAMP):
        return False
    with open(STAMP) as f:
        if f.read().strip() != _flags_key(extra):
            return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in SOURCES + HEADERS)


def build(force=False, verbose=False):
    extra = _extra()
    if not force and up_to_date(extra):
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    nccl = nccl_root()
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(HERE, "csrc"),
           "-I" + os.path.join(nccl, "include"), "-o", LIB, *SOURCES,
           "-L" + os.path.join(nccl, "lib"), "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(nccl, "lib")]
    if verbose:
        print(" ".join(cmd), flush=True)
    if os.path.exists(STAMP):
        os.unlink(STAMP)
    subprocess.run(cmd, check=True)
    with open(STAMP, "w") as f:
        f.write(_flags_key(extra) + "\n")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
