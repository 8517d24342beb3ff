"""Build librrq.so in-tree: nvcc (sm_100a, -lineinfo) for the kernels + C ABI, g++ for the
quad-precision host tables.  Called by __graft_entry__.build() and on import if the .so is stale."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "librrq.so")
ROOT = os.path.dirname(HERE)
SOURCES = [os.path.join(CSRC, f) for f in ("rrq_api.cu", "rrq_tables.cpp", "rrq_device.cuh", "k_build.cuh",
                                           "k_near.cuh", "k_patch.cuh", "k_smooth.cuh")] + [os.path.join(ROOT, "include", "rrq.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in SOURCES)


def build(force=False, verbose=False):
    if not force and not stale():
        return LIB
    tab_o = os.path.join(CSRC, "rrq_tables.o")
    subprocess.check_call(["g++", "-O2", "-fPIC", "-c", os.path.join(CSRC, "rrq_tables.cpp"), "-o", tab_o])
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
           "-Xptxas", "-v" if verbose else "-O3",
           os.path.join(CSRC, "rrq_api.cu"), tab_o, "-o", LIB + ".tmp", "-lquadmath"]
    subprocess.check_call(cmd)
    os.replace(LIB + ".tmp", LIB)
    return LIB


def build_variant(name, defines):
    """Experiment hook: the same sources with extra -D flags into variants/librrq_<name>.so (load it with
    RRQ_LIBRARY=<path>); the product library is untouched."""
    out_dir = os.path.join(ROOT, "variants")
    os.makedirs(out_dir, exist_ok=True)
    out = os.path.join(out_dir, f"librrq_{name}.so")
    tab_o = os.path.join(CSRC, "rrq_tables.o")
    if not os.path.exists(tab_o):
        subprocess.check_call(["g++", "-O2", "-fPIC", "-c", os.path.join(CSRC, "rrq_tables.cpp"), "-o", tab_o])
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-O3",
           *[f"-D{d}" for d in defines], os.path.join(CSRC, "rrq_api.cu"), tab_o, "-o", out, "-lquadmath"]
    subprocess.check_call(cmd)
    return out


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(LIB)
