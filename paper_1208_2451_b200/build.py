"""Build the in-tree CUDA library libprrp_b200.so for sm_100a with nvcc.

The library is the only compute path of the package; it is built in-tree so
that it travels with the repository snapshot to the GPU host.
"""
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIBNAME = "libprrp_b200.so"
SOURCES = ["prrp_b200.cu"]
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith(".cuh"))

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
    "-I" + os.path.join(ROOT, "include"),
] + (["-DPRRP_P64_PROF"] if os.environ.get("PRRP_P64_PROF") else []) + [
    "-D" + d for d in os.environ.get("PRRP_NVCC_DEFS", "").split(",") if d]


def nvcc():
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the CUDA 12.9 toolkit is required to build libprrp_b200.so")


def lib_path():
    return os.path.join(LIBDIR, LIBNAME)


def _stale(out):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "prrp_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force=False, verbose=False):
    os.makedirs(LIBDIR, exist_ok=True)
    out = lib_path()
    if not force and not _stale(out):
        return out
    tmp = out + ".tmp"
    cmd = [nvcc()] + NVCC_FLAGS + ["-o", tmp] + [os.path.join(CSRC, s) for s in SOURCES]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building %s" % LIBNAME)
    if verbose:
        sys.stderr.write(res.stderr)
    with open(os.path.join(LIBDIR, "ptxas.log"), "w") as fh:
        fh.write(res.stderr)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
