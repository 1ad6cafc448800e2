"""Build of libheatfem.so (sm_100a) in-tree with nvcc.  No JIT cache, no torch extension:
the shared library sits next to this file so it travels with the repository snapshot."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = [os.path.join(HERE, "csrc", "hf_lib.cu")]
DEPS = SRC + [os.path.join(HERE, "csrc", "hf_kernels.cuh"), os.path.join(HERE, "csrc", "hf_ablate.cuh"),
              os.path.join(ROOT, "include", "heatfem.h")]
LIB = os.path.join(HERE, "libheatfem.so")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    extra = os.environ.get("HF_NVCC_EXTRA", "").split()
    cmd = [nvcc()] + NVCC_FLAGS + extra + ["-I" + os.path.join(ROOT, "include"), "-o", LIB + ".tmp"] + SRC + ["-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    if verbose:
        print(res.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
