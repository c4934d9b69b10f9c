"""Build libpintgpu.so in-tree for sm_100a.

    python -m paper_1912_03106_b200.build

nvcc cross-compiles without a GPU; the .so lands in
paper_1912_03106_b200/lib/ (git-ignored, shipped to the GPU box by gpurun).
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "lib", "libpintgpu.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
         "-Xptxas", "-warn-spills"]
# no library kernels: the CUDA runtime is the only dependency
LIBS = ["-Xlinker", "-rpath=/usr/local/cuda/lib64", "-lpthread"]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)
                  if f.endswith((".cu", ".cuh", ".inc")))


def up_to_date():
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    deps = sources() + [os.path.join(ROOT, "include", "pintgpu.h")]
    return all(os.path.getmtime(s) <= t for s in deps)


def build(force=False, verbose=False):
    if not force and up_to_date():
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = ([nvcc] + ARCH + FLAGS + ["-I" + os.path.join(ROOT, "include"),
                                    os.path.join(CSRC, "pintgpu.cu"), "-o", OUT] + LIBS)
    if verbose:
        print(" ".join(cmd))
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{r.stdout}\n{r.stderr}")
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
