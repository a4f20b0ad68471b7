"""Build recipe of the native library (sm_100a only, in-tree output).

    python -m paper_1607_01039_b200.build

compiles csrc/bw_abi.cu (which includes the kernels) with nvcc into
lib/libbigwht_b200.so.  The .so is git-ignored but travels to the GPU box
with the gpurun snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "bw_abi.cu")
OUT = os.path.join(HERE, "lib", "libbigwht_b200.so")
DEPS = [os.path.join(HERE, "csrc", f) for f in ("bw_abi.cu", "bw_kernels.cuh", "bw_kernels32.cuh", "bw_layouts.h")] + [
    os.path.join(HERE, "..", "include", "bigwht_b200.h")
]

NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-Xcompiler", "-fPIC,-O3",
    "-shared",
]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in DEPS if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cmd = [nvcc(), *NVCC_FLAGS, "-o", OUT + ".tmp", SRC]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


STRESS_OUT = os.path.join(HERE, "lib", "libbigwht_b200_stress.so")


def build_stress(force: bool = False) -> str:
    """The race-stress build (-DBW_RACE_STRESS: random warp sleeps at every
    synchronisation point of the pass kernels; tools/race_stress.sh and
    tests/test_gpu_race_stress.py load it through BW_LIB_PATH).  Test
    infrastructure: the product path never loads it."""
    if not force and os.path.exists(STRESS_OUT) and all(
            os.path.getmtime(d) <= os.path.getmtime(STRESS_OUT) for d in DEPS if os.path.exists(d)):
        return STRESS_OUT
    os.makedirs(os.path.dirname(STRESS_OUT), exist_ok=True)
    cmd = [nvcc(), *NVCC_FLAGS, "-DBW_RACE_STRESS=1", "-o", STRESS_OUT + ".tmp", SRC]
    subprocess.run(cmd, check=True)
    os.replace(STRESS_OUT + ".tmp", STRESS_OUT)
    return STRESS_OUT


if __name__ == "__main__":
    if "--stress" in sys.argv:
        print(build_stress(force="--force" in sys.argv))
    else:
        print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
