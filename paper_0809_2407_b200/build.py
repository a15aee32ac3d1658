"""In-tree build of libcaqr_sm100.so (nvcc, sm_100a only)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SOURCES = [os.path.join(HERE, "csrc", "tsqr_sm100.cu")]
HEADERS = [os.path.join(HERE, "csrc", "tsqr_device.cuh"), os.path.join(HERE, "csrc", "dmma_ring.cuh"), os.path.join(HERE, "csrc", "dmma_apply.cuh"), os.path.join(HERE, "csrc", "split_leaf.cuh"), os.path.join(HERE, "csrc", "tm_leaf.cuh"), os.path.join(HERE, "csrc", "tm_tall.cuh"), os.path.join(HERE, "csrc", "tall_apply.cuh"), os.path.join(HERE, "csrc", "tree_factor128.cuh"), os.path.join(HERE, "csrc", "tree_apply_cp.cuh"), os.path.join(HERE, "csrc", "dense_geqr2.cuh"), os.path.join(ROOT, "include", "caqr_sm100.h")]
OUT = os.path.join(HERE, "lib", "libcaqr_sm100.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-shared", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if os.path.exists(cand) else "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(p) <= t for p in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cmd = [nvcc(), *NVCC_FLAGS, "-o", OUT, *SOURCES]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = res.stdout + res.stderr
    with open(os.path.join(HERE, "lib", "build.log"), "w") as fh:
        fh.write(" ".join(cmd) + "\n" + log)
    if res.returncode != 0:
        sys.stderr.write(log)
        raise RuntimeError(f"nvcc failed ({res.returncode})")
    if verbose:
        sys.stderr.write(log)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
