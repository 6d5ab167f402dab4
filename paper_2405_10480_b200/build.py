"""Build libleanattn.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

One object per translation unit (an engine family per kernel TU), compiled in parallel, then
linked into one shared library."""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SRC = [os.path.join(CSRC, f) for f in ("decode_tc5_bf16.cu", "decode_tc5_fp16.cu", "decode_gqa.cu", "decode_fp8.cu",
                                       "decode_mha.cu", "decode.cu", "api.cpp", "planner.cpp")]
DEPS = SRC + [os.path.join(CSRC, f) for f in ("la_internal.h", "ptx.cuh", "tc5.cuh", "decode_kernel.cuh")] + \
    [os.path.join(ROOT, "include", "la.h")]
OUT = os.path.join(HERE, "lib", "libleanattn.so")
OBJ = os.path.join(HERE, "lib", "obj")

NVCC_FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
              "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.exists(cand) or cand == "nvcc"):
            return cand
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in DEPS)


def _compile(src: str, extra) -> tuple:
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    cmd = [nvcc()] + NVCC_FLAGS + list(extra) + ["-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return src, obj, r


def build(force: bool = False, verbose: bool = False, extra_flags=(), out: str = OUT) -> str:
    """Compile every TU for sm_100a (in parallel) and link ``out``.  ``extra_flags`` (e.g.
    ``-DLA_MHA_NST=6``) build a variant library for sweeps (``LEANATTN_LIB`` selects it)."""
    if not force and out == OUT and not extra_flags and up_to_date():
        return out
    os.makedirs(OBJ, exist_ok=True)
    with ThreadPoolExecutor(max_workers=min(len(SRC), os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, extra_flags), SRC))
    bad = [(s, r) for s, _, r in results if r.returncode != 0]
    for s, r in bad:
        sys.stderr.write(f"---- {os.path.basename(s)}\n" + r.stdout + r.stderr)
    if bad:
        raise RuntimeError("nvcc failed building libleanattn.so: " + ", ".join(os.path.basename(s) for s, _ in bad))
    if verbose:
        for s, _, r in results:
            sys.stderr.write(f"---- {os.path.basename(s)}\n" + r.stderr)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", out + ".tmp"] + [o for _, o, _ in results]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libleanattn.so")
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
