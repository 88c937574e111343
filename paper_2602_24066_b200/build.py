"""Build libsigkit_b200.so in-tree: nvcc for sm_100a, static cudart, -lineinfo.

    python -m paper_2602_24066_b200.build
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libsigkit_b200.so")
SOURCES = ["sigb_api.cu", "sigb_plan.cu", "sigb_tables.cu", "sigb_trunc.cu", "sigb_frag.cu", "sigb_fragplan.cu", "sigb_jit.cu", "sigb_logsig.cu"]
DEPS = SOURCES + ["sigb_internal.h", "sigb_level.cu", "sigb_trunc.cuh", "sigb_trunc_tc.cuh", "sigb_frag.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
    "-Xptxas", "-v",
    # NVRTC compiles the word-set-specialised kernels at run time (sigb_jit.cu)
    "-lnvrtc", "-Xlinker", "-rpath,/usr/local/cuda/lib64",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.exists(cand) or cand == "nvcc"):
            return cand
    return "nvcc"


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = [s for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    deps = [os.path.join(CSRC, s) for s in DEPS if os.path.exists(os.path.join(CSRC, s))]
    deps.append(os.path.join(HERE, "..", "include", "sigkit_b200.h"))
    if not force and os.path.exists(OUT):
        mt = os.path.getmtime(OUT)
        if all(os.path.getmtime(p) <= mt for p in deps):
            return OUT
    cmd = [nvc for nvc in [nvcc()]] + NVCC_FLAGS + ["-o", OUT] + srcs
    res = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    log = os.path.join(CSRC, "build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed ({res.returncode}); see {log}")
    if verbose:
        sys.stdout.write(res.stdout + res.stderr)
    return OUT


def precompile_shipped() -> None:
    """NVRTC-compile the generated kernels of the shipped small word set (config 3,
    fp32 forward + backward) into jit_cache/ next to the library, host-only, so a
    device process (smoke, tests, bench) loads cubins instead of compiling."""
    import json

    import numpy as np

    from . import _lib
    from .wordset import build_custom

    words = os.path.join(os.path.dirname(HERE), "tests", "golden", "c3_words.json")
    if not os.path.exists(words):
        return
    cache = os.path.join(HERE, "jit_cache")
    if os.path.isdir(cache):  # drop cubins of earlier generator versions
        for name in os.listdir(cache):
            if name.endswith(".cubin"):
                os.remove(os.path.join(cache, name))
    with open(words) as f:
        ws = build_custom([tuple(w) for w in json.load(f)["words"]], 16)
    for backward in (False, True):
        _lib.jit_precompile(np.asarray(ws.codes), np.asarray(ws.lengths), ws.d, _lib.SIGB_F32, backward)


def build_ubench(force: bool = False) -> str:
    """tools/ubench_fma: the FFMA/DFMA pipe microbenchmark bench.py uses for the roofline peak."""
    root = os.path.dirname(HERE)
    src = os.path.join(root, "tools", "ubench_fma.cu")
    out = os.path.join(root, "tools", "ubench_fma")
    if not force and os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(src):
        return out
    subprocess.run([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", out, src], check=True,
                   capture_output=True)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
