"""Build libsigkit_b200.so in-tree: nvcc for sm_100a, static cudart, -lineinfo; one object per
translation unit under csrc/build/, recompiled when it or a header it includes changes.

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

COMPILE_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
]
LINK_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-shared", "-cudart", "static",
    # NVRTC compiles the word-set-specialised kernels at run time (sigb_jit.cu)
    "-lnvrtc", "-Xlinker", "-rpath,/usr/local/cuda/lib64",
]
OBJ = os.path.join(CSRC, "build")


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.exists(cand) or cand == "nvcc"):
            return cand
    return "nvcc"


def _local_deps(src: str, seen=None) -> set[str]:
    """The file plus every quoted #include it reaches (recursively)."""
    import re

    seen = set() if seen is None else seen
    if src in seen or not os.path.exists(src):
        return seen
    seen.add(src)
    with open(src) as f:
        for m in re.finditer(r'^\s*#include\s+"([^"]+)"', f.read(), re.M):
            _local_deps(os.path.normpath(os.path.join(os.path.dirname(src), m.group(1))), seen)
    return seen


def build(force: bool = False, verbose: bool = False) -> str:
    """nvcc each translation unit to build/*.o in parallel (only the stale ones), then link."""
    from concurrent.futures import ThreadPoolExecutor

    os.makedirs(OBJ, exist_ok=True)
    srcs = [s for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    jobs = []
    for s in srcs:
        src = os.path.join(CSRC, s)
        obj = os.path.join(OBJ, os.path.splitext(s)[0] + ".o")
        stale = force or not os.path.exists(obj) or any(
            os.path.getmtime(d) > os.path.getmtime(obj) for d in _local_deps(src))
        if stale:
            jobs.append((s, obj))

    def compile_one(job):
        s, obj = job
        cmd = [nvcc()] + COMPILE_FLAGS + ["-c", s, "-o", obj]
        res = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
        return s, cmd, res

    logs = []
    with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4) or 1) as ex:
        for s, cmd, res in ex.map(compile_one, jobs):
            logs.append(" ".join(cmd) + "\n" + res.stdout + res.stderr)
            if res.returncode != 0:
                sys.stderr.write(res.stdout + res.stderr)
                raise RuntimeError(f"nvcc failed on {s} ({res.returncode})")
    objs = [os.path.join(OBJ, os.path.splitext(s)[0] + ".o") for s in srcs]
    if jobs or not os.path.exists(OUT) or any(os.path.getmtime(o) > os.path.getmtime(OUT) for o in objs):
        cmd = [nvcc()] + LINK_FLAGS + ["-o", OUT] + objs
        res = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
        logs.append(" ".join(cmd) + "\n" + res.stdout + res.stderr)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc link failed ({res.returncode})")
    if logs:
        with open(os.path.join(CSRC, "build.log"), "w") as f:
            f.write("\n".join(logs))
        if verbose:
            sys.stdout.write("\n".join(logs))
    return OUT


def precompile_shipped() -> None:
    """NVRTC-compile the generated kernels of the shipped small word set (config 3,
    fp32 and fp64, forward + backward) into jit_cache/ next to the library, host-only, so a
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
    # fp32 for the autograd path, fp64 for the drop-in numpy API (signature_backward is float64)
    for dtype in (_lib.SIGB_F32, _lib.SIGB_F64):
        for backward in (False, True):
            _lib.jit_precompile(np.asarray(ws.codes), np.asarray(ws.lengths), ws.d, dtype, backward)


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
