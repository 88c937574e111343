"""Generate the golden fixtures under tests/golden/ by importing the REFERENCE.

Run in the build container only (needs /root/reference, which does not exist
on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Everything written here comes from the reference package `sigkit`
(/root/reference/pkg/src) run through its public API; the fixtures pin both
the C oracle (tests/test_oracle_golden.py) and the CUDA path (tests/test_gpu_*.py).
Inputs follow SURVEY.md 8(d): Brownian paths from numpy default_rng(seed).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

import sigkit  # noqa: E402
from sigkit import testkit  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from tests.configs import CONFIGS, brownian, c3_words, c3_words_generate  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def fingerprint(ws) -> str:
    return hashlib.sha256(",".join(ws.word_strings()).encode()).hexdigest()[:16]


def ref_wordset(name):
    if name == "c1":
        return sigkit.build_truncated(4, 4)
    if name == "c2":
        return sigkit.build_truncated(8, 5)
    if name == "c3":
        return sigkit.build_custom(c3_words_generate(), 16)
    if name == "c4":
        return sigkit.build_anisotropic(
            sigkit.AnisotropyWeights((1.0,) * 5 + (2.0,) * 5, 6.0)
        )
    if name == "c5":
        return sigkit.build_truncated(16, 4)
    raise KeyError(name)


def random_paths(rng, B, M, d, scale=1.0):
    return (rng.random((B, M + 1, d)) * 2.0 - 1.0) * scale


def main():
    meta = {"wordsets": {}}
    # -- word sets: fingerprints, level counts, table hashes -------------------
    for name in CONFIGS:
        ws = ref_wordset(name)
        counts = np.bincount(ws.lengths, minlength=ws.max_len + 1)[1:].tolist()
        meta["wordsets"][name] = {
            "W": len(ws),
            "max_len": ws.max_len,
            "sum_len": int(ws.lengths.sum()),
            "levels": counts,
            "fingerprint": fingerprint(ws),
            "codes_sha": sha(ws.codes),
            "lengths_sha": sha(ws.lengths),
            "letters_sha": sha(ws.letters),
            "prefix_sha": sha(ws.prefix_table),
            "suffix_sha": sha(ws.suffix_table),
            "is_full_truncation": bool(ws.is_full_truncation),
        }
    c3 = ref_wordset("c3")
    with open(os.path.join(HERE, "c3_words.json"), "w") as f:
        json.dump({"d": 16, "words": [list(map(int, w)) for w in c3_words_generate()]}, f)

    # -- small tables (full arrays) --------------------------------------------
    small_sets = {
        "trunc_3_3": sigkit.build_truncated(3, 3),
        "trunc_2_4_eps": sigkit.build_truncated(2, 4, include_empty=True),
        "trunc_1_3": sigkit.build_truncated(1, 3),
        "aniso_12_4": sigkit.build_anisotropic(sigkit.AnisotropyWeights((1.0, 2.0), 4.0)),
        "aniso_123_5": sigkit.build_anisotropic(sigkit.AnisotropyWeights((1.0, 2.0, 3.0), 5.0)),
        "custom_np1": sigkit.build_custom([(1, 0), (0, 0, 1), (1,)], 2),
        "custom_np2": sigkit.build_custom([(1, 0), (0, 1, 1), (1, 1, 0, 0)], 2),
        "custom_missing": sigkit.build_custom([(0, 1, 1), (1,)], 2),
        "c3": c3,
    }
    tables = {}
    for key, ws in small_sets.items():
        tables[f"{key}/d"] = np.array(ws.d)
        tables[f"{key}/codes"] = ws.codes
        tables[f"{key}/lengths"] = ws.lengths
        tables[f"{key}/letters"] = ws.letters
        tables[f"{key}/prefix"] = ws.prefix_table
        tables[f"{key}/suffix"] = ws.suffix_table
        tables[f"{key}/include_empty"] = np.array(ws.include_empty)
    np.savez_compressed(os.path.join(HERE, "tables.npz"), **tables)

    # -- forward ------------------------------------------------------------------
    fwd = {}
    # known-answer tests from the reference suite (test_sigcore.py:80-88)
    fwd["kat_segment/X"] = np.array([[[0.0, 0.0], [1.0, 2.0]]])
    fwd["kat_segment/S"] = sigkit.signature_forward(fwd["kat_segment/X"], sigkit.build_truncated(2, 2)).values
    fwd["kat_lpath/X"] = np.array([[[0.0, 0.0], [1.0, 0.0], [1.0, 1.0]]])
    fwd["kat_lpath/S"] = sigkit.signature_forward(fwd["kat_lpath/X"], sigkit.build_truncated(2, 2)).values
    # random small truncated cases (the 40-case oracle sweep, test_sigcore.py:113-123)
    rng = np.random.default_rng(42)
    cases = []
    for i in range(40):
        d = int(rng.integers(1, 4))
        N = int(rng.integers(1, 5))
        M = int(rng.integers(0, 6))
        B = int(rng.integers(1, 4))
        X = random_paths(rng, B, M, d)
        S = sigkit.signature_forward(X, sigkit.build_truncated(d, N)).values
        fwd[f"small{i}/X"] = X
        fwd[f"small{i}/S"] = S
        cases.append((d, N))
    fwd["small/dN"] = np.array(cases)
    # custom / anisotropic sets
    rng = np.random.default_rng(43)
    for key in ("custom_np1", "custom_np2", "custom_missing", "aniso_12_4", "aniso_123_5"):
        ws = small_sets[key]
        X = random_paths(rng, 3, 6, ws.d)
        fwd[f"{key}/X"] = X
        fwd[f"{key}/S"] = sigkit.signature_forward(X, ws).values
        X32 = X.astype(np.float32)
        fwd[f"{key}/X32"] = X32
        fwd[f"{key}/S32"] = sigkit.signature_forward(X32, ws).values
    # config-shaped subsets (Brownian)
    for name, B, L in (("c1", 32, 128), ("c2", 2, 64), ("c3", 4, 128), ("c4", 2, 64), ("c5", 2, 32)):
        cfg = CONFIGS[name]
        ws = ref_wordset(name)
        X = brownian(cfg["seed"], B, L, cfg["d"]).astype(cfg["dtype"])
        fwd[f"{name}/X"] = X
        fwd[f"{name}/S"] = sigkit.signature_forward(X, ws).values
        # fp64 oracle of the same (dtype-rounded) samples: the parity target
        fwd[f"{name}/S64"] = sigkit.signature_forward(X.astype(np.float64), ws).values
    # windows (test_sigcore.py:192-235)
    rng = np.random.default_rng(51)
    X = random_paths(rng, 3, 9, 2)
    pairs = np.array([[0, 4], [2, 7], [8, 9], [0, 9]])
    outs = sigkit.signature_windows(X, sigkit.build_truncated(2, 3), sigkit.WindowSpec(pairs))
    fwd["windows/X"] = X
    fwd["windows/pairs"] = pairs
    fwd["windows/S"] = np.stack([o.values for o in outs], axis=1)
    np.savez_compressed(os.path.join(HERE, "forward.npz"), **fwd)

    # -- backward -----------------------------------------------------------------
    bwd = {}
    rng = np.random.default_rng(4)
    cases = []
    for i in range(15):
        d = int(rng.integers(1, 4))
        N = int(rng.integers(1, 5))
        M = int(rng.integers(1, 9))
        B = int(rng.integers(1, 3))
        X = random_paths(rng, B, M, d)
        ws = sigkit.build_truncated(d, N)
        g = rng.normal(size=(B, len(ws)))
        out = sigkit.signature_backward(X, ws, g)
        bwd[f"small{i}/X"] = X
        bwd[f"small{i}/g"] = g
        bwd[f"small{i}/dX"] = out.path_grads
        bwd[f"small{i}/dInc"] = out.increment_grads
        cases.append((d, N))
    bwd["small/dN"] = np.array(cases)
    rng = np.random.default_rng(5)
    for key in ("custom_np1", "custom_np2", "custom_missing", "aniso_12_4", "aniso_123_5"):
        ws = small_sets[key]
        X = random_paths(rng, 2, 6, ws.d)
        g = rng.normal(size=(2, len(ws)))
        bwd[f"{key}/X"] = X
        bwd[f"{key}/g"] = g
        bwd[f"{key}/dX"] = sigkit.signature_backward(X, ws, g).path_grads
        bwd[f"{key}/dX_fd"] = testkit.finite_difference_grad(X, ws, g)
    # checkpoint stride (test_backward.py:225-234)
    rng = np.random.default_rng(10)
    X = random_paths(rng, 2, 30, 2)
    ws = sigkit.build_truncated(2, 3)
    g = rng.normal(size=(2, len(ws)))
    bwd["ckpt/X"] = X
    bwd["ckpt/g"] = g
    bwd["ckpt/dX_plain"] = sigkit.signature_backward(X, ws, g).path_grads
    bwd["ckpt/dX_c5"] = sigkit.signature_backward(X, ws, g, checkpoint_stride=5).path_grads
    # config-shaped subsets: gradients of the fp64-upcast samples
    for name, B, L in (("c1", 4, 128), ("c2", 1, 32), ("c3", 2, 64), ("c4", 1, 32), ("c5", 1, 16)):
        cfg = CONFIGS[name]
        ws = ref_wordset(name)
        X = brownian(cfg["seed"], B, L, cfg["d"]).astype(cfg["dtype"])
        g = np.random.default_rng(100 + cfg["seed"]).standard_normal((B, len(ws)))
        bwd[f"{name}/X"] = X
        bwd[f"{name}/g"] = g
        bwd[f"{name}/dX"] = sigkit.signature_backward(X, ws, g).path_grads
    np.savez_compressed(os.path.join(HERE, "backward.npz"), **bwd)

    with open(os.path.join(HERE, "meta.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote golden fixtures:", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
