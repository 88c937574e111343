"""The five BASELINE.json configurations and their synthetic inputs.

Shared by the tests, the golden-fixture generator and bench.py.  Pure numpy;
never touches /root/reference.
"""

from __future__ import annotations

import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

# length L = samples, M = L - 1 increments (decision 1)
CONFIGS = {
    "c1": dict(seed=1, kind="truncated", d=4, depth=4, B=32, L=128, dtype=np.float64, bwd=False),
    "c2": dict(seed=2, kind="truncated", d=8, depth=5, B=1024, L=1024, dtype=np.float32, bwd=True),
    "c3": dict(seed=3, kind="custom", d=16, B=4096, L=512, dtype=np.float32, bwd=True),
    "c4": dict(seed=4, kind="anisotropic", d=10, gamma=(1.0,) * 5 + (2.0,) * 5, r=6.0,
               B=4096, L=1024, dtype=np.float32, bwd=True),
    "c5": dict(seed=5, kind="truncated", d=16, depth=4, B=65536, L=512, dtype=np.float32, bwd=True),
}
# pathsig's own training benchmark rows (H200): context
# workloads for bench.py, not BASELINE configs.  (B, M, d) with M increments = L - 1.
PAPER_CONFIGS = {
    "p1": dict(seed=11, kind="truncated", d=4, depth=6, B=64, L=1001, dtype=np.float32, bwd=True,
               paper_ms=6.45, paper_row="(64, 1000, 4) N=6: pathsig 6.45 ms on H200"),
    "p2": dict(seed=12, kind="truncated", d=10, depth=4, B=256, L=201, dtype=np.float32, bwd=True,
               paper_ms=9.83, paper_row="(256, 200, 10) N=4: pathsig 9.83 ms on H200"),
}
ALL_CONFIGS = {**CONFIGS, **PAPER_CONFIGS}


def brownian(seed: int, B: int, L: int, d: int, chunk: int | None = None) -> np.ndarray:
    """Brownian paths on [0, 1]: X_0 = 0, dX ~ N(0, 1/(L-1)), fp64.

    Drawn in path-chunks from one Generator; numpy reproduces the one-shot
    array bit for bit.
    """
    rng = np.random.default_rng(seed)
    M = L - 1
    X = np.zeros((B, L, d), dtype=np.float64)
    chunk = chunk or B
    for s in range(0, B, chunk):
        e = min(B, s + chunk)
        dX = rng.standard_normal((e - s, M, d)) / np.sqrt(max(M, 1))
        np.cumsum(dX, axis=1, out=X[s:e, 1:])
    return X


def c3_words_generate() -> list[tuple[int, ...]]:
    """Seeded random prefix-closed trie, 2048 words, max length 5."""
    words = [(i,) for i in range(16)]
    seen = set(words)
    rng = np.random.default_rng(2602)
    while len(words) < 2048:
        parent = words[int(rng.integers(len(words)))]
        if len(parent) >= 5:
            continue
        child = parent + (int(rng.integers(16)),)
        if child not in seen:
            seen.add(child)
            words.append(child)
    return words


def c3_words() -> list[tuple[int, ...]]:
    path = os.path.join(HERE, "golden", "c3_words.json")
    if os.path.exists(path):
        with open(path) as f:
            return [tuple(w) for w in json.load(f)["words"]]
    return c3_words_generate()


def build_wordset(name: str, sk):
    """Build config `name`'s word set with module `sk` (this package or sigkit)."""
    cfg = ALL_CONFIGS[name]
    if cfg["kind"] == "truncated":
        return sk.build_truncated(cfg["d"], cfg["depth"])
    if cfg["kind"] == "custom":
        return sk.build_custom(c3_words(), cfg["d"])
    return sk.build_anisotropic(sk.AnisotropyWeights(cfg["gamma"], cfg["r"]))
