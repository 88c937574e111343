"""Golden fixtures for the log-signature and dense tensor-algebra rows, made by the REFERENCE.

Run in the build container only (needs /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_logsig.py

Writes tests/golden/logsig.npz from sigkit.logsignature_forward / _backward,
tensor_log / tensor_exp (logsig.py:42-192) and chen_concat / signature_inverse
(sigcore.py:321-352) on seeded random paths (tests/helpers.py random_paths
convention: uniform in [-1, 1]).
"""

from __future__ import annotations

import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

import sigkit  # noqa: E402
from sigkit import logsig as ref_logsig  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = [(1, 3, 2, 5), (2, 2, 3, 6), (2, 4, 2, 7), (3, 3, 3, 5), (4, 4, 2, 9), (3, 5, 2, 4)]  # (d, N, B, M)


def main():
    out = {}
    rng = np.random.default_rng(2602)
    for d, N, B, M in CASES:
        tag = f"d{d}N{N}"
        X = rng.random((B, M + 1, d)) * 2.0 - 1.0
        ls = sigkit.logsignature_forward(X, d, N)
        g = rng.standard_normal(ls.values.shape)
        gb = sigkit.logsignature_backward(X, d, N, g)
        compute_ws, lyndon_ws, terms = ref_logsig._lyndon_projection(d, N)
        out[f"{tag}_X"] = X
        out[f"{tag}_logsig"] = ls.values
        out[f"{tag}_g"] = g
        out[f"{tag}_dX"] = gb.path_grads
        out[f"{tag}_lyndon_codes"] = lyndon_ws.codes.astype(np.uint64)
        out[f"{tag}_lyndon_lengths"] = lyndon_ws.lengths.astype(np.int64)
        out[f"{tag}_compute_codes"] = compute_ws.codes.astype(np.uint64)
        out[f"{tag}_compute_lengths"] = compute_ws.lengths.astype(np.int64)
        out[f"{tag}_nterms"] = np.array([len(t) for t in terms], dtype=np.int64)
        # dense truncated tensor algebra on the same paths
        ws = sigkit.build_truncated(d, N)
        S = sigkit.signature_forward(X, ws)
        Y = rng.random((B, M + 1, d)) * 2.0 - 1.0
        S2 = sigkit.signature_forward(Y, ws)
        out[f"{tag}_Y"] = Y
        out[f"{tag}_sig"] = S.values
        out[f"{tag}_tlog"] = ref_logsig.tensor_log(S).values
        out[f"{tag}_texp"] = ref_logsig.tensor_exp(ref_logsig.tensor_log(S)).values
        out[f"{tag}_chen"] = sigkit.chen_concat(S, S2).values
        out[f"{tag}_inv"] = sigkit.signature_inverse(S).values
    np.savez_compressed(os.path.join(HERE, "logsig.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
