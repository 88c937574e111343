"""Quick per-config throughput probe (development tool, not the bench contract)."""

import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2602_24066_b200 as sk  # noqa: E402
from tests.configs import CONFIGS, build_wordset  # noqa: E402


def probe(name, B, L=None, reps=3, bwd=True):
    cfg = CONFIGS[name]
    L = L or cfg["L"]
    ws = build_wordset(name, sk)
    dt = torch.float64 if cfg["dtype"] == np.float64 else torch.float32
    X = torch.cumsum(torch.randn(B, L, cfg["d"], device="cuda", dtype=dt) / np.sqrt(L - 1), dim=1)
    plan = ws.plan()
    sumlen = int(ws.lengths.sum())
    out = torch.empty(B, len(ws), device="cuda", dtype=dt)
    g = torch.randn(B, len(ws), device="cuda", dtype=dt)
    dX = torch.empty_like(X)
    plan.forward(X, out, 0, False)
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    tf, tb = [], []
    for _ in range(reps):
        e0.record()
        plan.forward(X, out, 0, False)
        e1.record()
        if bwd:
            plan.backward(X, out, 0, False, g, 0, 0, dX)
        e2.record()
        torch.cuda.synchronize()
        tf.append(e0.elapsed_time(e1))
        tb.append(e1.elapsed_time(e2))
    tf, tb = min(tf), min(tb)
    M = L - 1
    ff = 2.0 * M * sumlen * B
    print(f"{name} B={B} L={L} W={len(ws)} parts={plan.num_parts} step_fmas={plan.step_fmas} sum|w|={sumlen}: "
          f"fwd {tf:.2f} ms ({B / tf * 1e3:.0f} paths/s, {ff / tf / 1e9:.2f} TF alg) | "
          f"bwd {tb:.2f} ms ({B / tb * 1e3:.0f} paths/s, {3 * ff / tb / 1e9:.2f} TF alg) | "
          f"fwd+bwd {B / (tf + tb) * 1e3:.0f} paths/s", flush=True)


if __name__ == "__main__":
    probe("c1", 32)
    probe("c3", 4096)
    probe("c2", 256)
    probe("c4", 256)
    probe("c5", 2048)
