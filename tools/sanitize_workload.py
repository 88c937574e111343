"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

Runs forward, backward (fp32 autograd and fp64 drop-in) and windows through every
kernel family (truncated, fragment, generated, level) on small word sets, so the sanitizer
sees every kernel of libsigkit_b200.so once:

    compute-sanitizer --tool racecheck python tools/sanitize_workload.py
"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_24066_b200 as sk  # noqa: E402
from paper_2602_24066_b200 import _lib  # noqa: E402


def brownian(seed, B, L, d):
    rng = np.random.default_rng(seed)
    X = np.zeros((B, L, d))
    X[:, 1:] = np.cumsum(rng.standard_normal((B, L - 1, d)) / np.sqrt(L - 1), axis=1)
    return X


def run(ws, B=3, L=40):
    X = brownian(1, B, L, ws.d)
    g = np.random.default_rng(2).standard_normal((B, ws.width))
    sk.signature_forward(X, ws)
    sk.signature_backward(X, ws, g)
    Xt = torch.from_numpy(X.astype(np.float32)).cuda().requires_grad_(True)
    sk.signature(Xt, ws).backward(torch.from_numpy(g).float().cuda())
    sk.signature_windows(X, ws, sk.WindowSpec(np.array([[0, L - 1], [3, 9], [5, 6]])))
    torch.cuda.synchronize()


def main():
    sets = {
        "trunc d=16 N=4": sk.build_truncated(16, 4),
        "trunc d=4 N=4 eps": sk.build_truncated(4, 4, include_empty=True),
        "trunc d=8 N=5": sk.build_truncated(8, 5),
        "aniso": sk.build_anisotropic(sk.AnisotropyWeights((1.0,) * 3 + (2.0,) * 3, 5.0)),
        "custom non-closed": sk.build_custom([(0, 1, 1), (1,), (2, 2, 2, 2), (3, 0)], 4),
        "sparse d=16 trie": sk.build_custom([(i,) for i in range(16)] + [(i, (3 * i) % 16) for i in range(16)]
                                            + [(i, (3 * i) % 16, (5 * i + 1) % 16) for i in range(0, 16, 2)], 16),
    }
    for policy in (0, 1, 2, 4):
        _lib.set_kernel_policy(policy)
        for name, ws in sets.items():
            B = 70 if "sparse" in name else (2 if "16" in name else 3)  # sparse: several 32-path blocks
            try:
                run(ws, B=B, L=24 if "16" in name else 40)
            except RuntimeError as e:  # policy 4 forces a generated kernel; report, keep going
                print(f"policy {policy} {name}: launch refused ({e!r}): {_lib.lib().sigb_last_error()}", flush=True)
                continue
            print(f"policy {policy} {name}: kernel kind {ws.plan().kernel_kind}", flush=True)
    _lib.set_kernel_policy(0)
    # round-2 paths: the tcgen05 kernels over several chunks (producer pipelines, both MMA groups),
    # checkpoint_stride on the truncated kernels, the parallel-in-time forward
    for d, N in ((16, 4), (8, 5)):
        ws = sk.build_truncated(d, N)
        run(ws, B=2, L=75)
        X = brownian(3, 2, 75, d)
        g = np.random.default_rng(4).standard_normal((2, ws.width))
        sk.signature_backward(X, ws, g, checkpoint_stride=5)
        Xt = torch.from_numpy(X.astype(np.float32)).cuda().requires_grad_(True)
        sk.signature(Xt, ws, checkpoint_stride=7).backward(torch.from_numpy(g).float().cuda())
        print(f"tcgen05 / checkpoint d={d} N={N}", flush=True)
    os.environ["SIGB_SCAN"] = "2"
    sk.signature_forward(brownian(5, 2, 300, 4), sk.build_truncated(4, 4))
    os.environ["SIGB_SCAN"] = "1"
    torch.cuda.synchronize()
    print("parallel-in-time forward", flush=True)
    _lib.set_kernel_policy(0)
    print("sanitize workload done")


if __name__ == "__main__":
    main()
