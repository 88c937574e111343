"""Forward time of the parallel-in-time route vs the sequential sweep (developer tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_24066_b200 as sk  # noqa: E402
from paper_2602_24066_b200.signature import forward_tensor  # noqa: E402

for d, N, B, L in [(4, 4, 32, 128), (4, 6, 64, 1001), (4, 6, 8, 1001), (4, 4, 4, 20001), (8, 4, 2, 10001),
                   (16, 4, 1, 4001), (4, 6, 1, 100001)]:
    ws = sk.build_truncated(d, N)
    X = torch.cumsum(torch.randn(B, L, d, device="cuda") / L ** 0.5, 1)
    res = {}
    for scan in ("0", "1"):
        os.environ["SIGB_SCAN"] = scan
        for _ in range(3):
            forward_tensor(X, ws)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(20):
            forward_tensor(X, ws)
        torch.cuda.synchronize()
        res[scan] = (time.perf_counter() - t0) / 20 * 1e6
    print(f"d={d} N={N} B={B} L={L}: sequential {res['0']:.0f} us, scan {res['1']:.0f} us", flush=True)
