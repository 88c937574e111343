"""c5 backward time vs path length (setup share per CTA; developer tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_24066_b200 as sk  # noqa: E402

ws = sk.build_truncated(16, 4)
plan = ws.plan()
B = 8192
for L in (33, 65, 129, 257, 513):
    X = torch.cumsum(torch.randn(B, L, 16, device="cuda") / (L - 1) ** 0.5, 1)
    S = torch.empty(B, len(ws), device="cuda")
    g = torch.randn(B, len(ws), device="cuda")
    dX = torch.empty_like(X)
    work = torch.empty(max(plan.workspace_bytes(torch.float32, B, L, 0), 1), dtype=torch.uint8, device="cuda")
    plan.forward(X, S, 0, False)
    for _ in range(2):
        plan.backward(X, S, 0, False, g, 0, 0, dX, work=work)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(3):
        plan.backward(X, S, 0, False, g, 0, 0, dX, work=work)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"L={L}: bwd {ms:.2f} ms for {B} paths ({ms / (L - 1) * 1e3:.1f} us per step)", flush=True)
