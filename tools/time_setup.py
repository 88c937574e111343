"""Backward time against path length on c5 (fixed per-CTA cost = the L = 2 time; developer tool).

    python tools/time_setup.py [L ...]
"""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2602_24066_b200 as sk
from tests.configs import build_wordset
ws = build_wordset("c5", sk); plan = ws.plan()
B = 8192
for L in ([int(a) for a in sys.argv[1:]] or (2, 3, 33, 65, 129, 513)):
    X = torch.cumsum(torch.randn(B, L, 16, device="cuda") / 22.6, 1)
    S = torch.empty(B, len(ws), device="cuda"); g = torch.randn(B, len(ws), device="cuda"); dX = torch.empty_like(X)
    work = torch.empty(plan.workspace_bytes(torch.float32, B, L, 0), dtype=torch.uint8, device="cuda")
    plan.forward(X, S, 0, False)
    for _ in range(2): plan.backward(X, S, 0, False, g, 0, 0, dX, work=work)
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    torch.cuda.synchronize(); e0.record()
    for _ in range(5): plan.forward(X, S, 0, False)
    e1.record()
    for _ in range(5): plan.backward(X, S, 0, False, g, 0, 0, dX, work=work)
    e2.record(); torch.cuda.synchronize()
    print(f"L={L}: fwd {e0.elapsed_time(e1)/5*8:.2f} ms  bwd {e1.elapsed_time(e2)/5*8:.2f} ms per 65536 paths", flush=True)
