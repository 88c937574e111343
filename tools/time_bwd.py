"""Time the c5 truncated backward (and forward) on a sub-batch with CUDA events (developer tool).

    SIGB_LIB_PATH=build/abl/lib_1.so python tools/time_bwd.py [paths] [config] [stride] [f32|f64]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_24066_b200 as sk  # noqa: E402
from tests.configs import CONFIGS, build_wordset  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
name = sys.argv[2] if len(sys.argv) > 2 else "c5"
stride = int(sys.argv[3]) if len(sys.argv) > 3 else 0
dt = torch.float64 if (len(sys.argv) > 4 and sys.argv[4] == "f64") else torch.float32
cfg = CONFIGS[name]
ws = build_wordset(name, sk)
plan = ws.plan()
L, d = cfg["L"], cfg["d"]
X = torch.cumsum(torch.randn(B, L, d, device="cuda", dtype=dt) / (L - 1) ** 0.5, 1)
S = torch.empty(B, len(ws), device="cuda", dtype=dt)
g = torch.randn(B, len(ws), device="cuda", dtype=dt)
dX = torch.empty_like(X)
work = torch.empty(max(plan.workspace_bytes(dt, B, L, stride), 1), dtype=torch.uint8, device="cuda")
plan.forward(X, S, 0, False)
for _ in range(2):
    plan.backward(X, S, 0, False, g, 0, stride, dX, work=work)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
torch.cuda.synchronize()
ev[0].record()
for _ in range(3):
    plan.forward(X, S, 0, False)
ev[1].record()
for _ in range(3):
    plan.backward(X, S, 0, False, g, 0, stride, dX, work=work)
ev[2].record()
torch.cuda.synchronize()
scale = cfg["B"] / B / 3
print(f"{os.environ.get('SIGB_LIB_PATH', 'default')}: fwd {ev[0].elapsed_time(ev[1]) * scale:.1f} ms  "
      f"bwd {ev[1].elapsed_time(ev[2]) * scale:.1f} ms  (per {cfg['B']} paths, {name}, stride {stride}, {dt})",
      flush=True)
