"""Sweep the generated (NVRTC) kernels' launch shapes on config 3 (development tool).

    python tools/jit_sweep.py [B] "FWARPS=4,FCH=8" "BCAP=48,BWARPS=8" ...

Each argument is a comma list of SIGB_JIT_* overrides; every setting builds a
fresh plan (the generator reads the environment at plan creation), checks
forward and backward on 2 paths against the fp64 oracle, and times the full
batch with CUDA events.
"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2602_24066_b200 as sk  # noqa: E402
from oracle import oracle as ora  # noqa: E402  (checker only)
from tests.configs import brownian, c3_words  # noqa: E402

KEYS = ("FWARPS", "FCH", "FMINB", "FCAP", "FPB", "BWARPS", "BCH", "BMINB", "BCAP", "BPB", "FLOCK", "BLOCK", "BMAXREG", "FMAXREG")


def run(B, setting, reps=5):
    for k in KEYS:
        os.environ.pop("SIGB_JIT_" + k, None)
    os.environ.pop("SIGB_JIT_NVRTC_OPTS", None)
    for kv in filter(None, setting.split(",")):
        k, v = kv.split("=", 1)
        os.environ["SIGB_JIT_" + k] = v.replace("+", " ")
    ws = sk.build_custom(c3_words(), 16)
    plan = ws.plan()
    assert plan.kernel_kind == 4, plan.kernel_kind
    L = 512
    Xn = brownian(3, B, L, 16).astype(np.float32)
    X = torch.from_numpy(Xn).cuda()
    out = torch.empty(B, len(ws), device="cuda")
    g = torch.from_numpy(np.random.default_rng(103).standard_normal((B, len(ws))).astype(np.float32)).cuda()
    dX = torch.empty_like(X)
    plan.forward(X, out, 0, False)
    plan.backward(X, out, 0, False, g, 0, 0, dX)
    torch.cuda.synchronize()
    k = 2
    x64 = Xn[:k].astype(np.float64)
    S64 = ora.forward(x64, ws.codes, ws.lengths, 16)
    _, d64 = ora.backward(x64, ws.codes, ws.lengths, 16, g[:k].double().cpu().numpy())
    ef = ora.rel_err(out[:k].cpu().numpy(), S64)
    eb = ora.rel_err(dX[:k].cpu().numpy(), d64)
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    tf, tb = [], []
    for _ in range(reps):
        e0.record()
        plan.forward(X, out, 0, False)
        e1.record()
        plan.backward(X, out, 0, False, g, 0, 0, dX)
        e2.record()
        torch.cuda.synchronize()
        tf.append(e0.elapsed_time(e1))
        tb.append(e1.elapsed_time(e2))
    reps_txt = " ".join(f"{a:.2f}/{b:.2f}" for a, b in zip(tf, tb))
    tf, tb = min(tf), min(tb)
    ff = 2.0 * (L - 1) * int(ws.lengths.sum()) * B
    print(f"[{setting or 'default'}] err fwd {ef:.1e} bwd {eb:.1e} | fwd {tf:.3f} ms ({ff / tf / 1e9:.1f} TF alg) "
          f"| bwd {tb:.3f} ms ({3 * ff / tb / 1e9:.1f} TF alg) | fwd+bwd {B / (tf + tb) * 1e3:.0f} paths/s [{reps_txt}]",
          flush=True)


if __name__ == "__main__":
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    for s in sys.argv[2:] or [""]:
        try:
            run(B, s)
        except Exception as e:  # keep sweeping
            print(f"[{s}] FAILED: {e}", flush=True)
