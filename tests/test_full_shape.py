"""Parity at the benchmarked shapes (SURVEY.md 8(c) "parity procedure").

The bench headline (c5: d=16, depth 4, L=512, fp32 fwd+bwd) and c2 (d=8,
depth 5, L=1024) run here at their full length on a GPU-sized sub-batch of the
exact bench inputs (``brownian(seed, B, L, d)`` reproduces the first B paths of
the full batch bit for bit).  The CUDA path runs through the public autograd
API, so the c5 forward is the tcgen05 kernel and the backward the fp32
register kernel, exactly as benched.  The fp64 oracle (oracle/, pinned to the
reference's outputs) then checks the first and last path of the batch and of
every rank's shard, on S and on dL/dX, with the reference's rel_err
(tests/helpers.py:6-11) against the north_star gates: fp32 1e-4, fp64 1e-10.
The kernels being replaced are /root/reference/pkg/src/sigkit/_kernels.py:40-58
(forward) and :85-183 (backward).

Every measured error is appended to ``gpurun_out/parity_full_shape.jsonl`` (or
``$SIGB_PARITY_LOG``) and printed, so the log carries the numbers, not only a pass.
"""

from __future__ import annotations

import json
import os

import numpy as np
import pytest
import torch

import paper_2602_24066_b200 as sk
from oracle import oracle as ora
from paper_2602_24066_b200.sharding import shard_range
from tests.configs import CONFIGS, brownian, build_wordset

pytestmark = pytest.mark.gpu

TOL32 = 1e-4
TOL64 = 1e-10
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _log(rec: dict) -> None:
    path = os.environ.get("SIGB_PARITY_LOG", os.path.join(ROOT, "gpurun_out", "parity_full_shape.jsonl"))
    try:
        os.makedirs(os.path.dirname(path), exist_ok=True)
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")
    except OSError:
        pass
    print(json.dumps(rec))


def _check_paths(name, X32, S, dX, g, picks, tol, tag):
    """fp64 oracle on the fp32-rounded samples of the picked paths."""
    ws = build_wordset(name, sk)
    d = ws.d
    x = X32[picks].astype(np.float64)
    ref = ora.forward(x, ws.codes, ws.lengths, d)
    _, dref = ora.backward(x, ws.codes, ws.lengths, d, g[picks].astype(np.float64))
    es = [ora.rel_err(S[i:i + 1], ref[k:k + 1]) for k, i in enumerate(picks)]
    eg = [ora.rel_err(dX[i:i + 1], dref[k:k + 1]) for k, i in enumerate(picks)]
    _log({"test": tag, "config": name, "paths": [int(p) for p in picks], "rel_err_S": es, "rel_err_dX": eg,
          "tol": tol})
    assert max(es) <= tol, es
    assert max(eg) <= tol, eg


def _shard_picks(B: int, worlds=(2, 4, 8)) -> list[int]:
    picks = {0, B - 1}
    for w in worlds:
        for r in range(w):
            lo, hi = shard_range(B, r, w)
            if hi > lo:
                picks.update((lo, hi - 1))
    return sorted(picks)


@pytest.mark.parametrize("name,B", [("c5", 256), ("c2", 64)])
def test_fp32_autograd_at_bench_shape(name, B):
    """c5: 256 paths x L=512 (tcgen05 forward + fp32 backward); c2: 64 paths x L=1024.
    Oracle on the first/last path of the batch and of each 2/4/8-rank shard."""
    cfg = CONFIGS[name]
    ws = build_wordset(name, sk)
    X32 = brownian(cfg["seed"], B, cfg["L"], cfg["d"]).astype(np.float32)
    g = np.random.default_rng(100 + cfg["seed"]).standard_normal((B, len(ws))).astype(np.float32)
    Xt = torch.from_numpy(X32).cuda().requires_grad_(True)
    St = sk.signature(Xt, ws)
    St.backward(torch.from_numpy(g).cuda())
    torch.cuda.synchronize()
    S = St.detach().cpu().numpy()
    dX = Xt.grad.cpu().numpy()
    assert np.isfinite(S).all() and np.isfinite(dX).all()
    # telescoping: each channel's dL/dX column sums to 0 (reference test_backward.py:207-214)
    assert float(np.abs(dX.sum(axis=1)).max() / max(1.0, np.abs(dX).max())) <= 1e-3
    picks = _shard_picks(B, worlds=(2, 4)) if name == "c2" else _shard_picks(B)
    _check_paths(name, X32, S, dX, g, picks, TOL32, "fp32_autograd_bench_shape")


def test_c5_shards_bitwise_equal_full_batch():
    """Batch sharding: a path's S and dL/dX do not depend on which rank's
    shard (or which CTA-mates) it ran with -- each 2-rank shard reproduces the full-batch
    rows bit for bit, so the sharded bench computes exactly the single-GPU result."""
    cfg = CONFIGS["c5"]
    ws = build_wordset("c5", sk)
    B = 300  # uneven tails inside a CTA
    X = torch.from_numpy(brownian(cfg["seed"], B, cfg["L"], cfg["d"]).astype(np.float32)).cuda()
    g = torch.from_numpy(np.random.default_rng(105).standard_normal((B, len(ws))).astype(np.float32)).cuda()

    def run(lo, hi):
        Xr = X[lo:hi].clone().requires_grad_(True)
        S = sk.signature(Xr, ws)
        S.backward(g[lo:hi])
        return S.detach(), Xr.grad

    S_full, dX_full = run(0, B)
    for r in range(2):
        lo, hi = shard_range(B, r, 2)
        S_r, dX_r = run(lo, hi)
        assert torch.equal(S_r, S_full[lo:hi]), r
        assert torch.equal(dX_r, dX_full[lo:hi]), r


def test_c5_fp64_dropin_backward_full_length():
    """The reference's own precision contract (backward.py:166-167: fp64 everywhere) at the
    c5 word set and length: numpy in, numpy out, within 1e-10 of the fp64 oracle."""
    cfg = CONFIGS["c5"]
    ws = build_wordset("c5", sk)
    B = 8
    X = brownian(cfg["seed"], B, cfg["L"], cfg["d"])
    g = np.random.default_rng(105).standard_normal((B, len(ws)))
    S = sk.signature_forward(X, ws).values
    dX = sk.signature_backward(X, ws, g).path_grads
    picks = [0, 3, 4, B - 1]
    ref = ora.forward(X[picks], ws.codes, ws.lengths, ws.d)
    _, dref = ora.backward(X[picks], ws.codes, ws.lengths, ws.d, g[picks])
    es = ora.rel_err(S[picks], ref)
    eg = ora.rel_err(dX[picks], dref)
    _log({"test": "fp64_dropin_full_length", "config": "c5", "paths": picks, "rel_err_S": es, "rel_err_dX": eg,
          "tol": TOL64})
    assert es <= TOL64 and eg <= TOL64, (es, eg)


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_fp32_autograd_bench_inputs_c3_c4(name):
    """c3 / c4 at full length on their exact bench inputs (the first 128 paths), oracle on the
    first/last path of the batch and of each 2/4-rank shard."""
    cfg = CONFIGS[name]
    ws = build_wordset(name, sk)
    B = 128
    X32 = brownian(cfg["seed"], B, cfg["L"], cfg["d"]).astype(np.float32)
    g = np.random.default_rng(100 + cfg["seed"]).standard_normal((B, len(ws))).astype(np.float32)
    Xt = torch.from_numpy(X32).cuda().requires_grad_(True)
    St = sk.signature(Xt, ws)
    St.backward(torch.from_numpy(g).cuda())
    S = St.detach().cpu().numpy()
    dX = Xt.grad.cpu().numpy()
    _check_paths(name, X32, S, dX, g, _shard_picks(B, worlds=(2, 4)), TOL32, "fp32_autograd_bench_inputs")


@pytest.mark.parametrize("stride", [1, 5, 7])
def test_checkpoint_stride_truncated_kernels(stride):
    """checkpoint_stride (reference backward.py:183-199, _kernels.py:122-141) on the truncated kernels:
    a replay stores the prefix levels every `stride` steps, the reverse sweep reloads them there.
    fp64 drop-in at the c5 word set against the oracle's own stride-`stride` backward (1e-10) and
    against stride 0 (the reference's test_backward.py:225-234 bar, 1e-9); fp32 autograd too."""
    cfg = CONFIGS["c5"]
    ws = build_wordset("c5", sk)
    B, L = 3, 77
    X = brownian(cfg["seed"], B, L, cfg["d"])
    g = np.random.default_rng(105).standard_normal((B, len(ws)))
    ck = sk.signature_backward(X, ws, g, checkpoint_stride=stride).path_grads
    plain = sk.signature_backward(X, ws, g).path_grads
    _, dref = ora.backward(X, ws.codes, ws.lengths, cfg["d"], g, stride=stride)
    assert ora.rel_err(ck, dref) <= TOL64
    assert ora.rel_err(ck, plain) <= 1e-9
    Xt = torch.from_numpy(X.astype(np.float32)).cuda().requires_grad_(True)
    sk.signature(Xt, ws, checkpoint_stride=stride).backward(torch.from_numpy(g).float().cuda())
    assert ora.rel_err(Xt.grad.cpu().numpy(), dref) <= TOL32
    for name in ("c1", "c2"):  # other truncated instantiations
        w2 = build_wordset(name, sk)
        X2 = brownian(CONFIGS[name]["seed"], 2, 40, w2.d)
        g2 = np.random.default_rng(7).standard_normal((2, len(w2)))
        _, d2 = ora.backward(X2, w2.codes, w2.lengths, w2.d, g2, stride=stride)
        assert ora.rel_err(sk.signature_backward(X2, w2, g2, checkpoint_stride=stride).path_grads, d2) <= TOL64


@pytest.mark.parametrize("stride", [1, 3, 7])
def test_checkpoint_stride_fragment_kernels(stride):
    """checkpoint_stride on the fragment kernels (frag_ckpt_kernel replay + reload in
    frag_backward_kernel): the c4 anisotropic set, a non-prefix-closed user set (closure state) and
    the c3 trie (whose generated kernels take no checkpoints: the fragment kernels serve it), each
    fp64 drop-in against the oracle's own stride-`stride` backward (1e-10) and stride 0 (1e-9, the
    reference's test_backward.py:225-234 bar), fp32 autograd against the oracle (1e-4)."""
    rng = np.random.default_rng(300 + stride)
    sets = [("c4", build_wordset("c4", sk)), ("c3", build_wordset("c3", sk)),
            ("non-closed", sk.build_custom([(0, 1, 1), (1,), (1, 0, 2), (2, 2, 2, 2), (0, 2), (3, 1, 0)], 4))]
    for name, ws in sets:
        if name == "c4":
            assert ws.plan().kernel_kind == 2, name  # the fragment family serves the set
        # (c3 and the small non-closed set plan the generated kernels, which take no checkpoints:
        # their checkpointed backward runs on the fragment kernels too)
        B, L = 3, 41
        X = brownian(int(rng.integers(1 << 30)), B, L, ws.d)
        g = rng.standard_normal((B, len(ws)))
        ck = sk.signature_backward(X, ws, g, checkpoint_stride=stride).path_grads
        plain = sk.signature_backward(X, ws, g).path_grads
        _, dref = ora.backward(X, ws.codes, ws.lengths, ws.d, g, stride=stride)
        assert ora.rel_err(ck, dref) <= TOL64, name
        assert ora.rel_err(ck, plain) <= 1e-9, name
        Xt = torch.from_numpy(X.astype(np.float32)).cuda().requires_grad_(True)
        sk.signature(Xt, ws, checkpoint_stride=stride).backward(torch.from_numpy(g).float().cuda())
        assert ora.rel_err(Xt.grad.cpu().numpy(), dref) <= TOL32, name
