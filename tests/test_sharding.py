"""Multi-process batch sharding on CPU (gloo, world_size 2) and the bench contract's host legs."""

import json
import os
import socket
import subprocess
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_24066_b200.sharding import gather_signatures, shard, shard_range

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("B", [0, 1, 5, 8, 65536, 65537])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_range_partitions_the_batch(B, world):
    spans = [shard_range(B, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == B
    for (a, b), (c, _) in zip(spans, spans[1:]):
        assert b == c
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 1
    assert max(sizes) == spans[0][1] - spans[0][0]
    with pytest.raises(ValueError):
        shard_range(B, world, world)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, B, W, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        full = torch.arange(B * W, dtype=torch.float32).reshape(B, W)
        X = torch.arange(B * 3 * 2, dtype=torch.float32).reshape(B, 3, 2)
        mine = shard(X, rank, world)
        lo, hi = shard_range(B, rank, world)
        assert torch.equal(mine, X[lo:hi])
        S_local = full[lo:hi].clone()  # stands in for this rank's signature rows
        G = gather_signatures(S_local, B)
        ok = torch.equal(G, full)
        # max over ranks, as bench.py times a step
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q.put((rank, ok, float(t.item())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("B", [7, 8])
def test_gather_world2_gloo(B):
    world, W = 2, 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B, W, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = sorted(q.get(timeout=5) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert [r for r, _, _ in res] == [0, 1]
    assert all(ok for _, ok, _ in res)
    assert all(m == float(world) for _, _, m in res)


def _bench(args, env_extra=None, timeout=300):
    env = dict(os.environ)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          env=env, timeout=timeout, cwd=ROOT)


def test_bench_reference_arm_line():
    """--impl reference times the oracle port on the host and prints the contract's JSON line."""
    r = _bench(["--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "1"])
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["unit"] == "paths/s" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": "paths/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}


def test_bench_reference_arm_nonzero_rank_is_silent():
    r = _bench(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "1"],
               {"RANK": "1", "WORLD_SIZE": "2"})
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == ""


def test_bench_ours_refuses_without_gpu():
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    r = _bench(["--config", "c1", "--steps", "1", "--warmup", "1"])
    assert r.returncode != 0
    assert "no CPU fallback" in (r.stderr + r.stdout)


def _nccl_worker(rank, world, port, q):
    """One rank of the 2-GPU run: its shard of a c5-shaped batch through the public autograd
    path, gathered back over NCCL, compared with the 1-rank result computed on cuda:0."""
    import numpy as np

    import paper_2602_24066_b200 as sk
    from paper_2602_24066_b200.sharding import sharded_signature
    from tests.configs import brownian

    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                            device_id=dev)
    try:
        ws = sk.build_truncated(16, 4)
        B = 37
        X = torch.from_numpy(brownian(5, B, 64, 16).astype(np.float32))
        g = torch.from_numpy(np.random.default_rng(105).standard_normal((B, len(ws))).astype(np.float32))
        lo, hi = shard_range(B, rank, world)
        Xl = X[lo:hi].to(dev).requires_grad_(True)
        S = sharded_signature(Xl, ws)
        S.backward(g[lo:hi].to(dev))
        G = gather_signatures(S.detach(), B)
        dG = gather_signatures(Xl.grad.reshape(hi - lo, -1), B)
        ok = True
        if rank == 0:
            Xr = X.to(dev).requires_grad_(True)
            S1 = sk.signature(Xr, ws)
            S1.backward(g.to(dev))
            ok = torch.equal(G, S1.detach()) and torch.equal(dG, Xr.grad.reshape(B, -1))
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_world2_nccl_bitwise():
    """Two ranks over NCCL: sharded fwd+bwd with no data-path collective, then the
    optional all-gather, bit for bit equal to the single-GPU batch (reference test_acceptance.py:332-353
    is its only scaling gate)."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_nccl_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    assert all(p.exitcode == 0 for p in procs)
    res = sorted(q.get(timeout=5) for _ in range(world))
    assert res == [(0, True), (1, True)]


def test_bench_self_launch_command(monkeypatch):
    """`bench.py --gpus N` outside torchrun re-runs itself under torch.distributed.run with N ranks."""
    sys.path.insert(0, ROOT)
    import bench

    seen = {}

    def fake_run(cmd, cwd=None):
        seen["cmd"] = cmd

        class R:
            returncode = 0
        return R()

    monkeypatch.setattr(bench.subprocess, "run", fake_run)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    with pytest.raises(SystemExit) as e:
        bench.main(["--gpus", "4", "--steps", "2"])
    assert e.value.code == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-3:] == ["--gpus", "4", "--steps", "2"][-3:] and cmd[-4] == "--gpus"
