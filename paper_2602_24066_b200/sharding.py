"""Batch sharding across the GPUs of one node.

Paths are independent: the forward and the backward of one path never read
another path, dL/dX is per path and the word-set plan is replicated per
device.  So the batch axis shards with no collective on the data path; the
only collective is the OPTIONAL all-gather of the signatures (NCCL
``all_gather_into_tensor`` over NVLink), kept out of the timed fwd/bwd.

The reference has no distributed layer (numba threads only, _kernels.py:19-37);
this module is the B200-native replacement of its ``prange`` over paths.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .autograd import signature
from .signature import forward_tensor
from .wordset import WordSet


def shard_range(B: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced slice [lo, hi) of B paths owned by `rank` (first B % world ranks get one more)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of size {world}")
    base, extra = divmod(int(B), world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard(X: torch.Tensor, rank: int, world: int) -> torch.Tensor:
    """This rank's paths of a (B, L, d) batch."""
    lo, hi = shard_range(X.shape[0], rank, world)
    return X[lo:hi]


def sharded_forward(X_local: torch.Tensor, ws: WordSet) -> torch.Tensor:
    """Signatures of this rank's paths (no communication)."""
    out, _ = forward_tensor(X_local.contiguous(), ws)
    return out


def sharded_signature(X_local: torch.Tensor, ws: WordSet, checkpoint_stride: int | None = None) -> torch.Tensor:
    """Differentiable signatures of this rank's paths; backward is rank-local too."""
    return signature(X_local, ws, checkpoint_stride)


def gather_signatures(S_local: torch.Tensor, B: int, group=None) -> torch.Tensor:
    """All-gather the row shards of S (B, W) produced by `shard_range` onto every rank.

    Uneven shards are padded to the largest shard for ``all_gather_into_tensor``
    (NCCL on CUDA tensors, gloo on CPU tensors) and trimmed afterwards, so the
    result is the (B, W) matrix in global path order.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = shard_range(B, rank, world)
    if S_local.shape[0] != hi - lo:
        raise ValueError(f"rank {rank} holds {S_local.shape[0]} rows, expected {hi - lo}")
    cap = shard_range(B, 0, world)[1]  # rank 0 holds the largest shard
    W = S_local.shape[1]
    buf = S_local.new_zeros((cap, W))
    buf[: hi - lo] = S_local
    out = S_local.new_empty((world * cap, W))
    if S_local.is_cuda:
        dist.all_gather_into_tensor(out, buf, group=group)
    else:
        parts = list(out.split(cap))
        dist.all_gather(parts, buf, group=group)
    rows = [out[r * cap: r * cap + (shard_range(B, r, world)[1] - shard_range(B, r, world)[0])] for r in range(world)]
    return torch.cat(rows, dim=0)
