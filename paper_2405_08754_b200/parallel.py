"""Host-side data-parallel plumbing for libhrp (one process per GPU).

Environments are independent, so each rank owns a contiguous shard of envs (global env
index = rank * E_local + i): its own windows, replay shard and per-rank random streams.
The only exchange of the hot path -- the gradient allreduce -- runs inside libhrp over
NCCL; this module only (a) hands every rank the NCCL unique id created on rank 0 and
(b) combines per-rank timings / counters.  Everything here runs unchanged on the CPU
`gloo` backend (tests/test_parallel_gloo.py).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def env_shard(n_envs_local: int, rank: int) -> int:
    """Global index of this rank's first environment."""
    return rank * n_envs_local


def broadcast_bytes(payload, nbytes: int, device=None) -> bytes:
    """Broadcast `nbytes` bytes from rank 0 (payload ignored elsewhere)."""
    dev = device if device is not None else torch.device("cpu")
    buf = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
    if dist.get_rank() == 0:
        buf.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
    dist.broadcast(buf, 0)
    return bytes(buf.cpu().numpy().tobytes())


def nccl_unique_id(device=None) -> bytes:
    """The 128-byte ncclUniqueId of rank 0 (hrp_nccl_unique_id), on every rank."""
    payload = None
    if dist.get_rank() == 0:
        from . import hrp
        payload = hrp.hrp_nccl_unique_id()
    return broadcast_bytes(payload, 128, device)


def max_over_ranks(x: float, device=None) -> float:
    """Max over ranks (multi-GPU times are the slowest rank's device time)."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    dev = device if device is not None else torch.device("cpu")
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device=None) -> float:
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    dev = device if device is not None else torch.device("cpu")
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
