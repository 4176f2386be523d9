"""Multi-GPU plumbing (one process per GPU): source sharding and the NCCL-id broadcast.

The source cloud is split contiguously and evenly across ranks; the target is replicated; every rank
calls lsgcpd_register with the same communicator, whose only data-path traffic is one 75-double
all-reduce of the M-step moments per EM iteration.
"""
from __future__ import annotations


def shard_range(n: int, rank: int, world: int):
    """Contiguous, balanced shard [lo, hi) of `n` items for `rank` of `world` (sizes differ by ≤ 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return n * rank // world, n * (rank + 1) // world


def broadcast_bytes(blob: bytes, src: int = 0, group=None) -> bytes:
    """Broadcast a small byte string from `src` over torch.distributed (gloo: CPU tensor, nccl: CUDA).

    `src` is a rank WITHIN `group` (the rank a communicator of that group sees); torch's broadcast takes a
    global rank, so it is translated for a non-default group."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return blob
    me = dist.get_rank(group)
    gsrc = src if group is None else dist.get_global_rank(group, src)
    n = torch.tensor([len(blob) if me == src else 0], dtype=torch.int64)
    on_gpu = dist.get_backend(group) == "nccl"
    dev = torch.device("cuda", torch.cuda.current_device()) if on_gpu else torch.device("cpu")
    n = n.to(dev)
    dist.broadcast(n, src=gsrc, group=group)
    buf = torch.zeros(int(n.item()), dtype=torch.uint8, device=dev)
    if me == src:
        buf.copy_(torch.frombuffer(bytearray(blob), dtype=torch.uint8).to(dev))
    dist.broadcast(buf, src=gsrc, group=group)
    return bytes(buf.cpu().numpy().tobytes())
