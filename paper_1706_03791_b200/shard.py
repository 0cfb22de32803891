"""Multi-GPU host logic: field sharding and max-over-ranks timing.

The path shards only where it shards naturally (BASELINE north_star):
independent fields go round-robin to ranks (field i -> rank i mod N), each
rank runs the whole pipeline on its fields with no data-path collective, and
``torch.distributed`` is used only for barriers and for reducing timings
(max over ranks) -- one process per GPU, NCCL on the GPU box, gloo in the CPU
tests.
"""

from __future__ import annotations


def field_shard(n_fields: int, rank: int, world: int) -> list[int]:
    """Indices of the fields rank `rank` owns (round robin)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    return list(range(rank, n_fields, world))


def reduce_max(values, device=None) -> list[float]:
    """Element-wise max of per-rank float values over the process group
    (identity without an initialised group)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.tolist()]


def reduce_sum(values, device=None) -> list[float]:
    """Element-wise sum of per-rank values (e.g. bytes processed)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [float(v) for v in t.tolist()]
