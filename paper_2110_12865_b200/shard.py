"""Multi-GPU partitioning of the evaluation.

The path partitions without a data-path collective: independent input value
sets are sharded across the ranks (one process per GPU, the device plan
replicated on each), every rank evaluates its shard with ``run_batch_csr``,
and NCCL is used only when one rank needs every CSR block afterwards
(``gather_csr``).  Timing across ranks is the max (``max_over_ranks``).

Works with any ``torch.distributed`` backend: NCCL on the B200 box, gloo in the
CPU tests (tests/test_shard.py, world size 2).
"""

from __future__ import annotations


def shard_value_sets(total: int, world: int, rank: int) -> tuple[int, int]:
    """(first value set, count) of ``rank``: contiguous, sizes differ by at most one."""
    if total < 0 or world < 1 or not 0 <= rank < world:
        raise ValueError("need total >= 0, world >= 1, 0 <= rank < world")
    base, extra = divmod(total, world)
    count = base + (1 if rank < extra else 0)
    first = rank * base + min(rank, extra)
    return first, count


def gather_csr(out_shard, total: int, dst: int = 0, group=None):
    """Gather every rank's [n_out, count] CSR block into [n_out, total] on ``dst`` (None elsewhere).

    Blocks are padded to the largest shard so one ``gather`` moves them all; the
    value-set order of the result is the global order of ``shard_value_sets``.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    counts = [shard_value_sets(total, world, r)[1] for r in range(world)]
    if out_shard.shape[1] != counts[rank]:
        raise ValueError(f"rank {rank} holds {out_shard.shape[1]} value sets, expected {counts[rank]}")
    width = max(counts) if counts else 0
    send = out_shard.new_zeros((out_shard.shape[0], width))
    send[:, : counts[rank]] = out_shard
    recv = [torch.empty_like(send) for _ in range(world)] if rank == dst else None
    dist.gather(send, recv, dst=dst, group=group)
    if rank != dst:
        return None
    return torch.cat([recv[r][:, : counts[r]] for r in range(world)], dim=1)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """The slowest rank's time (the job's time)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
