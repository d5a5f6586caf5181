"""Replicas over right-hand sides: the multi-GPU form of the solve.

The north star runs on one GPU, and a single solve does not shard without an exchange per tree
level. Many independent right-hand sides (config 5's 16 initial fields, parameter sweeps) do:
every rank holds the whole factorisation (built locally, or loaded from an archive) and solves a
contiguous slice of the RHS columns. The only collective is the final gather of the leaf
tabulations; timings are reduced as the max over ranks. One process per GPU; the process group
is any torch.distributed group (NCCL on the GPU box, gloo in the CPU tests).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def rhs_shard(n_total: int, rank: int, world: int) -> slice:
    """Contiguous, balanced slice of n_total RHS columns owned by `rank` (first ranks take the
    remainder)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside a world of {world}")
    base, extra = divmod(n_total, world)
    lo = rank * base + min(rank, extra)
    return slice(lo, lo + base + (1 if rank < extra else 0))


def max_over_ranks(x: float, group=None) -> float:
    """Max of a host scalar over the group (device-agnostic: a CPU tensor under gloo)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(x)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def gather_columns(local: torch.Tensor, n_total: int, group=None) -> torch.Tensor:
    """All-gather of per-rank column slices (..., n_local) into (..., n_total) in RHS order."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return local
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if local.shape[-1] != rhs_shard(n_total, rank, world).stop - rhs_shard(n_total, rank, world).start:
        raise ValueError("local slice does not match rhs_shard")
    width = -(-n_total // world)
    pad = torch.zeros(local.shape[:-1] + (width,), dtype=local.dtype, device=local.device)
    pad[..., :local.shape[-1]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad.contiguous(), group=group)
    cols = [parts[r][..., :rhs_shard(n_total, r, world).stop - rhs_shard(n_total, r, world).start]
            for r in range(world)]
    return torch.cat(cols, dim=-1)


def solve_replicated(solver, f: torch.Tensor, g: torch.Tensor, group=None) -> torch.Tensor:
    """Solve RHS columns f (|root ext|, n), g (n_leaves*m, n) split over the ranks of `group`.

    Each rank solves its slice with solver.solve_device (one program for its column count) and
    the leaf tabulations (n_leaves, P, n) are all-gathered, so every rank returns all columns.
    """
    n = g.shape[-1]
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    sl = rhs_shard(n, rank, world)
    if sl.stop > sl.start:
        uc = solver.solve_device(f[:, sl].contiguous(), g[:, sl].contiguous())["uc"].clone()
    else:  # more ranks than columns: contribute an empty slice
        nl, P = solver._n_leaves, solver.p ** 2
        uc = torch.zeros((nl, P, 0), dtype=g.dtype, device=g.device)
    return gather_columns(uc, n, group)
