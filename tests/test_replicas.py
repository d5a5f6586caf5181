"""Replica-over-RHS multi-GPU path (paper_1612_02736_b200/replicas.py): host logic on CPU with a
world_size-2 gloo group. The per-rank solve is a stand-in linear map (the GPU solve itself is
covered by the -m gpu parity tests); what is tested here is the sharding, the gather order and
the max-over-ranks timing reduction that bench.py --gpus N relies on."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1612_02736_b200.replicas import gather_columns, max_over_ranks, rhs_shard, solve_replicated


def test_rhs_shard_covers_and_balances():
    for n in (0, 1, 5, 16, 17):
        for world in (1, 2, 3, 8):
            sl = [rhs_shard(n, r, world) for r in range(world)]
            assert sl[0].start == 0 and sl[-1].stop == n
            assert all(a.stop == b.start for a, b in zip(sl, sl[1:]))
            sizes = [s.stop - s.start for s in sl]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        rhs_shard(4, 2, 2)


class _LinearSolver:
    """Stand-in for FactorizedSolver.solve_device: uc[l, i, j] = (l + 1) * sum_k g[k, j] + i * f[0, j]."""
    _n_leaves, p = 3, 2

    def solve_device(self, f, g):
        nl, P = self._n_leaves, self.p ** 2
        l = torch.arange(nl, dtype=g.dtype)[:, None, None] + 1
        i = torch.arange(P, dtype=g.dtype)[None, :, None]
        return {"uc": l * g.sum(0)[None, None, :] + i * f[0][None, None, :]}


def _worker(rank, world, port, n):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.manual_seed(0)
        # integer-valued data: every partial sum is exact, so sharding cannot change the result
        f = torch.randint(-50, 50, (4, n)).double()
        g = torch.randint(-50, 50, (6, n)).double()
        solver = _LinearSolver()
        full = solve_replicated(solver, f, g)
        ref = solver.solve_device(f, g)["uc"]
        assert full.shape == ref.shape
        assert torch.equal(full, ref)
        assert max_over_ranks(float(rank + 1)) == float(world)
        part = torch.full((2, rhs_shard(n, rank, world).stop - rhs_shard(n, rank, world).start), float(rank))
        cols = gather_columns(part, n)
        expect = torch.cat([torch.full((2, rhs_shard(n, r, world).stop - rhs_shard(n, r, world).start), float(r))
                            for r in range(world)], dim=-1)
        assert torch.equal(cols, expect)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("n", [16, 5, 1])
def test_replicated_solve_gloo_world2(n):
    mp.spawn(_worker, args=(2, _free_port(), n), nprocs=2, join=True)


def test_single_process_is_identity():
    solver = _LinearSolver()
    f = torch.randn(4, 3, dtype=torch.float64)
    g = torch.randn(6, 3, dtype=torch.float64)
    assert torch.equal(solve_replicated(solver, f, g), solver.solve_device(f, g)["uc"])
    assert max_over_ranks(2.5) == 2.5
