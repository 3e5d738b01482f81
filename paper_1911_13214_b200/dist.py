"""Multi-GPU orchestration of independent solves.

A sweep of memory limits over several chains (the paper's "Algorithm 1 for 10
different memory limits") is a set of independent (chain, limit)
tables.  One process per GPU (torch.distributed): the problems are sharded by
the native LPT partitioner (`rotor_partition_lpt`) on their nominal transition
counts, each rank solves its share with its own GPU, and only the results
(cost, status, op count, schedule) are gathered — there is no data-path
collective during the solve.
"""
from __future__ import annotations

import numpy as np


def problem_weights(chains, limits, slots: int):
    """Nominal transitions of every (chain, limit) problem, row-major by chain."""
    from . import transitions

    return np.array([transitions(int(ch.L), slots) for ch in chains for _ in limits[0]], dtype=np.float64)


def shard(weights, world: int):
    """part_of[p] = rank owning problem p (LPT, deterministic)."""
    from . import partition_lpt

    return partition_lpt(np.asarray(weights, dtype=np.float64), world)


def _default_solver(chains, limits, slots, pairs, **opts):
    """Solve the listed (chain index, limit index) pairs on this rank's GPU."""
    from . import solve

    out = []
    for i, j in pairs:
        r = solve(chains[i], limits[i][j], slots, **opts)
        out.append((r.status, r.cost, r.n_ops, r.ops))
    return out


def solve_batch_distributed(chains, limits, slots: int, group=None, solver=None, **opts):
    """Every rank returns the full (costs, status, n_ops, ops) of the sweep.

    `solver(chains, limits, slots, pairs, **opts)` solves a list of
    (chain, limit) index pairs and returns (status, cost, n_ops, ops) tuples;
    the default runs the CUDA path through the C ABI.  `group`: a
    torch.distributed process group (None = default group, or single process
    when torch.distributed is not initialised).
    """
    import torch.distributed as dist

    solver = solver or _default_solver
    nc, nl = len(chains), len(limits[0]) if chains else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    part = shard(problem_weights(chains, limits, slots), world)
    mine = [p for p in range(nc * nl) if part[p] == rank]
    local = solver(chains, limits, slots, [(p // nl, p % nl) for p in mine], **opts)
    payload = list(zip(mine, local))
    if world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, payload, group=group)
    else:
        gathered = [payload]
    costs = np.full((nc, nl), np.inf)
    status = np.zeros((nc, nl), dtype=np.int32)
    n_ops = np.zeros((nc, nl), dtype=np.int64)
    ops = [None] * (nc * nl)
    for part_payload in gathered:
        for p, (st, cost, k, o) in part_payload:
            costs[p // nl, p % nl] = cost
            status[p // nl, p % nl] = st
            n_ops[p // nl, p % nl] = k
            ops[p] = o
    return costs, status, n_ops, ops, part
