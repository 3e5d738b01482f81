"""Multi-process host logic on CPU (gloo, world_size 2): the sharded multi-limit sweep.

The per-problem solver is injected (the oracle here: the CUDA path needs a
GPU); the test checks that sharding + gathering reproduce the serial sweep and
that the LPT shards are balanced.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import chaingen as G


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_solver(chains, limits, slots, pairs, **opts):
    import oracle as O

    out = []
    for i, j in pairs:
        o = O.OracleSolve(chains[i], limits[i][j], slots)
        ops = o.reconstruct()
        c = o.cost
        st = 0 if ops is not None else 2
        out.append((st, c, len(ops) if ops else 0, ops))
    return out


def _sweep():
    chains, limits, S = G.config5(n_limits=5)
    return chains[:3], [l[:5] for l in limits[:3]], 60


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1911_13214_b200.dist import solve_batch_distributed

        chains, limits, S = _sweep()
        costs, status, n_ops, ops, part = solve_batch_distributed(chains, limits, S, solver=_oracle_solver)
        q.put((rank, costs, status, n_ops, [list(o) if o else None for o in ops], part.tolist()))
    finally:
        dist.destroy_process_group()


def test_sharded_sweep_gloo_world2():
    import __graft_entry__ as ge

    ge.build_library()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    chains, limits, S = _sweep()
    serial = _oracle_solver(chains, limits, S, [(i, j) for i in range(len(chains)) for j in range(len(limits[0]))])
    for rank, costs, status, n_ops, ops, part in res:
        assert set(part) == {0, 1}  # both ranks got work
        for p, (st, c, k, o) in enumerate(serial):
            i, j = divmod(p, len(limits[0]))
            assert costs[i, j] == c and status[i, j] == st and n_ops[i, j] == k
            assert ops[p] == (list(o) if o else None)
    # both ranks agree on everything
    assert np.array_equal(res[0][1], res[1][1])


def test_lpt_shards_balanced():
    import __graft_entry__ as ge

    ge.build_library()
    from paper_1911_13214_b200.dist import problem_weights, shard

    chains, limits, S = G.config5(n_limits=256)
    w = problem_weights(chains, limits, S)
    assert len(w) == 8 * 256
    for world in (1, 2, 4, 8):
        part = shard(w, world)
        loads = np.bincount(part, weights=w, minlength=world)
        assert loads.max() / loads.mean() < 1.01


def test_default_solver_grouping(monkeypatch):
    """dist's default per-rank solver packs a rank's (chain, limit) pairs into one
    padded chains x limits grid for the fused rotor_solve_batch, and maps every
    result back to its pair (a fake batch returns the limit as the cost)."""
    import __graft_entry__ as ge

    ge.build_library()
    import numpy as np

    import paper_1911_13214_b200 as R
    from paper_1911_13214_b200 import dist as D

    calls = []

    def fake(chains, grid, slots, with_ops=False, **opts):
        calls.append(len(chains))
        g = np.array(grid, dtype=np.float64)
        st = np.zeros(g.shape, dtype=np.int32)
        nops = np.arange(g.size, dtype=np.int64).reshape(g.shape)
        return g, st, nops, [np.full((1, 2), k, dtype=np.int32) for k in range(g.size)]

    monkeypatch.setattr(R, "solve_batch", fake)
    chains = ["c0", "c1", "c2"]
    limits = [[10, 11, 12, 13], [20, 21, 22, 23], [30, 31, 32, 33]]
    pairs = [(2, 1), (0, 3), (2, 0), (0, 0), (2, 3), (1, 2)]
    out = D._default_solver(chains, limits, 100, pairs)
    assert calls == [3]
    assert [c for _, c, _, _ in out] == [limits[i][j] for i, j in pairs]
    assert D._default_solver(chains, limits, 100, []) == []
