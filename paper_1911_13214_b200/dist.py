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


def tile_ranges(n_tiles: int, world: int):
    """Contiguous, balanced tile ranges [lo, hi) per rank (the first n % world ranks get one more)."""
    base, extra = divmod(n_tiles, world)
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


class CudaShardEngine:
    """This rank's share of a sharded single-table solve (rotor_sharded_* through the binding)."""

    def __init__(self, chain, mem_limit: int, slots: int, device=None, stream=None, **opts):
        import numpy as np
        import torch

        from . import Shard, max_ops, tile_blocks, tile_bytes, workspace_bytes

        self.torch = torch
        self.dev = torch.device("cuda") if device is None else torch.device(device)
        self.stream = stream
        self.L, self.S = int(chain.L), int(slots)
        self.d_chain = {k: torch.from_numpy(np.asarray(getattr(chain, k)).astype(
            np.float64 if k in ("uf", "ub") else np.int64)).to(self.dev) for k in ("uf", "ub", "wx", "wbx", "wy", "of", "ob")}
        self.ws = torch.empty(workspace_bytes(self.L, self.S, kernel="tiled"), dtype=torch.uint8, device=self.dev)
        self._args = (mem_limit, opts)
        self.shard = Shard(self.d_chain, self.L, mem_limit, self.S, self.ws, stream=stream, **opts)
        self.nb = tile_blocks(self.L)
        self.tile_bytes = tile_bytes(self.S)
        self.cap_ops = max_ops(self.L)
        self._bufs = {}

    def restart(self):
        """A fresh solve in the same workspace (precompute, leaf, flags again)."""
        from . import Shard

        self.shard.close()
        mem_limit, opts = self._args
        self.shard = Shard(self.d_chain, self.L, mem_limit, self.S, self.ws, stream=self.stream, **opts)

    def buffer(self, name: str, n_tiles: int):
        need = max(1, n_tiles) * self.tile_bytes
        b = self._bufs.get(name)
        if b is None or b.numel() < need:
            b = self.torch.empty(need, dtype=self.torch.uint8, device=self.dev)
            self._bufs[name] = b
        return b[:need]

    def step(self, delta, lo, hi):
        self.shard.step(delta, lo, hi, stream=self.stream)

    def pack(self, delta, lo, hi, buf):
        self.shard.pack(delta, lo, hi, buf, unpack=False, stream=self.stream)

    def unpack(self, delta, lo, hi, buf):
        """On the exchange stream (after the collective that filled `buf`)."""
        self.shard.pack(delta, lo, hi, buf, unpack=True, stream=self.comm_stream())

    # -- the exchange runs on its own stream, ordered against the compute
    #    stream by events (solve_sharded's pipeline) --
    def compute_stream(self):
        t = self.torch
        return self.stream if self.stream is not None else t.cuda.current_stream(self.dev)

    def comm_stream(self):
        if getattr(self, "_comm", None) is None:
            self._comm = self.torch.cuda.Stream(device=self.dev)
        return self._comm

    def comm_after_compute(self):
        """The exchange stream waits for everything enqueued on the compute stream so far (the pack)."""
        ev = self.torch.cuda.Event()
        ev.record(self.compute_stream())
        self.comm_stream().wait_event(ev)

    def compute_after_comm(self):
        """The compute stream waits for the exchange stream (the unpacked tiles)."""
        ev = self.torch.cuda.Event()
        ev.record(self.comm_stream())
        self.compute_stream().wait_event(ev)

    def comm_context(self):
        return self.torch.cuda.stream(self.comm_stream())

    def finish(self):
        t = self.torch
        out = dict(cost=t.empty(1, dtype=t.float64, device=self.dev),
                   ops=t.empty((self.cap_ops, 2), dtype=t.int32, device=self.dev),
                   n_ops=t.empty(1, dtype=t.int64, device=self.dev), status=t.empty(1, dtype=t.int32, device=self.dev))
        self.shard.finish(out, stream=self.stream)
        t.cuda.synchronize(self.dev)
        k = int(out["n_ops"].item())
        return int(out["status"].item()), float(out["cost"].item()), out["ops"][: max(k, 0)].cpu().numpy()


def _collective_timeout():
    """Seconds a per-diagonal collective may take (ROTOR_COLLECTIVE_TIMEOUT_S, default 300)."""
    import os

    return float(os.environ.get("ROTOR_COLLECTIVE_TIMEOUT_S", "300"))


class CollectiveError(RuntimeError):
    """A per-diagonal exchange failed or timed out (a rank died, NCCL error, hang)."""


def _all_gather_start(recv, send, group):
    import torch.distributed as dist

    return dist.all_gather_into_tensor(recv, send, group=group, async_op=True)


def _all_gather_finish(work, delta):
    """Wait for an all-gather started by _all_gather_start, with a timeout: a
    failed or hung peer surfaces as CollectiveError naming the tile diagonal
    instead of a silent hang (NCCL's own async error handling aborts the
    communicator).  On NCCL the wait orders the CURRENT stream after the
    collective (the host does not block); gloo blocks the host."""
    import datetime

    try:
        ok = work.wait(timeout=datetime.timedelta(seconds=_collective_timeout()))
    except Exception as e:  # NCCL / gloo error reported by the backend
        raise CollectiveError(f"all-gather of tile diagonal {delta} failed: {e}") from e
    if ok is False:
        raise CollectiveError(f"all-gather of tile diagonal {delta} timed out after {_collective_timeout()} s")


def _all_gather_checked(recv, send, group, delta):
    _all_gather_finish(_all_gather_start(recv, send, group), delta)


def local_span(ranges, prev_ranges, rank):
    """The tiles [a, b) of this rank's range on a tile diagonal whose two
    neighbours on the previous diagonal (tile I and I+1: (I, J-1) and (I+1, J))
    it computed itself, so they need nothing from that diagonal's exchange."""
    lo, hi = ranges[rank]
    if prev_ranges is None:
        return lo, hi
    plo, phi = prev_ranges[rank]
    a, b = max(lo, plo), min(hi, phi - 1)
    return (a, b) if a < b else (lo, lo)


def _nullcontext():
    import contextlib

    return contextlib.nullcontext()


def solve_sharded(engine, group=None):
    """one table sharded over the ranks of `group`.

    Per tile diagonal delta (every tile of which depends only on smaller
    diagonals) each rank computes a contiguous range of the tiles,
    packs them, the ranks all-gather the packed tiles (NCCL over NVLink on
    GPUs, gloo in the CPU tests) and every rank unpacks the others' tiles, so
    each rank ends with the full table and runs Algorithm 2 itself.

    The exchange of diagonal delta overlaps the compute of delta + 1: tile I of
    delta + 1 reads tiles I and I+1 of delta (its left / lower neighbours) and
    whole rows / columns of diagonals <= delta - 1, so the tiles whose two
    neighbours this rank computed itself (local_span: all but the range's
    edges) start at once, and only the edge tiles wait for delta's unpacked
    tiles.  The all-gather and the unpacks run on the engine's exchange
    stream, ordered against the compute stream by events; the send / receive
    buffers alternate between two sets (delta's are free again once delta + 1
    waited for its unpack).

    `engine` provides nb, tile_bytes, step, pack, unpack, buffer, finish and
    (optional: absent in the CPU tests) comm_after_compute, compute_after_comm,
    comm_context.
    """
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    tb = engine.tile_bytes
    after_compute = getattr(engine, "comm_after_compute", lambda: None)
    after_comm = getattr(engine, "compute_after_comm", lambda: None)
    comm_ctx = getattr(engine, "comm_context", _nullcontext)
    pending = None  # (delta, ranges, cap, recv, work) of the exchange in flight

    def complete(p):
        d, rngs, cap, recv, work = p
        with comm_ctx():
            _all_gather_finish(work, d)
            for r, (l, h) in enumerate(rngs):
                if r != rank and h > l:
                    engine.unpack(d, l, h, recv[r * cap * tb: (r * cap + (h - l)) * tb])
        after_comm()

    for delta in range(engine.nb):
        ranges = tile_ranges(engine.nb - delta, world)
        lo, hi = ranges[rank]
        if world == 1:
            engine.step(delta, lo, hi)
            continue
        a, b = local_span(ranges, pending[1] if pending else None, rank)
        if b > a:
            engine.step(delta, a, b)  # overlaps the exchange of delta - 1
        if pending:
            complete(pending)
        if a > lo:
            engine.step(delta, lo, a)
        if hi > b and b >= a:
            engine.step(delta, max(b, lo), hi)
        cap = max(h - l for l, h in ranges)
        send = engine.buffer(f"send{delta & 1}", cap)
        engine.pack(delta, lo, hi, send)
        recv = engine.buffer(f"recv{delta & 1}", cap * world)
        after_compute()
        with comm_ctx():
            work = _all_gather_start(recv, send, group)
        pending = (delta, ranges, cap, recv, work)
    if pending:
        complete(pending)
    return engine.finish()


def solve_sharded_virtual(engines):
    """The same pipelined schedule with len(engines) ranks emulated in one
    process: the all-gather becomes each engine unpacking the other engines'
    send buffers on its exchange stream, after their packs (events), while the
    local tiles of the next diagonal run on its compute stream."""
    world = len(engines)
    nb = engines[0].nb
    tb = engines[0].tile_bytes
    pending = None  # (delta, ranges, sends)

    def complete(p):
        d, rngs, sends = p
        for r, e in enumerate(engines):
            if hasattr(e, "comm_stream"):
                for q, f in enumerate(engines):  # r's exchange stream after every rank's pack
                    if q != r:
                        e.comm_stream().wait_event(f._packed)
            with (e.comm_context() if hasattr(e, "comm_context") else _nullcontext()):
                for q, (l, h) in enumerate(rngs):
                    if q != r and h > l:
                        e.unpack(d, l, h, sends[q][: (h - l) * tb])
            if hasattr(e, "compute_after_comm"):
                e.compute_after_comm()

    for delta in range(nb):
        ranges = tile_ranges(nb - delta, world)
        if world == 1:
            engines[0].step(delta, *ranges[0])
            continue
        spans = [local_span(ranges, pending[1] if pending else None, r) for r in range(world)]
        for r, e in enumerate(engines):
            a, b = spans[r]
            if b > a:
                e.step(delta, a, b)
        if pending:
            complete(pending)
        cap = max(h - l for l, h in ranges)
        sends = []
        for r, e in enumerate(engines):
            lo, hi = ranges[r]
            a, b = spans[r]
            if a > lo:
                e.step(delta, lo, a)
            if hi > b and b >= a:
                e.step(delta, max(b, lo), hi)
            snd = e.buffer(f"send{delta & 1}", cap)
            e.pack(delta, lo, hi, snd)
            if hasattr(e, "compute_stream"):
                e._packed = e.torch.cuda.Event()
                e._packed.record(e.compute_stream())
            sends.append(snd)
        pending = (delta, ranges, sends)
    if pending:
        complete(pending)
    return [e.finish() for e in engines]


def problem_weights(chains, limits, slots: int):
    """Nominal transitions of every (chain, limit) problem, row-major by chain."""
    from . import transitions

    return np.array([transitions(int(ch.L), slots) for ch in chains for _ in limits[0]], dtype=np.float64)


def shard(weights, world: int):
    """part_of[p] = rank owning problem p (LPT, deterministic)."""
    from . import partition_lpt

    return partition_lpt(np.asarray(weights, dtype=np.float64), world)


def _default_solver(chains, limits, slots, pairs, **opts):
    """Solve the listed (chain index, limit index) pairs on this rank's GPU with the
    fused batched kernel (rotor_solve_batch): the pairs are grouped per chain into
    one chains x limits grid, ragged rows padded by repeating their last limit
    (the padding's results are dropped)."""
    from . import solve_batch

    if not pairs:
        return []
    rows = {}
    for i, j in pairs:
        rows.setdefault(i, []).append(j)
    order = sorted(rows)
    width = max(len(v) for v in rows.values())
    grid = [[limits[i][j] for j in rows[i]] + [limits[i][rows[i][-1]]] * (width - len(rows[i])) for i in order]
    costs, status, n_ops, ops = solve_batch([chains[i] for i in order], grid, slots, with_ops=True, **opts)
    where = {(i, j): (a, b) for a, i in enumerate(order) for b, j in enumerate(rows[i])}
    out = []
    for i, j in pairs:
        a, b = where[(i, j)]
        out.append((int(status[a, b]), float(costs[a, b]), int(n_ops[a, b]), ops[a * width + b]))
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
