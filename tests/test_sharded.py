"""Sharded single-table solve.

CPU (gloo, world 2 and 3): the orchestration of paper_1911_13214_b200.dist.solve_sharded
with a fake engine whose tiles are the oracle's values — every rank must have all of a
tile's dependencies (its row to the left, its column below) before computing it, and
must end with the full table.
GPU: the same schedule with 2 and 3 ranks emulated on one B200 (separate workspaces,
packed tiles exchanged by unpacking the other ranks' buffers): every rank's table is
bit-identical to the single-GPU solve and to the oracle.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import chaingen as G

TB = 32


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cell(n, s, t):
    r = s - 1
    return r * n - r * (r - 1) // 2 + (t - s)


class FakeEngine:
    """Tiles come from a reference table; dependencies are checked, not assumed."""

    def __init__(self, ref, n, S):
        self.ref, self.n, self.S = ref, n, S
        self.nb = (n + TB - 1) // TB
        self.tile_bytes = TB * TB * (S + 1) * 8
        self.C = np.full_like(ref, np.nan)
        self.have = np.zeros(ref.shape[0], dtype=bool)
        for s in range(1, n + 1):  # the leaf diagonal (rotor_sharded_begin)
            self.C[_cell(n, s, s)] = ref[_cell(n, s, s)]
            self.have[_cell(n, s, s)] = True
        self._bufs = {}

    def _tile_cells(self, delta, I):
        J = I + delta
        for a in range(TB):
            for c in range(TB):
                s, t = I * TB + 1 + a, J * TB + 1 + c
                if s <= self.n and t <= self.n and s <= t:
                    yield a, c, s, t

    def buffer(self, name, n_tiles):
        need = max(1, n_tiles) * self.tile_bytes
        if name not in self._bufs or self._bufs[name].numel() < need:
            self._bufs[name] = torch.zeros(need, dtype=torch.uint8)
        return self._bufs[name][:need]

    def step(self, delta, lo, hi):
        n = self.n
        for I in range(lo, hi):
            cells = list(self._tile_cells(delta, I))
            own = {(s, t) for _, _, s, t in cells}
            for _, _, s, t in cells:
                if s == t:
                    continue
                for sp in range(s + 1, t + 1):  # Theorem 1 reads C[s, s'-1] and C[s', t]
                    for dep in ((s, sp - 1), (sp, t)):
                        assert dep in own or self.have[_cell(n, *dep)], f"tile ({I},{I + delta}) needs {dep}"
            for _, _, s, t in cells:
                self.C[_cell(n, s, t)] = self.ref[_cell(n, s, t)]
                self.have[_cell(n, s, t)] = True

    def pack(self, delta, lo, hi, buf):
        v = buf.view(torch.float64).numpy().reshape(-1, TB, TB, self.S + 1)
        for k, I in enumerate(range(lo, hi)):
            for a, c, s, t in self._tile_cells(delta, I):
                v[k, a, c] = self.C[_cell(self.n, s, t)]

    def unpack(self, delta, lo, hi, buf):
        v = buf.view(torch.float64).numpy().reshape(-1, TB, TB, self.S + 1)
        for k, I in enumerate(range(lo, hi)):
            for a, c, s, t in self._tile_cells(delta, I):
                self.C[_cell(self.n, s, t)] = v[k, a, c]
                self.have[_cell(self.n, s, t)] = True

    def finish(self):
        assert self.have.all()
        return self.C


def _reference():
    rng = G.SplitMix64(41)
    ch = G.random_chain(rng, 100, real_times=True)  # n = 101 -> 4 blocks, 4 tile diagonals
    return ch, int(sum(int(x) for x in ch.wbx) * 0.3), 12


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        from paper_1911_13214_b200.dist import solve_sharded

        ch, M, S = _reference()
        ref, _ = O.OracleSolve(ch, M, S).tables()
        C = solve_sharded(FakeEngine(ref, ch.L + 1, S))
        q.put((rank, bool(np.array_equal(C.view(np.uint64), ref.view(np.uint64)))))
    except Exception as e:  # surface the assertion to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_schedule_gloo(world):
    import __graft_entry__ as ge

    ge.build_library()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert [r for r, _ in res] == list(range(world))
    for r, ok in res:
        assert ok is True, (r, ok)


def test_tile_ranges():
    from paper_1911_13214_b200.dist import tile_ranges

    for n in range(0, 40):
        for w in range(1, 9):
            rs = tile_ranges(n, w)
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            sizes = [h - l for l, h in rs]
            assert max(sizes) - min(sizes) <= 1


def test_local_span():
    """The tiles a rank computes before the previous diagonal's exchange lands:
    both neighbours (tile I and I+1 of the previous diagonal) are its own, and
    the rest of its range is contiguous around them."""
    from paper_1911_13214_b200.dist import local_span, tile_ranges

    for nb in (1, 2, 5, 17, 32, 40):
        for w in range(1, 9):
            prev = None
            for d in range(nb):
                rs = tile_ranges(nb - d, w)
                for r in range(w):
                    lo, hi = rs[r]
                    a, b = local_span(rs, prev, r)
                    assert lo <= a <= b <= hi
                    if prev is None:
                        assert (a, b) == (lo, hi)
                        continue
                    plo, phi = prev[r]
                    for I in range(a, b):
                        assert plo <= I and I + 1 < phi
                    for I in range(lo, hi):  # every tile with both neighbours local is in the span
                        if plo <= I and I + 1 < phi:
                            assert a <= I < b
                prev = rs


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_virtual_ranks_gpu(world, oracle_mod):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge

    ge.build_library()
    import paper_1911_13214_b200 as R
    from paper_1911_13214_b200.dist import CudaShardEngine, solve_sharded_virtual

    O = oracle_mod
    for p in (G.config2(), G.config3()):
        ch = p.chain
        o = O.OracleSolve(ch, p.mem_limit, p.slots)
        Co, _ = o.tables()
        engines = [CudaShardEngine(ch, p.mem_limit, p.slots) for _ in range(world)]
        results = solve_sharded_virtual(engines)
        for status, cost, ops in results:
            assert status == R.OK and cost == o.cost
            assert [tuple(map(int, r)) for r in ops] == o.reconstruct()
        for e in engines:  # each rank's table (finish makes it the thread's last solve)
            e.finish()
            C, _ = R.export_tables(ch.L + 1, p.slots, D=False)
            assert np.array_equal(C.view(np.uint64), Co.view(np.uint64))
        del engines
        torch.cuda.empty_cache()


def _worker_stall(rank, world, port, q):
    """Rank 1 never joins the exchange: rank 0 must fail with CollectiveError
    naming the tile diagonal within ROTOR_COLLECTIVE_TIMEOUT_S, not hang."""
    import datetime

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["ROTOR_COLLECTIVE_TIMEOUT_S"] = "3"
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=20))
    try:
        if rank == 1:
            q.put((rank, "idle"))
            return
        import oracle as O
        from paper_1911_13214_b200.dist import CollectiveError, solve_sharded

        ch, M, S = _reference()
        ref, _ = O.OracleSolve(ch, M, S).tables()
        try:
            solve_sharded(FakeEngine(ref, ch.L + 1, S))
            q.put((rank, "no error"))
        except CollectiveError as e:
            q.put((rank, "CollectiveError: " + str(e)))
    except Exception as e:
        q.put((rank, repr(e)))


def test_sharded_exchange_timeout_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_stall, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=30)
        if p.is_alive():
            p.kill()
    assert out[1] == "idle"
    assert out[0].startswith("CollectiveError") and "tile diagonal" in out[0], out[0]
