"""The §5.2 comparison strategies.

CPU: the baseline generators and the product's Table-1 replay are pinned by
closed forms (store-all time and peak, sequential time = one extra forward of
every non-last segment) and by agreement with the oracle's independent
simulator; the DP optimum (oracle) never exceeds a sequential schedule that
fits the discretised budget (the sequential schedules are nested persistent
schedules, Theorem 1's space).
GPU: the sweep harness end to end (revolve / optimal solved by the library).
"""
import math

import numpy as np
import pytest

import chaingen as G
import paper_1911_13214_b200.strategies as ST


def int_chain(rng, L, size_max=6, time_max=9):
    """Integer sizes (bytes) and integer times: exact sums, slot = byte when S = M."""
    n = L + 1
    wx = [rng.randint(1, size_max) for _ in range(n)]
    wbx = [wx[i + 1] + rng.randint(0, size_max) if i + 1 <= L else rng.randint(1, size_max) for i in range(n)]
    return G.Chain(L=L, uf=[float(rng.randint(1, time_max)) for _ in range(n)],
                   ub=[float(rng.randint(1, time_max)) for _ in range(n)], wx=wx, wbx=wbx,
                   wy=wx + [rng.randint(1, size_max)], of=[rng.randint(0, 2) for _ in range(n)],
                   ob=[rng.randint(0, 2) for _ in range(n)])


def store_all_peak(ch):
    """Closed form of the store-all peak: forward l holds a^0, delta^n, abar^1..l, o_f^l;
    B^l holds a^0, abar^1..l, delta^l, o_b^l (its output delta^{l-1} uncharged)."""
    n = ch.L + 1
    wbx = [0] + [int(x) for x in ch.wbx]
    pre = np.cumsum(wbx)
    fwd = max(int(ch.wx[0]) + int(ch.wy[n]) + int(pre[l]) + int(ch.of[l - 1]) for l in range(1, n + 1))
    bwd = max(int(ch.wx[0]) + int(pre[l]) + int(ch.wy[l]) + int(ch.ob[l - 1]) for l in range(1, n + 1))
    return max(fwd, bwd)


def test_pytorch_schedule_closed_form():
    rng = G.SplitMix64(41)
    for _ in range(20):
        ch = int_chain(rng, 1 + rng.randint(0, 30))
        r = ST.replay(ST.pytorch_schedule(ch.L), ch)
        assert r.valid, r.error
        assert r.time == float(np.sum(ch.uf) + np.sum(ch.ub))
        assert r.peak == store_all_peak(ch)


def test_sequential_schedule_closed_form():
    rng = G.SplitMix64(42)
    for _ in range(20):
        L = 2 + rng.randint(0, 40)
        ch = int_chain(rng, L)
        n = L + 1
        for k in [1, 2, 3] + ST.sequential_segment_counts(L):
            ops = ST.sequential_schedule(L, k)
            r = ST.replay(ops, ch)
            assert r.valid, (k, r.error)
            b = ST.segment_bounds(n, k)
            twice = sum(float(ch.uf[l - 1]) for l in range(1, b[-2] + 1))  # non-last segments run twice
            assert r.time == float(np.sum(ch.uf) + np.sum(ch.ub)) + twice
            # one backward per stage, every forward of a non-last segment exactly twice
            assert sorted(l for o, l in ops if o == ST.BWD) == list(range(1, n + 1))
            fwd = [l for o, l in ops if o != ST.BWD]
            assert all(fwd.count(l) == (2 if l <= b[-2] else 1) for l in range(1, n + 1))
        assert ST.sequential_schedule(L, 1) == ST.pytorch_schedule(L)


def test_segment_counts_follow_the_paper():
    # "10 different number of segments, from 2 (always included) to 2 sqrt(L)"
    for L in (14, 56, 100, 300, 1000):
        ks = ST.sequential_segment_counts(L)
        assert ks[0] == 2 and ks[-1] == int(round(2 * math.sqrt(L))) and len(ks) <= 10
        assert ks == sorted(set(ks))


def test_replay_agrees_with_the_oracle_simulator(oracle_mod):
    """S = M makes one slot one byte: the oracle's slot sizes equal the bytes, so its
    simulator (independent code) must give the same validity, peak and time."""
    O = oracle_mod
    rng = G.SplitMix64(43)
    for it in range(25):
        L = 1 + rng.randint(0, 12)
        ch = int_chain(rng, L, size_max=4)
        M = int(np.sum(ch.wbx)) + int(np.sum(ch.wx)) + 20
        o = O.OracleSolve(ch, M, M)
        sz = o.sizes()
        schedules = [ST.pytorch_schedule(L)] + [ST.sequential_schedule(L, k) for k in (2, 3)]
        rec = o.reconstruct()
        if rec:
            schedules.append(rec)
        for ops in schedules:
            a = ST.replay(ops, ch)
            b = O.simulate(ops, sz, 10**12)
            assert a.valid == b.valid and a.peak == b.peak and a.time == b.makespan, (it, a, b)
        # an invalid sequence is rejected by both
        bad = [(ST.FNULL, 1), (ST.FNULL, 1)]
        assert not ST.replay(bad, ch).valid and not O.simulate(bad, sz, 10**12).valid


def test_optimal_never_above_a_fitting_sequential(oracle_mod):
    """The DP optimum over nested persistent schedules (Theorem 1) is <= every sequential
    schedule whose discretised peak fits the same budget (they are in that space)."""
    O = oracle_mod
    rng = G.SplitMix64(44)
    for it in range(12):
        L = 3 + rng.randint(0, 14)
        ch = int_chain(rng, L, size_max=5)
        for k in (2, 3, 4):
            ops = ST.sequential_schedule(L, k)
            peak = ST.replay(ops, ch).peak
            o = O.OracleSolve(ch, peak, peak)  # S = M = the schedule's peak: slot = byte
            assert o.cost <= ST.replay(ops, ch).time, (it, k)


@pytest.mark.gpu
def test_compare_sweep_on_gpu(oracle_mod):
    """The sweep end to end: every schedule replays valid; optimal <= revolve at each
    limit; optimal time non-increasing in the limit; each optimal schedule's replayed
    byte peak fits its limit; optimal at a limit <= any sequential schedule whose
    discretised peak fits it."""
    p = G.config2()
    ch = p.chain
    S = 500
    pts = ST.compare(ch, slots=S)
    opt = [q for q in pts if q.strategy == "optimal"]
    rev = [q for q in pts if q.strategy == "revolve"]
    seq = [q for q in pts if q.strategy == "sequential"]
    assert len(opt) == len(rev) == 10 and seq
    for a, b in zip(opt, rev):
        assert a.param == b.param
        if b.feasible:
            assert a.feasible and a.time <= b.time * (1 + 1e-12)
        if a.feasible:
            assert a.peak <= a.param
    times = [q.time for q in opt]
    assert all(x >= y * (1 - 1e-12) for x, y in zip(times, times[1:]))
    for q in opt:
        if not q.feasible:
            continue
        M = int(q.param)
        slot = lambda x: (int(x) * S + M - 1) // M
        for k in ST.sequential_segment_counts(ch.L):
            disc = G.Chain(L=ch.L, uf=ch.uf, ub=ch.ub, wx=[slot(x) for x in ch.wx], wbx=[slot(x) for x in ch.wbx],
                           wy=[slot(x) for x in ch.wy], of=[slot(x) for x in ch.of], ob=[slot(x) for x in ch.ob])
            r = ST.replay(ST.sequential_schedule(ch.L, k), disc)
            if r.peak <= S:  # the schedule is valid in the discretised problem
                assert q.time <= r.time * (1 + 1e-9), (M, k)
    assert ST.pareto(pts)
