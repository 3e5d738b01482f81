"""Pins for the ORACLE (CPU, `-m "not gpu"`).

Each test pins part of `oracle/` to something other than itself — the paper's
worked items, closed forms, exhaustive search, invariants — so that a dropped
term, a wrong index/sign or a transposed operand fails at least one of them.
Pin ids (P1..P10, Q-readings) are those of DESIGN.md §4 / SURVEY.md §8(c).
"""
import math
import os

import numpy as np
import pytest

import chaingen as G

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _solve(O, ch, M, S, **kw):
    return O.OracleSolve(ch, M, S, **kw)


# ---------------------------------------------------------------------------
# P10 discretisation (§5.2)
# ---------------------------------------------------------------------------
def test_discretisation_examples(oracle_mod):
    O = oracle_mod
    assert O.slots_of(0, 1000, 500) == 0  # zero size -> 0 slots
    assert O.slots_of(3, 1000, 500) == 2  # slot = 2 B: ceil(3/2)
    assert O.slots_of(2, 1000, 500) == 1  # exact division
    assert O.slots_of(1000, 1000, 500) == 500


def test_discretisation_bounds(oracle_mod):
    """ceil semantics: slots*(M/S) >= x > (slots-1)*(M/S) (at most one slot over)."""
    O = oracle_mod
    rng = G.SplitMix64(5)
    for _ in range(2000):
        M = rng.randint(1, 1 << 45)
        S = rng.randint(1, 5000)
        x = rng.randint(0, 3 * M)
        k = O.slots_of(x, M, S)
        assert k * M >= x * S  # exact integer arithmetic in Python
        if x > 0:
            assert (k - 1) * M < x * S
        else:
            assert k == 0


# ---------------------------------------------------------------------------
# P9 limits (§4.2) — SPEC examples + simulator-derived peaks
# ---------------------------------------------------------------------------
def test_limits_spec_examples(oracle_mod):
    O = oracle_mod
    o = _solve(O, G.unit_chain(1), 10, 10, fill=False)
    assert o.mall(1, 1) == 2  # emem[1,1] = max(1+1+0, 1+1+0) = 2
    ch = G.Chain(L=3, uf=[1] * 4, ub=[1] * 4, wx=[1, 1, 2, 1], wbx=[2] * 4, wy=[1, 1, 2, 1, 1],
                 of=[0] * 4, ob=[0] * 4)
    o = _solve(O, ch, 10, 10, fill=False)
    assert o.mnull(1, 3) == 4  # max(1+1+0, 1+max(1+2)) = 4


def test_limits_equal_simulated_peaks(oracle_mod):
    """m_all(s,s) = peak of (F_all^s, B^s); m_null(s,t) = peak of (F_ck^s, F_null^{s+1..t-1}),
    each from {a^{s-1}, delta^t} minus the uncounted a^{s-1}."""
    O = oracle_mod
    rng = G.SplitMix64(11)
    for _ in range(60):
        ch = G.tiny_chain(rng, rng.randint(1, 6), abar_ge_a=False, delta_eq_a=False)
        o = _solve(O, ch, 20, 20, fill=False)
        sz = o.sizes()
        for s in range(1, o.n + 1):
            r = O.simulate([(O.FALL, s), (O.BWD, s)], sz, 10**9, s, s)
            assert r.valid, r.failure
            assert r.peak - sz.wx[s - 1] == o.mall(s, s)
            for t in range(s + 1, o.n + 1):
                seq = [(O.FCK, s)] + [(O.FNULL, j) for j in range(s + 1, t)]
                r = O.simulate(seq, sz, 10**9, s, t)
                assert r.peak - sz.wx[s - 1] == o.mnull(s, t), (s, t)


# ---------------------------------------------------------------------------
# P1 exhaustive search (§4.1 persistency P:560-562; Theorem 1)
# ---------------------------------------------------------------------------
def test_dp_equals_bruteforce_top_cells(oracle_mod):
    """C[1,n,m] = optimal persistent makespan, every m, on 200 random chains
    (L <= 5, sizes 0..3, times 1..9, overheads 0..2, omega_delta = omega_a,
    omega_abar >= omega_a — the paper's modelling assumptions P:254-255)."""
    O = oracle_mod
    rng = G.SplitMix64(2024)
    checked = 0
    for _ in range(200):
        L = rng.randint(1, 5)
        ch = G.tiny_chain(rng, L)
        S = 14
        o = _solve(O, ch, S, S)
        sz = o.sizes()
        for m in range(0, S + 1 - sz.wx[0]):
            c, ops = O.brute_force(sz, m + sz.wx[0])
            assert o.cell(1, o.n, m) == c, (L, m)
            checked += 1
    assert checked > 1500


def test_dp_equals_bruteforce_interior_cells(oracle_mod):
    """Every (s,t,m) cell = the exhaustive optimum of the sub-chain s..t started from
    {a^{s-1}, delta^t} with budget m + omega_a^{s-1} (Theorem 1 definition)."""
    O = oracle_mod
    rng = G.SplitMix64(99)
    checked = 0
    for _ in range(40):
        L = rng.randint(2, 5)
        ch = G.tiny_chain(rng, L)
        S = 12
        o = _solve(O, ch, S, S)
        sz = o.sizes()
        for s in range(1, o.n + 1):
            for t in range(s, o.n + 1):
                for m in range(0, S + 1, 2):
                    c, _ = O.brute_force(sz, m + sz.wx[s - 1], s, t)
                    assert o.cell(s, t, m) == c, (s, t, m)
                    checked += 1
    assert checked > 1000


def test_bruteforce_bounds_general_chains(oracle_mod):
    """Outside the modelling assumptions (independent omega_delta, omega_abar < omega_a)
    the recurrence stays an upper bound of the persistent optimum (Q9/Q10), and the
    non-persistent optimum is never worse than the persistent one."""
    O = oracle_mod
    rng = G.SplitMix64(31337)
    for _ in range(120):
        L = rng.randint(1, 4)
        ch = G.tiny_chain(rng, L, abar_ge_a=False, delta_eq_a=False)
        S = 12
        o = _solve(O, ch, S, S)
        sz = o.sizes()
        for m in range(0, S + 1 - sz.wx[0], 3):
            cp, _ = O.brute_force(sz, m + sz.wx[0])
            cn, _ = O.brute_force(sz, m + sz.wx[0], persistent=False)
            assert cp <= o.cell(1, o.n, m)
            assert cn <= cp


def test_q10_nested_witness(oracle_mod):
    """a chain where a non-nested persistent schedule beats the recurrence
    (Theorem 1's proof assumes [s',t] completes before [s,s'-1] starts)."""
    O = oracle_mod
    ch = G.Chain(L=3, uf=[3, 1, 6, 9], ub=[2, 6, 4, 3], wx=[2, 2, 0, 0], wbx=[4, 3, 1, 2],
                 wy=[1, 0, 3, 1, 1], of=[2, 2, 0, 2], ob=[0, 1, 0, 0])
    S = 11
    o = _solve(O, ch, S, S)
    sz = o.sizes()
    m = S - sz.wx[0]
    cp, ops = O.brute_force(sz, S)
    assert o.cell(1, o.n, m) == 44.0
    assert cp == 38.0
    r = O.simulate(ops, sz, S)
    assert r.valid and r.makespan == 38.0


# ---------------------------------------------------------------------------
# P2 restricted ("revolve") mode vs the Griewank-Walther closed form
# ---------------------------------------------------------------------------
def test_griewank_closed_form_small(oracle_mod):
    O = oracle_mod
    # one checkpoint: l(l-1)/2 advances; enough checkpoints: l-1 advances
    for l in range(1, 30):
        assert O.griewank_t(l, 1) == l * (l - 1) // 2
        assert O.griewank_t(l, l) == max(0, l - 1)


def test_restricted_matches_griewank(oracle_mod):
    """Homogeneous chain u_f=1, u_b=0, all sizes 1, no overheads, F_all only right
    before B (the paper's "revolve" baseline): C[1,l,c+2] = l + t(l,c)
    (l taping forwards + t(l,c) advancing forwards with c checkpoints; a^0 is the
    first checkpoint, one slot holds delta, one the live abar)."""
    O = oracle_mod
    ch = G.unit_chain(40, uf=1.0, ub=0.0)
    S = 14
    r = _solve(O, ch, S, S, restricted=True)
    for l in range(1, 42):
        for c in range(1, 12):
            assert r.cell(1, l, c + 2) == l + O.griewank_t(l, c), (l, c)
    # with u_b = 1 every stage adds one backward unit
    ch = G.unit_chain(20, uf=1.0, ub=1.0)
    r = _solve(O, ch, S, S, restricted=True)
    for l in range(1, 22):
        for c in range(1, 12):
            assert r.cell(1, l, c + 2) == 2 * l + O.griewank_t(l, c)


def test_restricted_never_better(oracle_mod):
    O = oracle_mod
    rng = G.SplitMix64(8)
    for _ in range(20):
        ch = G.tiny_chain(rng, rng.randint(1, 8))
        S = 20
        C, _ = _solve(O, ch, S, S).tables()
        R, _ = _solve(O, ch, S, S, restricted=True).tables()
        assert np.all(R >= C)


# ---------------------------------------------------------------------------
# P3 store-all, P4 monotone, P5 lower bound, P6 infeasibility
# ---------------------------------------------------------------------------
def test_store_all(oracle_mod):
    """At a budget >= the store-all peak, the optimum is the store-all makespan
    sum_l (u_f + u_b) and, with every u_f > 0, the schedule is store-all."""
    O = oracle_mod
    rng = G.SplitMix64(77)
    for _ in range(60):
        L = rng.randint(1, 10)
        ch = G.tiny_chain(rng, L)
        n = L + 1
        sa = O.store_all_schedule(n)
        S = 400
        o = _solve(O, ch, S, S)
        sz = o.sizes()
        rep = O.simulate(sa, sz, 10**9)
        assert rep.valid
        expect = 0.0
        for l in range(n, 0, -1):  # w_1 + (w_2 + (... + w_n)) as the C_all chain nests
            expect = (ch.uf[l - 1] + ch.ub[l - 1]) + expect
        assert rep.makespan == sum(ch.uf) + sum(ch.ub)
        m = rep.peak - sz.wx[0]
        assert o.cell(1, n, m) == expect
        assert o.cell(1, n, S - sz.wx[0]) == expect
        assert o.reconstruct(1, n, m) == sa


def test_monotone_lower_bound_infeasible(oracle_mod):
    """P4: C[s,t,m+1] <= C[s,t,m]; P5: C >= sum_{k=s}^{t}(u_f+u_b) when finite;
    P6: C = inf when m < max_{l in [s,t]} (omega_delta^l + omega_abar^l + o_b^l)
    (every B^l must fit); no NaN (Q13)."""
    O = oracle_mod
    rng = G.SplitMix64(4242)
    for it in range(30):
        L = rng.randint(1, 12)
        ch = G.tiny_chain(rng, L, abar_ge_a=bool(it % 2), delta_eq_a=bool(it % 3), int_times=False,
                          allow_zero_time=True)
        S = 24
        o = _solve(O, ch, S, S)
        C, _ = o.tables()
        sz = o.sizes()
        assert not np.isnan(C).any()
        assert np.all(C[:, 1:] <= C[:, :-1])
        n = o.n
        for s in range(1, n + 1):
            for t in range(s, n + 1):
                row = C[O.cell_index(n, s, t)]
                lb = sum(ch.uf[s - 1 : t]) + sum(ch.ub[s - 1 : t])
                fin = np.isfinite(row)
                assert np.all(row[fin] >= lb * (1 - 1e-12))
                need = max(sz.wy[l] + sz.wbx[l] + sz.ob[l] for l in range(s, t + 1))
                assert np.all(np.isinf(row[:need]))


def test_monotone_config2(oracle_mod):
    O = oracle_mod
    p = G.config2()
    o = _solve(O, p.chain, p.mem_limit, p.slots)
    C, D = o.tables()
    assert np.all(C[:, 1:] <= C[:, :-1])
    assert np.isfinite(o.cost)
    # infeasible exactly where D says so
    assert np.array_equal(np.isinf(C), D == O.NONE)


def test_monotone_in_m_every_cell_both_modes(oracle_mod):
    """P4 for every cell of config-5-shaped tables in both modes (the property
    k_batch's candidate bound rests on, DESIGN 5.3): C[s,t,m+1] <= C[s,t,m]
    exactly, including the +inf prefix of each row."""
    O = oracle_mod
    chains, limits, S = G.config5(n_limits=3)
    for ch, lims in zip(chains[:3], limits[:3]):
        for restricted in (False, True):
            o = O.OracleSolve(ch, lims[-1], S, restricted=restricted)
            C, _ = o.tables()
            assert np.all(C[:, 1:] <= C[:, :-1]), (ch.L, restricted)


def test_unit_chain_first_feasible(oracle_mod):
    O = oracle_mod
    for L in range(1, 12):
        o = _solve(O, G.unit_chain(L), 20, 20)
        row = [o.cell(1, o.n, m) for m in range(0, 6)]
        assert math.isinf(row[2]) and math.isfinite(row[3])  # P6: first feasible m = 3 for l >= 2
    o = _solve(O, G.unit_chain(3), 1, 5)  # slot = 0.2 B: a^0 alone needs 5 slots
    assert o.m_top == 0 and math.isinf(o.cost)
    o = _solve(O, G.unit_chain(3), 1, 1)  # M = 1 B: only a^0 fits, m_top = 0
    assert math.isinf(o.cost)


# ---------------------------------------------------------------------------
# P7 reconstruction (Algorithm 2, Q4) replays in the simulator
# ---------------------------------------------------------------------------
def _check_schedule(O, o, ops, sz, s, t, m, exact):
    assert ops is not None
    r = O.simulate(ops, sz, m + sz.wx[s - 1], s, t)
    assert r.valid, r.failure
    assert r.peak <= m + sz.wx[s - 1]
    c = o.cell(s, t, m)
    if exact:
        assert r.makespan == c
    else:
        assert abs(r.makespan - c) <= len(ops) * math.ulp(c)
    bw = [l for op, l in ops if op == O.BWD]
    assert sorted(bw) == list(range(s, t + 1))
    fa = {l for op, l in ops if op == O.FALL}
    assert fa == set(range(s, t + 1))


def test_reconstruct_replays(oracle_mod):
    O = oracle_mod
    rng = G.SplitMix64(555)
    n_checked = 0
    for it in range(80):
        L = rng.randint(1, 9)
        exact = it % 2 == 0
        ch = G.tiny_chain(rng, L, int_times=exact, allow_zero_time=(it % 4 == 0))
        S = 20
        o = _solve(O, ch, S, S)
        sz = o.sizes()
        for s in range(1, o.n + 1):
            for t in range(s, o.n + 1):
                for m in range(0, S + 1):
                    if math.isinf(o.cell(s, t, m)):
                        assert o.reconstruct(s, t, m) is None
                        continue
                    _check_schedule(O, o, o.reconstruct(s, t, m), sz, s, t, m, exact)
                    n_checked += 1
    assert n_checked > 3000


def test_reconstruct_config2(oracle_mod):
    O = oracle_mod
    p = G.config2()
    o = _solve(O, p.chain, p.mem_limit, p.slots)
    ops = o.reconstruct()
    _check_schedule(O, o, ops, o.sizes(), 1, o.n, o.m_top, exact=False)


def test_decision_fill_equals_algorithm2(oracle_mod):
    """The argmin recorded during Algorithm 1's scan (Q11 tie rule) equals the decision
    Algorithm 2 takes by testing C = C_ck(s,s',t,m) for s' ascending."""
    O = oracle_mod
    rng = G.SplitMix64(1)
    for it in range(25):
        ch = G.tiny_chain(rng, rng.randint(1, 12), allow_zero_time=True, time_max=3)
        S = 30
        o = _solve(O, ch, S, S)
        _, D = o.tables()
        assert np.array_equal(D, o.decision_table())
    p = G.config2()
    o = _solve(O, p.chain, p.mem_limit, p.slots)
    _, D = o.tables()
    assert np.array_equal(D, o.decision_table())


def _read_kv(path):
    kv = {}
    with open(path) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            k, *v = line.split()
            kv[k] = v
    return kv


def test_paper_sequence_section_3_1(oracle_mod):
    """the 13-op L=4 sequence is valid (simulator), and is Algorithm 2's
    output on a chain where it is optimal (fixture chain, optimality by brute force)."""
    O = oracle_mod
    kv = _read_kv(os.path.join(GOLDEN, "paper_seq_L4.txt"))
    seq = list(map(int, kv["seq"]))
    seq = [(seq[2 * i], seq[2 * i + 1]) for i in range(len(seq) // 2)]
    assert len(seq) == 13
    # valid on the unit chain with ample memory, makespan = sum of op times
    o = _solve(O, G.unit_chain(4), 100, 100, fill=False)
    r = O.simulate(seq, o.sizes(), 100)
    assert r.valid and r.makespan == 13.0
    f = lambda k: [int(x) for x in kv[k]]
    ch = G.Chain(L=4, uf=f("uf"), ub=f("ub"), wx=f("wx"), wbx=f("wbx"), wy=f("wy"), of=f("of"), ob=f("ob"))
    S, M = int(kv["S"][0]), int(kv["M"][0])
    o = _solve(O, ch, M, S)
    assert o.reconstruct() == seq
    c, _ = O.brute_force(o.sizes(), S)
    assert o.cost == c
    r = O.simulate(seq, o.sizes(), S)
    assert r.valid and r.makespan == o.cost


# ---------------------------------------------------------------------------
# P8 config-1 golden row, Fig. 3 regression (Q15)
# ---------------------------------------------------------------------------
def test_config1_golden(oracle_mod):
    O = oracle_mod
    path = os.path.join(GOLDEN, "cfg1_unit_L10.txt")
    rows = []
    with open(path) as f:
        for line in f:
            if line.startswith("#") or line.startswith("m "):
                continue
            m, c, r = line.split()
            rows.append((int(m), float(c), float(r)))
    assert len(rows) >= 9
    p = G.config1()
    o = _solve(O, p.chain, p.mem_limit, p.slots)
    ro = _solve(O, p.chain, p.mem_limit, p.slots, restricted=True)
    for m, c, r in rows:
        assert o.cell(1, o.n, m) == c, m
        assert ro.cell(1, ro.n, m) == r, m
    assert o.cost == 22.0  # store-all: 11 * (1 + 1)


def fig3_chain(nn):
    """Fig. 3 with the figure's edge sizes, abar = a, delta = 0, o = 0 (Q15)."""
    L = nn + 2
    k = nn - 1
    uf = [0.0] * (L + 1)
    uf[0], uf[1] = float(k), 2.0
    wx = [0, 1, 2] + [3] * (L - 3) + [4]
    wbx = wx[1:] + [0]
    return G.Chain(L=L, uf=uf, ub=[0.0] * (L + 1), wx=wx, wbx=wbx, wy=[0] * (L + 2), of=[0] * (L + 1),
                   ob=[0] * (L + 1), name=f"fig3_{nn}")


def test_fig3_regression(oracle_mod):
    """P:662 "computing F^L requires a memory of 7" holds in this model; DP = exhaustive
    persistent optimum; non-persistent optimum <= persistent.  (The paper's 3n+1 / 2n+2
    are not reproducible in the Table-1 model, Q15.)"""
    O = oracle_mod
    for nn in range(2, 6):
        ch = fig3_chain(nn)
        o = _solve(O, ch, 8, 8)
        sz = o.sizes()
        L = ch.L
        assert sz.wx[L - 1] + sz.wx[L] == 7
        cp, ops = O.brute_force(sz, 8)
        assert o.cost == cp == 3 * nn - 1
        cn, _ = O.brute_force(sz, 8, persistent=False)
        assert cn <= cp
        r = O.simulate(o.reconstruct(), sz, 8)
        assert r.valid and r.makespan == o.cost


# ---------------------------------------------------------------------------
# simulator examples (Table 1 rows; SPEC simulator examples)
# ---------------------------------------------------------------------------
def test_simulator_examples(oracle_mod):
    O = oracle_mod
    o = _solve(O, G.unit_chain(2), 100, 100, fill=False)
    sz = o.sizes()
    assert not O.simulate([], sz, 100).valid  # delta^0 never produced
    r = O.simulate([(O.BWD, 1)], sz, 100)
    assert not r.valid and "delta" in r.failure
    r = O.simulate([(O.FNULL, 1), (O.FNULL, 2), (O.FALL, 3), (O.BWD, 3)], sz, 100)
    assert not r.valid  # B^3 needs a^2 (consumed? no: present) -> then B^2 missing abar^2
    r = O.simulate(O.store_all_schedule(3), sz, 100)
    assert r.valid and r.makespan == 6.0
    # peak of store-all on unit L=2: a^0 + abar^1..3 + delta^3 during F_all^3 = 5
    assert r.peak == 5
    r = O.simulate(O.store_all_schedule(3), sz, 4)
    assert not r.valid and "budget" in r.failure
    # F_null cannot consume abar (Q17)
    r = O.simulate([(O.FALL, 1), (O.FNULL, 2)], sz, 100)
    assert not r.valid


def test_generators_shapes():
    assert G.config1().chain.L == 10
    assert G.config2().chain.L == 100
    assert G.config3().chain.L == 300
    p4 = G.config4()
    assert p4.chain.L == 1000 and p4.slots == 4000
    chains, limits, S = G.config5()
    assert [c.L for c in chains] == [14, 22, 22, 39, 56, 29, 37, 43]
    assert len(limits[0]) == 256 and S == 500
    # determinism
    a, b = G.config4().chain, G.config4().chain
    assert np.array_equal(a.wx, b.wx) and np.array_equal(a.uf, b.uf)
    for p in (G.config2(), G.config3(), p4):
        ch = p.chain
        assert np.all(ch.wbx[:-1] >= ch.wx[1:])  # abar includes a
        assert np.array_equal(ch.wy[:-1], ch.wx)  # omega_delta = omega_a


def test_window_mode_equals_full_table(oracle_mod):
    """Windowed fill (used for sampled parity at full size) reproduces the full table bit for bit."""
    O = oracle_mod
    p = G.config2()
    full = _solve(O, p.chain, p.mem_limit, p.slots)
    C, _ = full.tables()
    n = full.n
    for (s0, t0) in [(1, 30), (40, 101), (70, 75), (101, 101)]:
        w = _solve(O, p.chain, p.mem_limit, p.slots, window=(s0, t0))
        Cw, Dw = w.tables()
        nw = t0 - s0 + 1
        for s in range(s0, t0 + 1):
            for t in range(s, t0 + 1):
                a = C[O.cell_index(n, s, t)]
                b = Cw[O.cell_index(nw, s - s0 + 1, t - s0 + 1)]
                assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


# ---------------------------------------------------------------------------
# §8(d)(ii): the all-core oracle is the same computation (bit-identical)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("restricted", [False, True])
def test_threaded_fill_bit_identical(oracle_mod, restricted):
    """OpenMP over the cells of each diagonal (oracle_fill_threads) reproduces the
    single-thread fill bit for bit (C and D), on config 2 and random tiny chains;
    keep_d=False changes nothing in C."""
    O = oracle_mod
    cases = [(G.config2().chain, G.config2().mem_limit, G.config2().slots)]
    rng = G.SplitMix64(77)
    for _ in range(6):
        ch = G.random_chain(rng, rng.randint(3, 40), real_times=True)
        cases.append((ch, G.budget_ref(ch) // 3, 60))
    for ch, M, S in cases:
        a = _solve(O, ch, M, S, restricted=restricted)
        for thr in (2, 5):
            b = _solve(O, ch, M, S, restricted=restricted, threads=thr)
            Ca, Da = a.tables()
            Cb, Db = b.tables()
            assert np.array_equal(Ca.view(np.uint64), Cb.view(np.uint64))
            assert np.array_equal(Da, Db)
        c = _solve(O, ch, M, S, restricted=restricted, threads=3, keep_d=False)
        assert np.array_equal(Ca.view(np.uint64), c.table_view().view(np.uint64))
        assert c.reconstruct() == a.reconstruct()


def test_threaded_fill_window_config3(oracle_mod):
    """A 120-stage window of config 3 (S=2000): threaded == single thread."""
    O = oracle_mod
    p = G.config3()
    a = _solve(O, p.chain, p.mem_limit, p.slots, window=(90, 209), keep_d=False)
    b = _solve(O, p.chain, p.mem_limit, p.slots, window=(90, 209), keep_d=False, threads=O.max_threads())
    assert np.array_equal(a.table_view().view(np.uint64), b.table_view().view(np.uint64))


# ---------------------------------------------------------------------------
# checksum module of the full-size golden (tests/table_hash.py)
# ---------------------------------------------------------------------------
def test_table_hash_definition_and_sensitivity(oracle_mod):
    """The vectorised checksums equal their definition written with Python ints,
    and flipping any single bit of any value changes the checksum of its cell's
    s and d (so the config-4 golden localises a mismatch)."""
    import table_hash as TH

    O = oracle_mod
    p = G.config1()
    o = _solve(O, p.chain, p.mem_limit, p.slots)
    C = o.table_view().copy()
    n = o.n
    hs = TH.hash_canonical_table(C, n, chunk=7)
    K = [int(x) for x in TH.row_keys(C.shape[1])]
    K2 = [int(x) for x in TH.cell_keys(n)]
    M = (1 << 64) - 1
    H = [0] * (n + 1)
    Gd = [0] * n
    for s in range(1, n + 1):
        for t in range(s, n + 1):
            row = C[TH.cell_index(n, s, t)].view(np.uint64)
            h = sum(int(b) * k for b, k in zip(row, K)) & M
            H[s] = (H[s] + h * K2[t]) & M
            Gd[t - s] = (Gd[t - s] + h * K2[s]) & M
    assert [int(x) for x in hs.H] == H and [int(x) for x in hs.G] == Gd
    rng = G.SplitMix64(3)
    for _ in range(50):
        s = rng.randint(1, n)
        t = rng.randint(s, n)
        m = rng.randint(0, C.shape[1] - 1)
        bit = rng.randint(0, 63)
        D = C.copy()
        D.view(np.uint64)[TH.cell_index(n, s, t), m] ^= np.uint64(1 << bit)
        h2 = TH.hash_canonical_table(D, n)
        assert (h2.H != hs.H).sum() == 1 and h2.H[s] != hs.H[s]
        assert (h2.G != hs.G).sum() == 1 and h2.G[t - s] != hs.G[t - s]


def test_cfg4_golden_file_consistent():
    """The committed config-4 golden (scripts/make_golden_cfg4.py, oracle only) is
    well formed: cost = its top row at m_top, checksums for every s and d, and an
    Algorithm-2 schedule with exactly one B per stage (P7)."""
    import table_hash as TH

    path = os.path.join(GOLDEN, "cfg4_L1000_S4000.txt")
    g = TH.read_golden(path)
    L, S, m_top = int(g["L"]), int(g["S"]), int(g["m_top"])
    n = L + 1
    assert len(g["top"]) == S + 1 and len(g["H"]) == n and len(g["G"]) == n
    assert g["top"][m_top] == int(g["cost"], 16)
    assert np.float64(float(g["cost_float"])).view(np.uint64) == np.uint64(int(g["cost"], 16))
    ops = [(x >> 32, x & 0xFFFFFFFF) for x in g["ops"]]
    assert len(ops) == int(g["n_ops"])
    assert sorted(st for op, st in ops if op == 3) == list(range(1, n + 1))
    top = np.array(g["top"], dtype=np.uint64).view(np.float64)
    assert np.all(top[1:] <= top[:-1])  # P4 monotone in m
    p = G.config4()
    assert (L, S, int(g["M"])) == (p.chain.L, p.slots, p.mem_limit)
    # P7: the schedule replays valid within the budget and reproduces the cost (Q14)
    O = pytest.importorskip("oracle")
    sz = O.OracleSolve(p.chain, p.mem_limit, p.slots, fill=False).sizes()
    rep = O.simulate(ops, sz, S)
    cost = float(g["cost_float"])
    assert rep.valid, rep.failure
    assert abs(rep.makespan - cost) <= len(ops) * math.ulp(cost)
    assert cost >= float(np.sum(p.chain.uf) + np.sum(p.chain.ub)) * (1 - 1e-12)  # P5
