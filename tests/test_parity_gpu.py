"""GPU parity: the CUDA path (through the C ABI) against the independent oracle.

Bar (north_star): bit-exact fp64 C tables (compared as uint64
bit patterns, tolerance 0 ulp), identical argmin tables D (uint16), identical
costs and identical Algorithm-2 schedules; replaying the GPU schedule in the
oracle's simulator is valid within the limit and reproduces the cost.
"""
import math

import numpy as np
import pytest

import chaingen as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge

    ge.build_library()
    import paper_1911_13214_b200 as R

    return R


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def assert_tables_equal(Cg, Co, what=""):
    if not np.array_equal(bits(Cg), bits(Co)):
        bad = np.argwhere(bits(Cg) != bits(Co))
        i, m = bad[0]
        raise AssertionError(f"{what}: {len(bad)} cells differ; first cell {i} m={m}: gpu={Cg[i, m]!r} oracle={Co[i, m]!r}")


KERNELS = ["wavefront", "tiled"]


def gpu_full(R, ch, M, S, **opts):
    res = R.solve(ch, M, S, **opts)
    C, D = R.export_tables(ch.L + 1, S)
    return res, C, D


def check_against_oracle(R, O, ch, M, S, restricted=False, kernel="wavefront", keep_argmin=False):
    o = O.OracleSolve(ch, M, S, restricted=restricted)
    Co, Do = o.tables()
    res, Cg, Dg = gpu_full(R, ch, M, S, restricted=restricted, kernel=kernel, keep_argmin=keep_argmin)
    assert_tables_equal(Cg, Co, f"{ch.name} M={M} S={S} {kernel}")
    assert np.array_equal(Dg, Do), f"argmin tables differ ({kernel}, keep_argmin={keep_argmin})"
    oc = o.cost
    if math.isinf(oc):
        assert res.status == R.INFEASIBLE and math.isinf(res.cost)
    else:
        assert res.status == R.OK
        assert bits(np.array([res.cost])) == bits(np.array([oc]))
        ops_o = o.reconstruct()
        assert res.op_list() == ops_o
        sz = o.sizes()
        rep = O.simulate(res.op_list(), sz, S)
        assert rep.valid, rep.failure
        assert abs(rep.makespan - oc) <= len(ops_o) * math.ulp(oc)
    return o, res


@pytest.mark.parametrize("kernel", KERNELS)
def test_tiny_random_chains(R, oracle_mod, kernel):
    """Random small chains: ties (integer/zero times), zero sizes, huge abar/a,
    general (independent delta, abar < a) chains, L = 1, infeasible limits."""
    O = oracle_mod
    rng = G.SplitMix64(17)
    for it in range(60):
        L = 1 + rng.randint(0, 24)
        kind = it % 4
        if kind == 0:
            ch = G.tiny_chain(rng, L, size_max=5, time_max=3, allow_zero_time=True)
        elif kind == 1:
            ch = G.tiny_chain(rng, L, size_max=6, abar_ge_a=False, delta_eq_a=False)
        elif kind == 2:
            ch = G.tiny_chain(rng, L, size_max=4, int_times=False)
        else:
            ch = G.random_chain(rng, L, real_times=bool(it % 8 == 3), big=True)
        S = [7, 16, 33, 64, 130][rng.randint(0, 4)]
        if kind == 3:
            M = max(1, int(sum(int(x) for x in ch.wbx) * (0.05 + 0.5 * rng.uniform())))
        else:
            M = S
        check_against_oracle(R, O, ch, M, S, kernel=kernel, keep_argmin=(it % 5 == 0 and kernel == "wavefront"))


@pytest.mark.parametrize("kernel", KERNELS)
def test_restricted_mode(R, oracle_mod, kernel):
    O = oracle_mod
    rng = G.SplitMix64(23)
    for it in range(10):
        ch = G.tiny_chain(rng, 3 + rng.randint(0, 20), size_max=4)
        check_against_oracle(R, O, ch, 40, 40, restricted=True, kernel=kernel)
    check_against_oracle(R, O, G.unit_chain(40, ub=0.0), 14, 14, restricted=True, kernel=kernel)


@pytest.mark.parametrize("kernel", KERNELS)
def test_config1_and_2_full_tables(R, oracle_mod, kernel):
    O = oracle_mod
    for p in (G.config1(), G.config2()):
        check_against_oracle(R, O, p.chain, p.mem_limit, p.slots, kernel=kernel)


@pytest.mark.parametrize("kernel", KERNELS)
def test_edge_cases(R, oracle_mod, kernel):
    O = oracle_mod
    # L = 1, ample memory -> [F_all1, F_all2, B2, B1]
    o, res = check_against_oracle(R, O, G.unit_chain(1), 100, 100, kernel=kernel)
    assert res.op_list() == [(0, 1), (0, 2), (3, 2), (3, 1)]
    # infeasible: a^0 alone exceeds M (m_top < 0)
    ch = G.unit_chain(3, size=10)
    res = R.solve(ch, 5, 5, kernel=kernel)
    assert res.status == R.INFEASIBLE and math.isinf(res.cost)
    # infeasible: m_top >= 0 but too small
    res = R.solve(G.unit_chain(5), 3, 3, kernel=kernel)
    assert res.status == R.INFEASIBLE
    # all sizes zero, S = 1: store-all at zero memory
    z = G.Chain(L=4, uf=[1, 2, 3, 4, 5], ub=[1] * 5, wx=[0] * 5, wbx=[0] * 5, wy=[0] * 6, of=[0] * 5, ob=[0] * 5)
    check_against_oracle(R, O, z, 1, 1, kernel=kernel)
    # one huge item (clamped slot count > S) must behave like the oracle's uncapped count
    ch = G.unit_chain(6)
    ch.wbx[3] = 10**15
    check_against_oracle(R, O, ch, 20, 20, kernel=kernel)
    # ops truncation reports ETRUNC with the full count
    p = G.config1()
    full = R.solve(p.chain, p.mem_limit, 12, kernel=kernel)
    tr = R.solve(p.chain, p.mem_limit, 12, ops_cap=5, kernel=kernel)
    assert tr.status == R.ETRUNC and tr.n_ops == full.n_ops and tr.op_list() == full.op_list()[:5]


@pytest.mark.parametrize("L", [30, 31, 32, 33, 63, 64, 71, 95, 96, 127, 160])
def test_tiled_block_boundaries(R, oracle_mod, L):
    """Chains whose length straddles the 32-stage tiles / 8-stage sub-tiles of the tiled
    fill (partial last block, exact multiples, one stage over), with wide shifts (large
    abar/a relative to the slot size) and a ragged S: full tables bit-exact, both modes."""
    O = oracle_mod
    rng = G.SplitMix64(1000 + L)
    ch = G.random_chain(rng, L, real_times=True, big=True)
    S = 37 + (L % 23)
    M = max(1, int(sum(int(x) for x in ch.wbx) * 0.22))
    check_against_oracle(R, O, ch, M, S, kernel="tiled")
    check_against_oracle(R, O, ch, M, S, kernel="tiled", restricted=True)
    # integer times: ties everywhere (the fill keeps no argmin; Algorithm 2 re-derives it)
    ch2 = G.tiny_chain(rng, L, size_max=3, time_max=2, allow_zero_time=True)
    check_against_oracle(R, O, ch2, 24, 24, kernel="tiled")


@pytest.mark.parametrize("S", [15, 16, 17, 31, 32, 33, 63, 64, 127, 128, 129, 255, 257, 520])
def test_tiled_m_chunk_boundaries(R, oracle_mod, S):
    """S + 1 around the m-chunks of the tiled kernels (32 m per wide middle item,
    16 m per exact middle item and sub-product warp, 128 m per leaf CTA,
    32 / 128 look-back chunks), with
    shifts from a fraction of a chunk to several chunks (big sizes, tight and
    loose limits): full tables bit-exact, both modes."""
    O = oracle_mod
    rng = G.SplitMix64(5000 + S)
    ch = G.random_chain(rng, 70, real_times=True, big=True)
    for f in (0.12, 0.35):
        M = max(1, int(sum(int(x) for x in ch.wbx) * f))
        check_against_oracle(R, O, ch, M, S, kernel="tiled")
    check_against_oracle(R, O, ch, M, S, kernel="tiled", restricted=True)


_VARIANT_SCRIPT = r"""
import sys
import numpy as np
import __graft_entry__ as ge
ge.build_library()
import chaingen as G, oracle as O, paper_1911_13214_b200 as R
cases = [(G.config2().chain, G.config2().mem_limit, G.config2().slots)]
for L, S in ((95, 33), (64, 129)):
    ch = G.random_chain(G.SplitMix64(7000 + L), L, real_times=True, big=True)
    cases.append((ch, max(1, int(sum(int(x) for x in ch.wbx) * 0.22)), S))
for ch, M, S in cases:
    res = R.solve(ch, M, S, kernel="tiled")
    C, _ = R.export_tables(ch.L + 1, S, D=False)
    o = O.OracleSolve(ch, M, S)
    Co, _ = o.tables()
    assert np.array_equal(C.view(np.uint64), Co.view(np.uint64)), (ch.name, ch.L, S)
    assert res.op_list() == (o.reconstruct() or [])
print("ok")
"""


VARIANTS = {
    "exact": {"ROTOR_MIDDLE": "exact"},  # the unpruned fp64 k_tile_middle
    "nocoarse": {"ROTOR_COARSE": "0"},  # the pruned middle without its coarse bounds
    "ring28": {"ROTOR_WRING": "28"},  # the pruned middle with 8 ring stages of 2 splits
    "ring44": {"ROTOR_WRING": "44"},  # 4 ring stages of 4 splits (the default before the 8 x 2 ring)
    "leaf_tab": {"ROTOR_LEAF": "tab"},  # k_sub_leaf_row<false>: right-range operands not staged
    "prod4": {"ROTOR_PROD": "1"},  # k_sub_product_async at 4 CTAs/SM
}


@pytest.mark.parametrize("variant", sorted(VARIANTS))
def test_kernel_variants(R, variant):
    """The non-default kernels of the tiled fill (selected once per process by
    ROTOR_MIDDLE / ROTOR_COARSE / ROTOR_LEAF / ROTOR_PROD, kept for A/B
    measurements) stay bit-exact against the oracle — run in a subprocess with
    the variable set."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PYTHONPATH=root, **VARIANTS[variant])
    r = subprocess.run([sys.executable, "-c", _VARIANT_SCRIPT], cwd=root, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_device_resident_path(R, oracle_mod):
    import torch

    O = oracle_mod
    p = G.config2()
    ch = p.chain
    dev = torch.device("cuda:0")
    d = {k: torch.from_numpy(np.asarray(getattr(ch, k)).astype(np.float64 if k in ("uf", "ub") else np.int64)).to(dev)
         for k in ("uf", "ub", "wx", "wbx", "wy", "of", "ob")}
    ws = torch.empty(R.workspace_bytes(ch.L, p.slots), dtype=torch.uint8, device=dev)
    cap = R.max_ops(ch.L)
    out = dict(cost=torch.empty(1, dtype=torch.float64, device=dev), ops=torch.empty((cap, 2), dtype=torch.int32, device=dev),
               n_ops=torch.empty(1, dtype=torch.int64, device=dev), status=torch.empty(1, dtype=torch.int32, device=dev))
    st = torch.cuda.current_stream()
    R.solve_device(d, ch.L, p.mem_limit, p.slots, ws, out, stream=st)
    torch.cuda.synchronize()
    o = O.OracleSolve(ch, p.mem_limit, p.slots)
    assert int(out["status"].item()) == R.OK
    assert out["cost"].item() == o.cost
    k = int(out["n_ops"].item())
    ops = [tuple(map(int, r)) for r in out["ops"][:k].cpu().numpy()]
    assert ops == o.reconstruct()
    C, _ = R.export_tables(ch.L + 1, p.slots, D=False)
    assert_tables_equal(C, o.tables()[0], "device path")


def test_batched_equals_single(R, oracle_mod):
    O = oracle_mod
    chains, limits, S = G.config5(n_limits=6)
    chains, limits = chains[:4], limits[:4]
    costs, status, n_ops, ops = R.solve_batch(chains, limits, S, with_ops=True)
    for i, ch in enumerate(chains):
        for j, M in enumerate(limits[i]):
            o = O.OracleSolve(ch, M, S)
            c = o.cost
            if math.isinf(c):
                assert status[i, j] == R.INFEASIBLE and math.isinf(costs[i, j])
            else:
                assert status[i, j] == R.OK
                assert costs[i, j] == c
                got = [tuple(map(int, r)) for r in ops[i * len(limits[i]) + j]]
                assert got == o.reconstruct()


def test_config5_batched_sweep(R, oracle_mod):
    """The full config-5 sweep (8 chains x 256 limits = 2048 tables) in one fused
    launch: a seeded sample of 40 problems matches the oracle bit for bit (cost and
    schedule); every feasible schedule replays valid within its limit with its cost."""
    O = oracle_mod
    chains, limits, S = G.config5()
    costs, status, n_ops, ops = R.solve_batch(chains, limits, S, with_ops=True)
    nl = len(limits[0])
    rng = G.SplitMix64(5)
    sample = {(rng.randint(0, len(chains) - 1), rng.randint(0, nl - 1)) for _ in range(40)}
    for i, j in sorted(sample):
        o = O.OracleSolve(chains[i], limits[i][j], S)
        c = o.cost
        if math.isinf(c):
            assert status[i, j] == R.INFEASIBLE and math.isinf(costs[i, j])
        else:
            assert status[i, j] == R.OK and bits(np.array([costs[i, j]])) == bits(np.array([c]))
            assert [tuple(map(int, r)) for r in ops[i * nl + j]] == o.reconstruct()
    n_feasible = 0
    for i, ch in enumerate(chains):
        for j in range(nl):
            if status[i, j] != R.OK:
                assert status[i, j] == R.INFEASIBLE
                continue
            n_feasible += 1
            sz = O.OracleSolve(ch, limits[i][j], S, fill=False).sizes()
            seq = [tuple(map(int, r)) for r in ops[i * nl + j]]
            rep = O.simulate(seq, sz, S)
            assert rep.valid, (i, j, rep.failure)
            assert abs(rep.makespan - costs[i, j]) <= len(seq) * math.ulp(costs[i, j])
    assert n_feasible > 1000


@pytest.mark.parametrize("kernel", KERNELS)
def test_config3_full_table(R, oracle_mod, kernel):
    """DenseNet-shaped chain, L=300, S=2000 (9.2e9 transitions): full-table bit parity."""
    O = oracle_mod
    p = G.config3()
    check_against_oracle(R, O, p.chain, p.mem_limit, p.slots, kernel=kernel)


def _window_cells(s0, t0):
    return [(s, t) for d in range(0, t0 - s0 + 1) for s in range(s0, t0 - d + 1) for t in [s + d]]


@pytest.mark.parametrize("kernel", KERNELS)
def test_config4_full_size_sampled(R, oracle_mod, kernel):
    """L=1000, S=4000 in the bench's launch configuration: every cell of several
    windows of stages (start, middle, end with the loss stage, one long window)
    is bit-identical to the oracle's windowed fill; the top schedule replays
    valid within S slots with the reported cost; rows are monotone in m."""
    O = oracle_mod
    p = G.config4()
    ch = p.chain
    res = R.solve(ch, p.mem_limit, p.slots, kernel=kernel)
    assert res.status == R.OK
    n = ch.L + 1
    for (s0, t0) in [(1, 40), (480, 530), (950, n), (300, 420)]:
        o = O.OracleSolve(ch, p.mem_limit, p.slots, window=(s0, t0))
        Co, _ = o.tables()
        cells = _window_cells(s0, t0)
        Cg = R.export_rows(cells, p.slots)
        nw = t0 - s0 + 1
        Co_rows = np.stack([Co[O.cell_index(nw, s - s0 + 1, t - s0 + 1)] for s, t in cells])
        assert_tables_equal(Cg, Co_rows, f"cfg4 window {s0}..{t0}")
        assert np.all(Cg[:, 1:] <= Cg[:, :-1])
    # top cell: schedule replay in the oracle simulator (the oracle cannot fill L=1000 in a test)
    o = O.OracleSolve(ch, p.mem_limit, p.slots, fill=False)
    sz = o.sizes()
    rep = O.simulate(res.op_list(), sz, p.slots)
    assert rep.valid, rep.failure
    assert abs(rep.makespan - res.cost) <= res.n_ops * math.ulp(res.cost)
    lb = float(np.sum(ch.uf) + np.sum(ch.ub))
    assert res.cost >= lb * (1 - 1e-12)
    top = R.export_rows([(1, n)], p.slots)[0]
    assert top[S_top(sz, p.slots)] == res.cost


def S_top(sz, S):
    return S - sz.wx[0]


@pytest.mark.parametrize("kernel", KERNELS)
def test_config4_full_table_golden(R, kernel):
    """Config 4 (L=1000, S=4000, the bench's workload and launch configuration):
    the WHOLE table against the oracle's full fill, through the checksums of
    tests/golden/cfg4_L1000_S4000.txt (scripts/make_golden_cfg4.py, oracle only):
    every row's fp64 bits enter the per-s and per-d checksums, so any differing
    value fails and is located to its cell (s, s+d).  Also bit-equal: the cost
    (P:824), the whole top row C[1,L+1,0..S] and Algorithm 2's schedule."""
    import os

    import table_hash as TH

    g = TH.read_golden(os.path.join(os.path.dirname(__file__), "golden", "cfg4_L1000_S4000.txt"))
    p = G.config4()
    ch = p.chain
    n = ch.L + 1
    assert (ch.L, p.slots, p.mem_limit) == (int(g["L"]), int(g["S"]), int(g["M"]))
    res = R.solve(ch, p.mem_limit, p.slots, kernel=kernel)
    assert res.status == R.OK
    assert int(bits(np.array([res.cost]))[0]) == int(g["cost"], 16)
    ops = [(x >> 32, x & 0xFFFFFFFF) for x in g["ops"]]
    assert res.op_list() == ops
    top = R.export_rows([(1, n)], p.slots)[0]
    assert [int(x) for x in bits(top)] == g["top"]
    hs = TH.TableHasher(n)
    for s0 in range(1, n + 1, 32):
        cells = [(s, t) for s in range(s0, min(s0 + 32, n + 1)) for t in range(s, n + 1)]
        rows = R.export_rows(cells, p.slots)
        hs.add([c[0] for c in cells], [c[1] for c in cells], TH.row_hashes(rows))
    assert hs.complete()
    H = [int(x) for x in hs.H[1:]]
    Gd = [int(x) for x in hs.G]
    bad_s = [s + 1 for s in range(n) if H[s] != g["H"][s]]
    bad_d = [d for d in range(n) if Gd[d] != g["G"][d]]
    assert not bad_s and not bad_d, f"{kernel}: rows differ from the oracle at s in {bad_s[:10]}, d in {bad_d[:10]}"


def test_counters(R, oracle_mod):
    """options.counters: the pruned middle's work counts are consistent with the
    geometry (visits = middle warps x splits; every fired split also passed the
    coarse bound; the middle never compares more than it visits), the nominal
    count is rotor_transitions, and counting changes no result."""
    O = oracle_mod
    p = G.config3()
    ch = p.chain
    res0 = R.solve(ch, p.mem_limit, p.slots, kernel="tiled")
    res = R.solve(ch, p.mem_limit, p.slots, kernel="tiled", counters=True)
    assert res.cost == res0.cost and res.op_list() == res0.op_list()
    c = R.last_counters()
    assert c["nominal"] == R.transitions(ch.L, p.slots)
    n, TB = ch.L + 1, 32
    nb = (n + TB - 1) // TB
    n_mc = (p.slots + 1 + 31) // 32
    visits = sum((nb - d) * n_mc * 16 * (d - 1) * TB for d in range(2, nb))
    assert c["middle_split_visits"] == visits
    assert c["exact_splits"] <= c["coarse_pass"] <= c["middle_split_visits"]
    assert c["quadrant_compares"] <= 4 * c["coarse_pass"]
    assert 0 < c["middle_nominal"] < c["nominal"]
    assert c["evaluated"] == 512.0 * c["quadrant_compares"] + 2048.0 * c["exact_splits"] + c["dependent_nominal"]
    assert c["evaluated"] < c["nominal"]


@pytest.mark.parametrize("halo_mode", [0, 1])
@pytest.mark.parametrize("ranks", [2, 3])
def test_solve_sharded_device_list(R, oracle_mod, halo_mode, ranks):
    """rotor_solve_sharded (one process, a device list; §8(b)/(e) 2): config 2 and
    config 3 with the table sharded over `ranks` entries of device 0 (each entry
    its own workspace and stream; tiles exchanged by pack + peer copy or by the
    fused peer pull) — full table, cost and schedule bit-identical to the oracle."""
    O = oracle_mod
    for p in (G.config2(), G.config3()):
        ch = p.chain
        o = O.OracleSolve(ch, p.mem_limit, p.slots, threads=O.max_threads(), keep_d=False)
        res = R.solve_sharded(ch, p.mem_limit, p.slots, [0] * ranks, halo_mode=halo_mode)
        assert res.status == R.OK and res.cost == o.cost
        assert res.op_list() == o.reconstruct()
        C, _ = R.export_tables(ch.L + 1, p.slots, D=False)
        assert_tables_equal(C, o.table_view(), f"sharded x{ranks} halo {halo_mode} {ch.name}")
    R.release()


def test_solve_sharded_config4_golden(R):
    """Config 4 sharded over two entries of device 0 (2 x 48.5 GB workspaces),
    fused peer pull: cost bits, schedule and top row equal the oracle golden."""
    import os

    import table_hash as TH

    g = TH.read_golden(os.path.join(os.path.dirname(__file__), "golden", "cfg4_L1000_S4000.txt"))
    p = G.config4()
    n = p.chain.L + 1
    res = R.solve_sharded(p.chain, p.mem_limit, p.slots, [0, 0], halo_mode=1)
    assert res.status == R.OK
    assert int(bits(np.array([res.cost]))[0]) == int(g["cost"], 16)
    assert res.op_list() == [(x >> 32, x & 0xFFFFFFFF) for x in g["ops"]]
    top = R.export_rows([(1, n)], p.slots)[0]
    assert [int(x) for x in bits(top)] == g["top"]
    R.release()


def test_batch_device_list(R, oracle_mod):
    """rotor_solve_batch over a device list (§8(b)/(e) 1: LPT-split problems, one
    worker thread per entry; here three entries of device 0) equals the
    single-device batch bit for bit, and the oracle on a sample; costs-only mode
    reports OK (not ETRUNC) for feasible problems."""
    O = oracle_mod
    chains, limits, S = G.config5(n_limits=16)
    c1, s1, n1, o1 = R.solve_batch(chains, limits, S, with_ops=True)
    c3, s3, n3, o3 = R.solve_batch(chains, limits, S, with_ops=True, devices=[0, 0, 0])
    assert np.array_equal(bits(c1), bits(c3)) and np.array_equal(s1, s3) and np.array_equal(n1, n3)
    assert all(np.array_equal(a, b) for a, b in zip(o1, o3))
    c0, s0, _, _ = R.solve_batch(chains, limits, S, with_ops=False, devices=[0, 0])
    assert np.array_equal(bits(c0), bits(c1))
    assert set(np.unique(s0)) <= {R.OK, R.INFEASIBLE} and np.array_equal(s0 == R.OK, s1 == R.OK)
    for i in range(0, len(chains), 3):
        for j in (0, 7, 15):
            o = O.OracleSolve(chains[i], limits[i][j], S)
            assert (math.isinf(o.cost) and math.isinf(c3[i, j])) or c3[i, j] == o.cost


def test_cached_workspace_threads(R, oracle_mod):
    """Library workspaces are leased per call: two threads solving concurrently on
    one device with the default (cached) workspace both get the oracle's result,
    and exporting tables that a later call reused is refused, not misread."""
    import threading

    O = oracle_mod
    p = G.config2()
    ch = p.chain
    limits = [p.mem_limit, p.mem_limit // 2]
    want = [O.OracleSolve(ch, M, p.slots).cost for M in limits]
    got = [None, None]
    errs = []

    def run(k):
        try:
            for _ in range(6):
                got[k] = R.solve(ch, limits[k], p.slots).cost
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=run, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs and got == want and want[0] != want[1]
    R.solve(ch, p.mem_limit, p.slots)
    R.export_rows([(1, 2)], p.slots)  # still this thread's tables
    other = threading.Thread(target=lambda: R.solve(ch, limits[1], p.slots))
    other.start()
    other.join()
    with pytest.raises(R.RotorError):
        R.export_rows([(1, 2)], p.slots)


@pytest.mark.parametrize("schedule", ["diagonal", "dag"])
def test_tiled_schedules(R, oracle_mod, schedule):
    """Both schedules of the tiled fill (the tile DAG over several streams, the
    default; diagonal by diagonal on one stream) give the oracle's full table,
    cost and schedule — config 3 and chains whose lengths end mid-tile."""
    O = oracle_mod
    cases = [G.config3()]
    rng = G.SplitMix64(911)
    for L in (33, 95, 160):
        ch = G.random_chain(rng, L, real_times=True, big=True)
        cases.append(G.Problem(ch, mem_limit=max(1, int(sum(int(x) for x in ch.wbx) * 0.2)), slots=97, name=f"r{L}"))
    for p in cases:
        ch = p.chain
        o = O.OracleSolve(ch, p.mem_limit, p.slots, threads=O.max_threads(), keep_d=False)
        res = R.solve(ch, p.mem_limit, p.slots, kernel="tiled", schedule=schedule)
        C, _ = R.export_tables(ch.L + 1, p.slots, D=False)
        assert_tables_equal(C, o.table_view(), f"{schedule} {p.name}")
        assert res.cost == o.cost and res.op_list() == (o.reconstruct() or [])


def test_dag_shared_streams_long_chain(R, oracle_mod):
    """A chain long enough for more tile rows than DAG streams (L = 2100: 66 tile
    rows on 64 streams, rows sharing a stream): the DAG schedule's full table
    equals the diagonal schedule's bit for bit, and both equal the oracle on
    windows at both ends of the chain and on the top cost / schedule replay."""
    O = oracle_mod
    rng = G.SplitMix64(2100)
    ch = G.random_chain(rng, 2100, real_times=True, big=True)
    S = 30
    M = max(1, int(sum(int(x) for x in ch.wbx) * 0.05))
    n = ch.L + 1
    r1 = R.solve(ch, M, S, kernel="tiled", schedule="dag")
    C1, _ = R.export_tables(n, S, D=False)
    r2 = R.solve(ch, M, S, kernel="tiled", schedule="diagonal")
    C2, _ = R.export_tables(n, S, D=False)
    assert_tables_equal(C1, C2, "dag vs diagonal, L=2100")
    assert r1.cost == r2.cost and r1.op_list() == r2.op_list()
    for (s0, t0) in [(1, 70), (2040, n)]:
        o = O.OracleSolve(ch, M, S, window=(s0, t0), threads=O.max_threads(), keep_d=False)
        cells = _window_cells(s0, t0)
        nw = t0 - s0 + 1
        Co = o.table_view()
        got = np.stack([C1[O.cell_index(n, s, t)] for s, t in cells])
        want = np.stack([Co[O.cell_index(nw, s - s0 + 1, t - s0 + 1)] for s, t in cells])
        assert_tables_equal(got, want, f"L=2100 window {s0}..{t0}")
    if r1.status == R.OK:
        sz = O.OracleSolve(ch, M, S, fill=False).sizes()
        rep = O.simulate(r1.op_list(), sz, S)
        assert rep.valid and abs(rep.makespan - r1.cost) <= r1.n_ops * math.ulp(r1.cost)


@pytest.mark.parametrize("restricted", [False, True])
def test_config5_all_costs_vs_oracle(R, oracle_mod, restricted):
    """The whole config-5 sweep (8 chains x 256 limits = 2048 tables, S=500) in one
    fused launch: EVERY cost bit-equal to the oracle's (all-core OpenMP fill,
    bit-identical to one thread), in both modes (restricted = the paper's
    revolve baseline, used by strategies.compare); statuses agree
    (infeasible exactly where the oracle's cost is +inf); a sample of schedules
    equals the oracle's Algorithm 2."""
    O = oracle_mod
    chains, limits, S = G.config5()
    costs, status, n_ops, ops = R.solve_batch(chains, limits, S, with_ops=True, restricted=restricted)
    nl = len(limits[0])
    thr = O.max_threads()
    rng = G.SplitMix64(55 + restricted)
    sample = {(rng.randint(0, len(chains) - 1), rng.randint(0, nl - 1)) for _ in range(24)}
    for i, ch in enumerate(chains):
        for j in range(nl):
            o = O.OracleSolve(ch, limits[i][j], S, restricted=restricted, threads=thr, keep_d=False)
            c = o.cost
            if math.isinf(c):
                assert status[i, j] == R.INFEASIBLE and math.isinf(costs[i, j]), (i, j)
            else:
                assert status[i, j] == R.OK, (i, j, status[i, j])
                assert bits(np.array([costs[i, j]])) == bits(np.array([c])), (i, j, costs[i, j], c)
                if (i, j) in sample:
                    assert [tuple(map(int, r)) for r in ops[i * nl + j]] == o.reconstruct(), (i, j)


_PRUNE_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, '.')
import chaingen as G
import paper_1911_13214_b200 as R
chains, limits, S = G.config5(n_limits=12)
for restricted in (False, True):
    costs, status, n_ops, ops = R.solve_batch(chains, limits, S, with_ops=True, restricted=restricted)
    print(int(restricted), ' '.join('%016x' % v for v in np.ascontiguousarray(costs).view(np.uint64).ravel()))
    print(int(restricted), ' '.join(str(int(x)) for x in np.asarray(status).ravel()))
    print(int(restricted), ' '.join(str(int(x)) for x in np.asarray(n_ops).ravel()))
"""


@pytest.mark.parametrize("mode", ["0", "2", "4"])
def test_batch_prune_modes(R, oracle_mod, mode):
    """The batch fill's alternative candidate paths (ROTOR_BATCH_PRUNE, read once
    per process, so each runs in a subprocess): 0 = every candidate
    (wavefront_cell), 2 / 4 = the monotone-in-m bound per 16 / 8 m.  Costs,
    statuses and schedule lengths equal the default path's (bound per 32 m) in
    both modes, and a sample of costs equals the oracle's."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for m in ("1", mode):
        env = dict(os.environ, ROTOR_BATCH_PRUNE=m)
        r = subprocess.run([sys.executable, "-c", _PRUNE_SCRIPT], cwd=root, env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs[m] = r.stdout.split("\n")
    assert outs["1"] == outs[mode]
    O = oracle_mod
    chains, limits, S = G.config5(n_limits=12)
    first = outs[mode][0].split()[1:]
    for i in range(0, len(chains), 3):
        for j in (0, 5, 11):
            c = O.OracleSolve(chains[i], limits[i][j], S, keep_d=False).cost
            assert first[i * 12 + j] == "%016x" % int(bits(np.array([c]))[0])


def test_batch_long_chains_several_bound_passes(R, oracle_mod):
    """k_batch on chains long enough that a cell's candidates span several
    32-candidate bound passes (t - s up to 150 > 64) and chains of mixed length
    in one launch (ragged L_max padding), in both modes: every cost equals the
    oracle's bit for bit, a sample of schedules equals its Algorithm 2."""
    O = oracle_mod
    chains = [G.long_chain(L=150, seed=21), G.block_chain("resnet", 70, seed=22), G.unit_chain(9)]
    S = 120
    nl = 5
    limits = [[max(1, (i * G.budget_ref(c)) // (nl + 1)) for i in range(2, nl + 2)] for c in chains]
    for restricted in (False, True):
        costs, status, n_ops, ops = R.solve_batch(chains, limits, S, with_ops=True, restricted=restricted)
        for i, ch in enumerate(chains):
            for j in range(nl):
                o = O.OracleSolve(ch, limits[i][j], S, restricted=restricted)
                c = o.cost
                if math.isinf(c):
                    assert status[i, j] == R.INFEASIBLE and math.isinf(costs[i, j]), (i, j)
                    continue
                assert status[i, j] == R.OK, (i, j, status[i, j])
                assert bits(np.array([costs[i, j]])) == bits(np.array([c])), (i, j, costs[i, j], c)
                if j in (1, 4):
                    assert [tuple(map(int, r)) for r in ops[i * nl + j]] == o.reconstruct(), (i, j)
