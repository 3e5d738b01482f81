"""ORACLE — TEST INFRASTRUCTURE ONLY.

Independent CPU reference for arXiv 1911.13214 ("Rotor").  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline` leg and the
`--impl reference` arm) may import this package.  It shares no code with the
CUDA product (`paper_1911_13214_b200/`) and never imports it.

Contents
  * `OracleSolve` — ctypes wrapper of `rotor_oracle.c` (plain C DP: §5.2
    discretisation P:893-900, limits P:702-715, Theorem 1 P:717-739,
    Algorithm 1, Algorithm 2).
  * `simulate` — Table 1 + §3.1 schedule replay.
  * `brute_force` — Dijkstra over memory states (persistent per §4.1 P:560-562,
    or unrestricted), the exhaustive pin P1 for the DP.
  * `griewank_t` — the binomial (revolve) closed form, pin P2.
  * `store_all_schedule` — the "PyTorch" strategy of P:938-940, pin P3.

Every function's pins are in tests/test_oracle_*.py.
"""
from __future__ import annotations

import ctypes
import heapq
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "rotor_oracle.c")
LIB = os.path.join(HERE, "librotor_oracle.so")

FALL, FCK, FNULL, BWD = 0, 1, 2, 3
OP_NAMES = {FALL: "Fall", FCK: "Fck", FNULL: "Fnull", BWD: "B"}
NONE = 0xFFFF


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, no fast-math, no FP contraction)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
             "-o", tmp, SRC, "-lm"]
        )
        os.replace(tmp, LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P = ctypes.POINTER
        d, u64, i64, i32 = ctypes.c_double, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int
        L.oracle_new.restype = ctypes.c_void_p
        L.oracle_new.argtypes = [i32, i32, P(d), P(d), P(u64), P(u64), P(u64), P(u64), P(u64), u64, i32]
        L.oracle_free.argtypes = [ctypes.c_void_p]
        L.oracle_fill.argtypes = [ctypes.c_void_p]
        L.oracle_fill.restype = i32
        L.oracle_fill_threads.argtypes = [ctypes.c_void_p, i32]
        L.oracle_fill_threads.restype = i32
        L.oracle_set_keep_d.argtypes = [ctypes.c_void_p, i32]
        L.oracle_set_keep_d.restype = i32
        L.oracle_table.argtypes = [ctypes.c_void_p]
        L.oracle_table.restype = ctypes.c_void_p
        L.oracle_max_threads.argtypes = []
        L.oracle_max_threads.restype = i32
        L.oracle_cost.argtypes = [ctypes.c_void_p]
        L.oracle_cost.restype = d
        L.oracle_cell.argtypes = [ctypes.c_void_p, i32, i32, i64]
        L.oracle_cell.restype = d
        L.oracle_m_top.argtypes = [ctypes.c_void_p]
        L.oracle_m_top.restype = i64
        L.oracle_decision.argtypes = [ctypes.c_void_p, i32, i32, i64]
        L.oracle_decision.restype = i32
        L.oracle_reconstruct.argtypes = [ctypes.c_void_p, i32, i32, i64, P(ctypes.c_int32), i64]
        L.oracle_reconstruct.restype = i64
        L.oracle_export.argtypes = [ctypes.c_void_p, P(d), P(ctypes.c_uint16)]
        L.oracle_export.restype = i32
        L.oracle_decision_table.argtypes = [ctypes.c_void_p, P(ctypes.c_uint16)]
        L.oracle_decision_table.restype = i32
        L.oracle_slots.argtypes = [ctypes.c_void_p] + [P(i64)] * 5
        L.oracle_mnull.argtypes = [ctypes.c_void_p, i32, i32]
        L.oracle_mnull.restype = i64
        L.oracle_mall.argtypes = [ctypes.c_void_p, i32, i32]
        L.oracle_mall.restype = i64
        L.oracle_cells.argtypes = [ctypes.c_void_p]
        L.oracle_cells.restype = i64
        L.oracle_slots_of.argtypes = [u64, u64, i32]
        L.oracle_slots_of.restype = i64
        L.oracle_set_window.argtypes = [ctypes.c_void_p, i32, i32]
        L.oracle_set_window.restype = i32
        _lib = L
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def max_threads() -> int:
    """OpenMP threads the oracle would use by default (OMP_NUM_THREADS / nproc)."""
    return int(lib().oracle_max_threads())


def slots_of(x: int, M: int, S: int) -> int:
    return int(lib().oracle_slots_of(int(x), int(M), int(S)))


def cell_index(n: int, s: int, t: int) -> int:
    """Canonical table layout (include/rotor.h): s-major, then t."""
    r = s - 1  # s-major: row r holds cells (s, s..n)
    return r * n - r * (r - 1) // 2 + (t - s)


@dataclass
class Sizes:
    """Discretised chain (slots), 1-based arrays of length n+2 as in the paper."""
    L: int
    n: int
    S: int
    wx: list
    wbx: list
    wy: list
    of: list
    ob: list
    uf: list  # 1-based, float
    ub: list


class OracleSolve:
    """One DP table for (chain, M, S) — Algorithm 1 then Algorithm 2."""

    def __init__(self, chain, mem_limit: int, slots: int, restricted: bool = False, fill: bool = True,
                 window=None, threads: int = 1, keep_d: bool = True):
        """window=(s0, t0): store and fill only the cells s0 <= s <= t <= t0 (same values).
        threads > 1: the cells of each diagonal are spread over OpenMP threads (bit-identical).
        keep_d=False: do not store the fill's argmin table (Algorithm 2 needs only C)."""
        self.chain = chain
        self.L, self.n, self.S = chain.L, chain.L + 1, int(slots)
        self.M = int(mem_limit)
        self._keep = [np.ascontiguousarray(x) for x in (chain.uf, chain.ub, chain.wx, chain.wbx, chain.wy, chain.of, chain.ob)]
        uf, ub, wx, wbx, wy, of, ob = self._keep
        d, u64 = ctypes.c_double, ctypes.c_uint64
        self.h = lib().oracle_new(self.L, self.S, _p(uf, d), _p(ub, d), _p(wx, u64), _p(wbx, u64), _p(wy, u64),
                                  _p(of, u64), _p(ob, u64), self.M, 1 if restricted else 0)
        if not self.h:
            raise ValueError("oracle_new rejected the input")
        self.window = window
        if window is not None and lib().oracle_set_window(self.h, int(window[0]), int(window[1])) != 0:
            raise ValueError(f"bad window {window}")
        if not keep_d and lib().oracle_set_keep_d(self.h, 0) != 0:
            raise ValueError("oracle_set_keep_d failed")
        self.threads = int(threads)
        self.filled = False
        if fill:
            self.fill()

    def __del__(self):
        if getattr(self, "h", None):
            lib().oracle_free(self.h)
            self.h = None

    def fill(self):
        if lib().oracle_fill_threads(self.h, self.threads) != 0:
            raise MemoryError("oracle_fill: out of memory")
        self.filled = True
        return self

    @property
    def m_top(self) -> int:
        return int(lib().oracle_m_top(self.h))

    @property
    def cost(self) -> float:
        return float(lib().oracle_cost(self.h))

    def cell(self, s, t, m) -> float:
        return float(lib().oracle_cell(self.h, s, t, m))

    def decision(self, s, t, m) -> int:
        return int(lib().oracle_decision(self.h, s, t, m))

    def mnull(self, s, t) -> int:
        return int(lib().oracle_mnull(self.h, s, t))

    def mall(self, s, t) -> int:
        return int(lib().oracle_mall(self.h, s, t))

    @property
    def cells(self) -> int:
        return int(lib().oracle_cells(self.h))

    def reconstruct(self, s=1, t=None, m=None):
        """Algorithm 2 from (s,t,m); default the top cell.  None when infeasible."""
        t = self.n if t is None else t
        m = self.m_top if m is None else m
        if m < 0:
            return None
        cap = 1 << 12
        while True:
            buf = np.zeros(2 * cap, dtype=np.int32)
            cnt = int(lib().oracle_reconstruct(self.h, s, t, m, _p(buf, ctypes.c_int32), cap))
            if cnt == -1:
                return None
            if cnt < 0:
                raise RuntimeError(f"oracle_reconstruct error {cnt}")
            if cnt <= cap:
                return [(int(buf[2 * i]), int(buf[2 * i + 1])) for i in range(cnt)]
            cap = cnt

    def tables(self):
        """(C, D) in the canonical layout, shape (cells, S+1)."""
        C = np.empty((self.cells, self.S + 1), dtype=np.float64)
        D = np.empty((self.cells, self.S + 1), dtype=np.uint16)
        assert lib().oracle_export(self.h, _p(C, ctypes.c_double), _p(D, ctypes.c_uint16)) == 0
        return C, D

    def table_view(self) -> np.ndarray:
        """The filled C table itself (no copy), shape (cells, S+1); valid while self lives."""
        ptr = lib().oracle_table(self.h)
        if not ptr:
            raise RuntimeError("table not filled")
        buf = (ctypes.c_double * (self.cells * (self.S + 1))).from_address(ptr)
        return np.frombuffer(buf, dtype=np.float64).reshape(self.cells, self.S + 1)

    def decision_table(self):
        D = np.empty((self.cells, self.S + 1), dtype=np.uint16)
        assert lib().oracle_decision_table(self.h, _p(D, ctypes.c_uint16)) == 0
        return D

    def sizes(self) -> Sizes:
        n = self.n
        arrs = [np.zeros(n + 2, dtype=np.int64) for _ in range(5)]
        lib().oracle_slots(self.h, *[_p(a, ctypes.c_int64) for a in arrs])
        wx, wbx, wy, of, ob = [list(map(int, a)) for a in arrs]
        uf = [0.0] + list(map(float, self.chain.uf)) + [0.0]
        ub = [0.0] + list(map(float, self.chain.ub)) + [0.0]
        return Sizes(self.L, n, self.S, wx, wbx, wy, of, ob, uf, ub)


# ----------------------------------------------------------------------------
# Simulator: Table 1 and §3.1
# ----------------------------------------------------------------------------
@dataclass
class SimReport:
    valid: bool
    peak: int
    makespan: float
    n_ops: int
    failure: str = ""


def simulate(ops, sz: Sizes, budget: int, s: int = 1, t: int | None = None) -> SimReport:
    """Replay `ops` on the (sub-)chain of stages s..t.

    Initial memory {a^{s-1}, delta^t} ("the memory contains {a^0 = x}";
    delta^{L+1} present from the start, Q19).  Each op needs its inputs
    present; the memory during an op is the data present + its new output +
    its overhead, except that B^l's output delta^{l-1}
    is not charged (Q8, the convention of m_all P:708).  F_null needs a^{l-1}
    itself (Q17); B^l consumes a^{l-1} when present, else keeps abar^{l-1}
    (Table 1 second row, Q18).  Producing an item already in memory is
    rejected (never emitted by the DP).  Valid iff every op is valid, the peak
    is <= budget, and delta^{s-1} is present at the end.
    """
    t = sz.n if t is None else t
    A = {s - 1}  # present a^i
    AB = set()  # present abar^i
    dlt = t  # index of the one present delta
    cur = sz.wx[s - 1] + sz.wy[t]
    peak = 0
    time = 0.0

    def fail(i, why):
        return SimReport(False, peak, time, len(ops), f"op {i} {OP_NAMES.get(ops[i][0], '?')} {ops[i][1]}: {why}")

    for i, (op, l) in enumerate(ops):
        if not (s <= l <= t):
            return fail(i, "stage out of range")
        if op in (FALL, FCK):
            if not ((l - 1) in A or (l - 1 >= s and (l - 1) in AB)):
                return fail(i, "input a^{l-1} / abar^{l-1} missing")
            if op == FALL:
                if l in AB:
                    return fail(i, "abar already present")
                during = cur + sz.wbx[l] + sz.of[l]
                AB.add(l)
                cur += sz.wbx[l]
            else:
                if l > sz.L or l in A:
                    return fail(i, "a^l does not exist or already present")
                during = cur + sz.wx[l] + sz.of[l]
                A.add(l)
                cur += sz.wx[l]
            time += sz.uf[l]
        elif op == FNULL:
            if (l - 1) not in A:
                return fail(i, "a^{l-1} missing (F_null cannot use abar, Q17)")
            if l > sz.L or l in A:
                return fail(i, "a^l does not exist or already present")
            during = cur + sz.wx[l] + sz.of[l]
            A.discard(l - 1)
            A.add(l)
            cur += sz.wx[l] - sz.wx[l - 1]
            time += sz.uf[l]
        elif op == BWD:
            if dlt != l:
                return fail(i, f"delta^{l} missing (have delta^{dlt})")
            if l not in AB:
                return fail(i, "abar^l missing")
            has_a = (l - 1) in A
            has_ab = (l - 1 >= s) and (l - 1) in AB
            if not (has_a or has_ab):
                return fail(i, "a^{l-1} / abar^{l-1} missing")
            during = cur + sz.ob[l]  # Q8: delta^{l-1} not charged during B^l
            AB.discard(l)
            cur -= sz.wbx[l]
            if has_a:
                A.discard(l - 1)
                cur -= sz.wx[l - 1]
            cur += sz.wy[l - 1] - sz.wy[l]
            dlt = l - 1
            time += sz.ub[l]
        else:
            return fail(i, "bad opcode")
        peak = max(peak, during)
        if during > budget:
            return SimReport(False, peak, time, len(ops), f"op {i}: memory {during} > budget {budget}")
    if dlt != s - 1:
        return SimReport(False, peak, time, len(ops), f"final delta^{dlt}, expected delta^{s - 1}")
    return SimReport(True, peak, time, len(ops))


def store_all_schedule(n: int):
    """The "PyTorch" strategy: F_all^1..F_all^n then B^n..B^1."""
    return [(FALL, l) for l in range(1, n + 1)] + [(BWD, l) for l in range(n, 0, -1)]


# ----------------------------------------------------------------------------
# Exhaustive search (pin P1): Dijkstra over memory states
# ----------------------------------------------------------------------------
def brute_force(sz: Sizes, budget: int, s: int = 1, t: int | None = None, persistent: bool = True,
                max_states: int = 5_000_000):
    """Minimal makespan over all valid sequences of Table-1 ops on stages s..t.

    State = (present a^i, 'kept' a^i, present abar^i, delta index).  Same memory
    accounting as `simulate`.  With `persistent`, an a^i that served as the
    retained input of F_ck^{i+1} / F_all^{i+1} (a checkpoint, "any
    checkpointed value is kept in memory until it is used in the backward
    phase") may afterwards be consumed only by B^{i+1}, not by F_null^{i+1}
    (Q20); a^{s-1} is such a checkpoint from the start.  Without it every valid
    sequence is searched (the non-persistent problem of P:676-686).
    Returns (cost, ops) or (inf, None).
    """
    t = sz.n if t is None else t
    wx, wbx, wy, of, ob, uf, ub = sz.wx, sz.wbx, sz.wy, sz.of, sz.ob, sz.uf, sz.ub
    # bit i of A/K: a^{i}; bit i of B: abar^{i}
    A0 = 1 << (s - 1)
    K0 = A0 if persistent else 0
    start = (A0, K0, 0, t)

    cur0 = wx[s - 1] + wy[t]
    dist = {start: 0.0}
    prev = {start: None}
    heap = [(0.0, start, cur0)]
    while heap:
        c, st, cur = heapq.heappop(heap)
        if c > dist.get(st, math.inf):
            continue
        A, K, B, dl = st
        if dl == s - 1:
            ops = []
            while prev[st] is not None:
                st, op = prev[st]
                ops.append(op)
            return c, ops[::-1]
        if len(dist) > max_states:
            raise RuntimeError("brute force: state space too large")
        succ = []
        for l in range(s, dl + 1):
            in_a = (A >> (l - 1)) & 1
            in_ab = (l - 1 >= s) and ((B >> (l - 1)) & 1)
            if not (in_a or in_ab):
                continue
            # F_all^l: keeps its input; if the input is a^{l-1} it becomes a checkpoint
            if not (B >> l) & 1 and cur + wbx[l] + of[l] <= budget:
                if in_ab:
                    succ.append(((A, K, B | (1 << l), dl), uf[l], (FALL, l), wbx[l]))
                if in_a:
                    k2 = (K | (1 << (l - 1))) if persistent else K
                    succ.append(((A, k2, B | (1 << l), dl), uf[l], (FALL, l), wbx[l]))
            if l <= min(t - 1, sz.L) and not (A >> l) & 1 and cur + wx[l] + of[l] <= budget:
                # F_ck^l
                if in_ab:
                    succ.append(((A | (1 << l), K, B, dl), uf[l], (FCK, l), wx[l]))
                if in_a:
                    k2 = (K | (1 << (l - 1))) if persistent else K
                    succ.append(((A | (1 << l), k2, B, dl), uf[l], (FCK, l), wx[l]))
                # F_null^l: consumes a^{l-1}, which must not be a kept checkpoint
                if in_a and not (K >> (l - 1)) & 1:
                    A2 = (A & ~(1 << (l - 1))) | (1 << l)
                    succ.append(((A2, K, B, dl), uf[l], (FNULL, l), wx[l] - wx[l - 1]))
        # B^dl
        l = dl
        if (B >> l) & 1 and cur + ob[l] <= budget:
            in_a = (A >> (l - 1)) & 1
            in_ab = (l - 1 >= s) and ((B >> (l - 1)) & 1)
            if in_a or in_ab:
                A2, K2 = A, K
                dm = wy[l - 1] - wy[l] - wbx[l]
                if in_a:
                    A2 &= ~(1 << (l - 1))
                    K2 &= ~(1 << (l - 1))
                    dm -= wx[l - 1]
                succ.append(((A2, K2, B & ~(1 << l), l - 1), ub[l], (BWD, l), dm))
        for st2, dc, op, dm in succ:
            c2 = c + dc
            if c2 < dist.get(st2, math.inf):
                dist[st2] = c2
                prev[st2] = (st, op)
                heapq.heappush(heap, (c2, st2, cur + dm))
    return math.inf, None


# ----------------------------------------------------------------------------
# Griewank-Walther binomial closed form (pin P2, cited P:45-47)
# ----------------------------------------------------------------------------
def beta(c: int, r: int) -> int:
    return math.comb(c + r, c)


def griewank_t(l: int, c: int) -> int:
    """Minimal number of forward (advance) steps to reverse l steps with c checkpoints.

    t(l,c) = r*l - beta(c+1, r-1), r the smallest integer with beta(c, r) >= l.
    """
    if l <= 1:
        return 0
    r = 0
    while beta(c, r) < l:
        r += 1
    return r * l - beta(c + 1, r - 1)
