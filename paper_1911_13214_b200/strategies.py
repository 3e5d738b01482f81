"""The paper's comparison strategies (§5.2) and the simulated
throughput-vs-memory sweep of SURVEY §8(f) rank 3, on synthetic profiles.

Strategies:
  * ``pytorch``    — store all: F_all^1..F_all^n, B^n..B^1;
  * ``sequential`` — PyTorch's checkpoint_sequential with k segments: in the
    forward phase only the input of every segment is kept, so every forward
    but those of the last segment runs twice; k takes 10 values from 2 to
    2·sqrt(L);
  * ``revolve``    — the optimal AD-model schedule made valid by keeping only
    activations a and running F_all right before each backward:
    the restricted DP (F_all only on single stages), solved on the GPU;
  * ``optimal``    — Algorithm 1 at 10 memory limits equally spaced between 0
    and the memory of the pytorch strategy, solved on the GPU.

Host-side logic only: the baseline generators build op lists, `replay` runs
Table 1 on byte sizes to get each schedule's peak memory and time,
and the DP solves go through the C ABI (`solve_batch`).  `replay` is the
product's own simulator (the oracle's, in `oracle/`, is independent test
infrastructure; tests/test_strategies.py checks the two agree).

A chain is laid out as `rotor_chain` (include/rotor.h): uf/ub/of/ob/wbx index
stage l = 1..n at [l-1], wx index a^l (l = 0..L) at [l], wy index delta^l
(l = 0..n) at [l]; n = L + 1 (the loss is stage n).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

FALL, FCK, FNULL, BWD = 0, 1, 2, 3


# ----------------------------------------------------------------------------
# baseline generators
# ----------------------------------------------------------------------------
def pytorch_schedule(L: int):
    """Store all: F_all^1..F_all^n, B^n..B^1."""
    n = L + 1
    return [(FALL, l) for l in range(1, n + 1)] + [(BWD, l) for l in range(n, 0, -1)]


def segment_bounds(n: int, k: int):
    """Stages 1..n cut into k contiguous, non-empty segments (sizes differ by <= 1)."""
    k = max(1, min(k, n))
    return [round(i * n / k) for i in range(k + 1)]


def sequential_schedule(L: int, k: int):
    """checkpoint_sequential with k segments.

    Forward: every segment but the last keeps its input (F_ck on its first stage,
    F_null on the others); the last segment saves all (F_all).  Backward, last
    segment first: B over the saved segment, then for every earlier segment a
    recomputation with F_all from its kept input followed by its B steps.
    """
    n = L + 1
    b = segment_bounds(n, k)
    ops = []
    for j in range(len(b) - 2):  # non-last segments
        ops.append((FCK, b[j] + 1))
        ops += [(FNULL, l) for l in range(b[j] + 2, b[j + 1] + 1)]
    ops += [(FALL, l) for l in range(b[-2] + 1, n + 1)]
    ops += [(BWD, l) for l in range(n, b[-2], -1)]
    for j in range(len(b) - 3, -1, -1):
        ops += [(FALL, l) for l in range(b[j] + 1, b[j + 1] + 1)]
        ops += [(BWD, l) for l in range(b[j + 1], b[j], -1)]
    return ops


def sequential_segment_counts(L: int, count: int = 10):
    """`count` segment numbers from 2 (always included) to 2·sqrt(L)."""
    hi = max(2, int(round(2 * math.sqrt(L))))
    vals = sorted({int(round(2 + (hi - 2) * i / max(1, count - 1))) for i in range(count)})
    return [v for v in vals if v <= L + 1]


# ----------------------------------------------------------------------------
# Table 1 replay on byte sizes
# ----------------------------------------------------------------------------
@dataclass
class Replay:
    valid: bool
    peak: int  # bytes (or whatever unit the sizes are in)
    time: float
    error: str = ""


def replay(ops, chain) -> Replay:
    """Run `ops` on `chain` under Table 1.

    Memory starts as {a^0, delta^n} (the loss gradient is present from
    the start).  During an op the memory holds the data present, its new output
    and its overhead; B^l's output delta^{l-1} is not
    charged (the m_all convention of P:708, DESIGN Q8).  F_null needs a^{l-1}
    itself (Table 1 has no abar row for it); B^l consumes a^{l-1} when present,
    else uses abar^{l-1}, which stays (Table 1, second row).  The sequence is
    valid when every op finds its inputs and delta^0 is present at the end.
    """
    n = int(chain.L) + 1
    wx = [int(x) for x in chain.wx]
    wbx = [0] + [int(x) for x in chain.wbx]
    wy = [int(x) for x in chain.wy]
    of = [0] + [int(x) for x in chain.of]
    ob = [0] + [int(x) for x in chain.ob]
    uf = [0.0] + [float(x) for x in chain.uf]
    ub = [0.0] + [float(x) for x in chain.ub]
    have_a = {0}
    have_ab = set()
    grad = n
    mem = wx[0] + wy[n]
    peak = 0
    t = 0.0
    for i, (op, l) in enumerate(ops):
        op, l = int(op), int(l)
        if not 1 <= l <= n:
            return Replay(False, peak, t, f"op {i}: stage {l} out of range")
        if op in (FALL, FCK, FNULL):
            if op == FNULL:
                ok = (l - 1) in have_a
            else:
                ok = (l - 1) in have_a or (l - 1) in have_ab
            if not ok:
                return Replay(False, peak, t, f"op {i}: input of forward {l} missing")
            if op == FALL:
                if l in have_ab:
                    return Replay(False, peak, t, f"op {i}: abar^{l} already present")
                out = wbx[l]
            else:
                if l == n or l in have_a:
                    return Replay(False, peak, t, f"op {i}: a^{l} does not exist or is present")
                out = wx[l]
            peak = max(peak, mem + out + of[l])
            mem += out
            if op == FALL:
                have_ab.add(l)
            else:
                have_a.add(l)
            if op == FNULL:
                have_a.discard(l - 1)
                mem -= wx[l - 1]
            t += uf[l]
        elif op == BWD:
            if grad != l or l not in have_ab:
                return Replay(False, peak, t, f"op {i}: delta^{l} or abar^{l} missing")
            use_a = (l - 1) in have_a
            if not (use_a or (l - 1) in have_ab):
                return Replay(False, peak, t, f"op {i}: a^{l - 1} missing")
            peak = max(peak, mem + ob[l])
            have_ab.discard(l)
            mem -= wbx[l]
            if use_a:
                have_a.discard(l - 1)
                mem -= wx[l - 1]
            mem += wy[l - 1] - wy[l]
            grad = l - 1
            t += ub[l]
        else:
            return Replay(False, peak, t, f"op {i}: opcode {op}")
    if grad != 0:
        return Replay(False, peak, t, f"ends with delta^{grad}")
    return Replay(True, peak, t)


# ----------------------------------------------------------------------------
# the sweep
# ----------------------------------------------------------------------------
@dataclass
class Point:
    strategy: str
    param: float  # segments (sequential) or memory limit in bytes (optimal / revolve)
    peak: int  # replayed peak memory, bytes
    time: float  # replayed makespan of one training iteration, seconds
    feasible: bool = True

    @property
    def throughput(self) -> float:
        return 1.0 / self.time if self.feasible and self.time > 0 else 0.0


def compare(chain, slots: int = 500, n_limits: int = 10, seg_counts=None):
    """The §5.2 comparison on one chain: pytorch, sequential (2..2·sqrt(L)
    segments), and revolve / optimal at `n_limits` limits i/n_limits × the
    pytorch peak (i = 1..n_limits), the DP solves batched on the GPU.
    Returns a list of `Point` (every schedule replayed on byte sizes)."""
    from . import INFEASIBLE, OK, solve_batch

    L = int(chain.L)
    pts = []
    base = replay(pytorch_schedule(L), chain)
    pts.append(Point("pytorch", 0, base.peak, base.time))
    for k in seg_counts or sequential_segment_counts(L):
        r = replay(sequential_schedule(L, k), chain)
        pts.append(Point("sequential", k, r.peak, r.time, r.valid))
    limits = [max(1, base.peak * i // n_limits) for i in range(1, n_limits + 1)]
    for name, restricted in (("revolve", True), ("optimal", False)):
        costs, status, _, ops = solve_batch([chain], [limits], slots, with_ops=True, restricted=restricted)
        for j, M in enumerate(limits):
            st = int(status[0, j])
            if st == INFEASIBLE:
                pts.append(Point(name, M, 0, math.inf, False))
                continue
            assert st == OK, st
            r = replay([tuple(o) for o in ops[j]], chain)
            assert r.valid, r.error
            pts.append(Point(name, M, r.peak, r.time))
    return pts


def pareto(points):
    """Best throughput reachable at each peak memory (the envelope the paper plots)."""
    out = []
    best = 0.0
    for p in sorted((p for p in points if p.feasible), key=lambda p: (p.peak, -p.throughput)):
        if p.throughput > best:
            out.append(p)
            best = p.throughput
    return out
