"""Seeded synthetic chain generators — shared test/bench INPUT module.

This module is deliberately *outside* both the oracle (`oracle/`) and the
product (`paper_1911_13214_b200/`).  It only draws numbers: it contains none of
the method's arithmetic (no discretisation, no limits, no DP, no simulation).
Both sides receive the same arrays from here and nothing else is shared.

A chain follows the paper's model (§3.1, Table 1):
stages l = 1..L+1 (stage L+1 is the loss) with

  uf[l-1], ub[l-1]   forward / backward time of stage l       (fp64 seconds)
  wx[l]              size of a^l,      l = 0..L                 (uint64 bytes)
  wbx[l-1]           size of abar^l,   l = 1..L+1
  wy[l]              size of delta^l,  l = 0..L+1
  of[l-1], ob[l-1]   forward / backward memory overhead of stage l

Array index conventions are those of `include/rotor.h` (rotor_chain).

Random numbers: splitmix64(seed) counter stream; u = (x >> 11) * 2^-53;
z = Box-Muller N(0,1).  The per-config recipes are the ones stated in
DESIGN.md §"Input recipe".
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

MASK64 = (1 << 64) - 1
MiB = 1 << 20


class SplitMix64:
    """splitmix64 counter generator (Steele, Lea, Flood 2014)."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def uniform(self) -> float:
        """u in [0, 1) with 53 random bits."""
        return (self.next_u64() >> 11) * (2.0 ** -53)

    def normal(self) -> float:
        """Box-Muller N(0,1) (cosine branch only; two draws per sample)."""
        u1 = 1.0 - self.uniform()  # (0, 1]
        u2 = self.uniform()
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)

    def randint(self, lo: int, hi: int) -> int:
        """Integer in [lo, hi] inclusive (modulo bias irrelevant for tests)."""
        return lo + self.next_u64() % (hi - lo + 1)


@dataclass
class Chain:
    """A heterogeneous chain of L stages + the loss stage (L+1 stages in all)."""

    L: int
    uf: np.ndarray  # float64 [L+1]
    ub: np.ndarray  # float64 [L+1]
    wx: np.ndarray  # uint64  [L+1]  a^0..a^L
    wbx: np.ndarray  # uint64 [L+1]  abar^1..abar^{L+1}
    wy: np.ndarray  # uint64  [L+2]  delta^0..delta^{L+1}
    of: np.ndarray  # uint64  [L+1]
    ob: np.ndarray  # uint64  [L+1]
    name: str = ""

    def __post_init__(self):
        n = self.L + 1
        self.uf = np.ascontiguousarray(self.uf, dtype=np.float64)
        self.ub = np.ascontiguousarray(self.ub, dtype=np.float64)
        for f in ("wx", "wbx", "of", "ob"):
            setattr(self, f, np.ascontiguousarray(getattr(self, f), dtype=np.uint64))
        self.wy = np.ascontiguousarray(self.wy, dtype=np.uint64)
        assert self.L >= 1
        for f in ("uf", "ub", "wx", "wbx", "of", "ob"):
            assert getattr(self, f).shape == (n,), (f, getattr(self, f).shape)
        assert self.wy.shape == (n + 1,)

    @property
    def n(self) -> int:
        return self.L + 1

    def window(self, s: int, t: int) -> "Chain":
        """The sub-chain of stages s..t (1-based, t <= L+1) as a chain of its own.

        Stage s of the parent becomes stage 1; a^{s-1} becomes a^0; the last stage
        t becomes the 'loss' stage index.  Used for sampled parity (every cell
        C[s',t',m] with s <= s' <= t' <= t depends only on stages s..t).
        """
        assert 1 <= s <= t <= self.n
        Lw = t - s  # stages s..t -> t-s+1 stages -> L = t-s
        return Chain(
            L=Lw,
            uf=self.uf[s - 1 : t].copy(),
            ub=self.ub[s - 1 : t].copy(),
            wx=self.wx[s - 1 : t].copy(),  # a^{s-1} .. a^{t-1}
            wbx=self.wbx[s - 1 : t].copy(),
            wy=self.wy[s - 1 : t + 1].copy(),  # delta^{s-1} .. delta^{t}
            of=self.of[s - 1 : t].copy(),
            ob=self.ob[s - 1 : t].copy(),
            name=f"{self.name}[{s}:{t}]",
        )


@dataclass
class Problem:
    chain: Chain
    mem_limit: int  # bytes
    slots: int  # S
    name: str = ""
    meta: dict = field(default_factory=dict)


def budget_ref(ch: Chain) -> int:
    """A reference memory scale for choosing limits M = f * budget_ref.

    Only a number used to *pick* a memory limit (generator convention, not the
    method): input + every abar + the loss gradient + the largest overhead.
    """
    return int(
        int(ch.wx[0])
        + int(ch.wbx.sum())
        + int(ch.wy[-1])
        + int(max(int(ch.of.max()), int(ch.ob.max())))
    )


def _u64(x: float) -> int:
    return max(0, int(round(x)))


# ----------------------------------------------------------------------------
# config 1: homogeneous unit chain (SURVEY §8(d) cfg 1)
# ----------------------------------------------------------------------------
def unit_chain(L: int, uf: float = 1.0, ub: float = 1.0, size: int = 1) -> Chain:
    n = L + 1
    return Chain(
        L=L,
        uf=np.full(n, uf),
        ub=np.full(n, ub),
        wx=np.full(n, size),
        wbx=np.full(n, size),
        wy=np.full(n + 1, size),
        of=np.zeros(n),
        ob=np.zeros(n),
        name=f"unit{L}",
    )


def config1() -> Problem:
    ch = unit_chain(10)
    return Problem(ch, mem_limit=50, slots=50, name="cfg1_unit_L10_S50")


# ----------------------------------------------------------------------------
# shaped generators (configs 2-5)
# ----------------------------------------------------------------------------
LOSS_UF = 10e-6
LOSS_UB = 10e-6
LOSS_WBX = 128
LOSS_WY = 4


def _finish(rng, L, wa, ufs, c_abar=(2.5, 1.5), name="", wbx_override=None) -> Chain:
    """Common tail: abar, overheads, backward times and the loss stage.

    wa:  list of L+1 activation sizes a^0..a^L (float bytes)
    ufs: list of L forward times for stages 1..L
    """
    assert len(wa) == L + 1 and len(ufs) == L
    n = L + 1
    uf = np.zeros(n)
    ub = np.zeros(n)
    wbx = np.zeros(n, dtype=np.uint64)
    of = np.zeros(n, dtype=np.uint64)
    ob = np.zeros(n, dtype=np.uint64)
    wx = np.array([_u64(x) for x in wa], dtype=np.uint64)
    for l in range(1, L + 1):
        a = float(wx[l])
        r = c_abar[0] + c_abar[1] * rng.uniform()
        wbx[l - 1] = _u64(a * r) if wbx_override is None else wbx_override[l - 1]
        of[l - 1] = _u64(a * 0.5 * rng.uniform())
        ob[l - 1] = _u64(a * rng.uniform())
        uf[l - 1] = ufs[l - 1]
        ub[l - 1] = ufs[l - 1] * (1.8 + 0.4 * rng.uniform())
    # loss stage L+1
    uf[n - 1] = LOSS_UF
    ub[n - 1] = LOSS_UB
    wbx[n - 1] = LOSS_WBX
    wy = np.zeros(n + 1, dtype=np.uint64)
    wy[: n] = wx  # omega_delta = omega_a "in practice"
    wy[n] = LOSS_WY
    return Chain(L=L, uf=uf, ub=ub, wx=wx, wbx=wbx, wy=wy, of=of, ob=ob, name=name)


def resnet_chain(L_target: int, groups=(3, 4, 23, 3), batch=32, seed=1, name="resnet101") -> Chain:
    """ResNet-shaped chain: 1 stem stage + bottleneck blocks x 3 stages.

    With groups (3,4,23,3) this is 1 + 33*3 = 100 stages (config 2).  Group g
    output a = A0 * 2^-g * (0.95 + 0.1u), A0 = B*256*56^2*4 B; the first two
    stages of a block (1x1 reduce, 3x3) use 1/4 of that.  u_f = 1 ms * c *
    (0.9+0.2u), c = 1 (1x1) or 2.25 (3x3).
    """
    rng = SplitMix64(seed)
    A0 = batch * 256 * 56 * 56 * 4
    wa = [batch * 3 * 224 * 224 * 4]  # a^0: input image
    ufs = []
    # stem: conv7x7 + pool -> 64 x 56 x 56
    wa.append(batch * 64 * 56 * 56 * 4 * (0.95 + 0.1 * rng.uniform()))
    ufs.append(1e-3 * 2.25 * (0.9 + 0.2 * rng.uniform()))
    for g, nb in enumerate(groups):
        for _ in range(nb):
            for st in range(3):
                base = A0 * 2.0 ** (-g) * (0.95 + 0.1 * rng.uniform())
                wa.append(base * (0.25 if st < 2 else 1.0))
                c = 2.25 if st == 1 else 1.0
                ufs.append(1e-3 * c * (0.9 + 0.2 * rng.uniform()))
    L = len(ufs)
    assert L == L_target, (L, L_target)
    return _finish(rng, L, wa, ufs, name=name)


def config2() -> Problem:
    ch = resnet_chain(100, seed=1)
    return Problem(ch, mem_limit=int(0.4 * budget_ref(ch)), slots=500, name="cfg2_resnet101_L100_S500")


def densenet_chain(seed=2, batch=32, blocks=(6, 12, 48, 32), name="densenet201") -> Chain:
    """DenseNet-201-shaped chain (config 3): 2 stem + 98 layers x 3 + 3 transitions + 1 head = 300.

    Layer i of block b: a = B*c*H_b^2*4*(0.95+0.1u), c = c0_b + 32 i,
    c0 = (64,128,256,896), H_b = 56/2^b; abar = a*(4+6u) (large abar/a).
    """
    rng = SplitMix64(seed)
    c0 = (64, 128, 256, 896)
    wa = [batch * 3 * 224 * 224 * 4]
    ufs = []
    # stem: conv 7x7 (64 x 112^2) and pool (64 x 56^2)
    wa.append(batch * 64 * 112 * 112 * 4 * (0.95 + 0.1 * rng.uniform()))
    ufs.append(1e-3 * 2.25 * (0.9 + 0.2 * rng.uniform()))
    wa.append(batch * 64 * 56 * 56 * 4 * (0.95 + 0.1 * rng.uniform()))
    ufs.append(1e-3 * 1.0 * (0.9 + 0.2 * rng.uniform()))
    for b, nl in enumerate(blocks):
        H = 56 // (2 ** b)
        for i in range(nl):
            c = c0[b] + 32 * i
            for st in range(3):
                wa.append(batch * c * H * H * 4 * (0.95 + 0.1 * rng.uniform()))
                cc = 2.25 if st == 1 else 1.0
                ufs.append(1e-3 * cc * (0.9 + 0.2 * rng.uniform()))
        if b < len(blocks) - 1:  # transition: 1x1 conv + 2x2 pool
            cout = (c0[b] + 32 * nl) // 2
            wa.append(batch * cout * (H // 2) ** 2 * 4 * (0.95 + 0.1 * rng.uniform()))
            ufs.append(1e-3 * 1.0 * (0.9 + 0.2 * rng.uniform()))
    # head: global pool + fc
    wa.append(batch * 1000 * 4)
    ufs.append(1e-3 * 0.2 * (0.9 + 0.2 * rng.uniform()))
    L = len(ufs)
    assert L == 300, L
    # abar/a in [4, 10)
    return _finish(rng, L, wa, ufs, c_abar=(4.0, 6.0), name=name)


def config3() -> Problem:
    ch = densenet_chain(seed=2)
    return Problem(ch, mem_limit=int(0.3 * budget_ref(ch)), slots=2000, name="cfg3_densenet201_L300_S2000")


def long_chain(L=1000, seed=4, name="long") -> Chain:
    """Long heterogeneous chain (config 4).

    a = 16 MiB * exp(clip(z, +-2.5)); abar = a*(1+5u); u_f = 1 ms *
    exp(0.7*clip(z', +-2.5)); u_b = u_f*(1.5+u); o_f = a*0.5u; o_b = a*u.
    """
    rng = SplitMix64(seed)
    clip = lambda z: max(-2.5, min(2.5, z))
    n = L + 1
    wa = [16 * MiB * math.exp(clip(rng.normal())) for _ in range(L + 1)]
    ufs = [1e-3 * math.exp(0.7 * clip(rng.normal())) for _ in range(L)]
    uf = np.zeros(n)
    ub = np.zeros(n)
    wbx = np.zeros(n, dtype=np.uint64)
    of = np.zeros(n, dtype=np.uint64)
    ob = np.zeros(n, dtype=np.uint64)
    wx = np.array([_u64(x) for x in wa], dtype=np.uint64)
    for l in range(1, L + 1):
        a = float(wx[l])
        wbx[l - 1] = _u64(a * (1.0 + 5.0 * rng.uniform()))
        of[l - 1] = _u64(a * 0.5 * rng.uniform())
        ob[l - 1] = _u64(a * rng.uniform())
        uf[l - 1] = ufs[l - 1]
        ub[l - 1] = ufs[l - 1] * (1.5 + rng.uniform())
    uf[n - 1] = LOSS_UF
    ub[n - 1] = LOSS_UB
    wbx[n - 1] = LOSS_WBX
    wy = np.zeros(n + 1, dtype=np.uint64)
    wy[:n] = wx
    wy[n] = LOSS_WY
    return Chain(L=L, uf=uf, ub=ub, wx=wx, wbx=wbx, wy=wy, of=of, ob=ob, name=name)


def config4(f: float = 0.25) -> Problem:
    ch = long_chain(1000, seed=4)
    return Problem(ch, mem_limit=int(f * budget_ref(ch)), slots=4000, name="cfg4_long_L1000_S4000")


# config 5: 8 ResNet/VGG-shaped chains at block granularity
CFG5_CHAINS = (
    ("resnet18", 14), ("resnet34", 22), ("resnet50", 22), ("resnet101", 39),
    ("resnet152", 56), ("vgg11", 29), ("vgg16", 37), ("vgg19", 43),
)


def block_chain(kind: str, L: int, seed: int, batch: int = 32) -> Chain:
    """Block-granularity ResNet / VGG shaped chain with exactly L stages.

    ResNet: activations halve every quarter of the chain (4 groups), the first
    stage is the stem on a 224^2 input.  VGG: activations halve at 5 pooling
    points spread evenly, early activations large, u_f proportional to the
    conv FLOPs (channels^2 * H^2 up to a constant).
    """
    rng = SplitMix64(seed)
    wa = [batch * 3 * 224 * 224 * 4]
    ufs = []
    if kind.startswith("resnet"):
        A0 = batch * 256 * 56 * 56 * 4
        for l in range(L):
            g = min(3, (4 * l) // L)
            wa.append(A0 * 2.0 ** (-g) * (0.95 + 0.1 * rng.uniform()))
            ufs.append(3e-3 * (0.9 + 0.2 * rng.uniform()))
        return _finish(rng, L, wa, ufs, name=f"{kind}_L{L}")
    # VGG
    ch, H = 64, 224
    pools = {int(round((k + 1) * L / 6.0)) for k in range(5)}
    for l in range(L):
        if l in pools:
            H //= 2
            ch = min(512, ch * 2)
        wa.append(batch * ch * H * H * 4 * (0.95 + 0.1 * rng.uniform()))
        flops = ch * ch * H * H * 9.0
        ufs.append(1e-3 * flops / (64 * 64 * 224 * 224 * 9.0) * (0.9 + 0.2 * rng.uniform()) + 1e-4)
    return _finish(rng, L, wa, ufs, c_abar=(1.5, 1.0), name=f"{kind}_L{L}")


def config5_chains():
    return [block_chain(k, L, seed=10 + i) for i, (k, L) in enumerate(CFG5_CHAINS)]


def config5(n_limits: int = 256, slots: int = 500):
    """256 limits x 8 chains: M_i = (i/n_limits) * budget_ref for i = 1..n_limits."""
    chains = config5_chains()
    limits = [[max(1, (i * budget_ref(c)) // n_limits) for i in range(1, n_limits + 1)] for c in chains]
    return chains, limits, slots


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4}


# ----------------------------------------------------------------------------
# tiny random chains for pins (sizes given directly in slots: M = S, slot = 1 B)
# ----------------------------------------------------------------------------
def tiny_chain(
    rng: SplitMix64,
    L: int,
    size_max: int = 3,
    time_max: int = 9,
    ovh_max: int = 2,
    abar_ge_a: bool = True,
    delta_eq_a: bool = True,
    int_times: bool = True,
    allow_zero_time: bool = False,
) -> Chain:
    """Random small chain with integer byte sizes (to be used with M = S)."""
    n = L + 1
    wx = [rng.randint(0, size_max) for _ in range(n)]
    wbx = []
    for l in range(1, n + 1):
        a = wx[l] if l <= L else 0
        lo = a if abar_ge_a else 0
        wbx.append(rng.randint(lo, max(lo, size_max + (1 if abar_ge_a else 0))))
    if delta_eq_a:
        wy = wx + [rng.randint(0, size_max)]
    else:
        wy = [rng.randint(0, size_max) for _ in range(n + 1)]
    of = [rng.randint(0, ovh_max) for _ in range(n)]
    ob = [rng.randint(0, ovh_max) for _ in range(n)]
    lo_t = 0 if allow_zero_time else 1
    if int_times:
        uf = [float(rng.randint(lo_t, time_max)) for _ in range(n)]
        ub = [float(rng.randint(lo_t, time_max)) for _ in range(n)]
    else:
        uf = [rng.uniform() * time_max + (0.0 if allow_zero_time else 1e-3) for _ in range(n)]
        ub = [rng.uniform() * time_max + (0.0 if allow_zero_time else 1e-3) for _ in range(n)]
    return Chain(L=L, uf=uf, ub=ub, wx=wx, wbx=wbx, wy=wy, of=of, ob=ob, name=f"tiny{L}")


def random_chain(rng: SplitMix64, L: int, real_times: bool = True, big: bool = False) -> Chain:
    """Random heterogeneous chain with byte sizes spread over a wide range."""
    n = L + 1
    scale = 1 << 20
    wx = [int(scale * math.exp(rng.normal())) if rng.uniform() > 0.05 else 0 for _ in range(n)]
    wbx = [int((wx[l] if l <= L else 0) * (1.0 + (8.0 if big else 3.0) * rng.uniform())) + rng.randint(0, 1024)
           for l in range(1, n + 1)]
    wy = wx + [rng.randint(0, 4096)]
    of = [int(scale * 0.5 * rng.uniform()) for _ in range(n)]
    ob = [int(scale * rng.uniform()) for _ in range(n)]
    if real_times:
        uf = [1e-3 * math.exp(0.7 * rng.normal()) for _ in range(n)]
        ub = [x * (1.5 + rng.uniform()) for x in uf]
    else:
        uf = [float(rng.randint(0, 20)) for _ in range(n)]
        ub = [float(rng.randint(0, 20)) for _ in range(n)]
    return Chain(L=L, uf=uf, ub=ub, wx=wx, wbx=wbx, wy=wy, of=of, ob=ob, name=f"rand{L}")
