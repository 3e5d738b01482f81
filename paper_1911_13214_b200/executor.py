"""The paper's nn.Sequential tool (§4):
parameter estimation, optimal sequence computation, sequence processing.

  * `profile(stages, x, target)` — parameter estimation: every
    stage's forward F_all and backward run once on a sample, one after the
    other; measured are u_f, u_b (CUDA events, median of `repeat` runs), the
    sizes of a^l (the stage output), abar^l (the tensors autograd saves for
    the stage's backward, plus its output: abar^l includes a^l),
    delta^l (= a^l; the loss gradient is a scalar), and the overheads o_f, o_b
    (peak allocation during the op beyond its inputs and outputs).
    Returns a `rotor_chain`-shaped chain (stage L+1 = the loss).
  * the sequence is computed by the GPU solver (`solve`, Algorithm 1 + 2).
  * `execute(stages, ops, x, target)` — sequence processing: runs an op list
    under Table 1 with torch autograd: F_all^l keeps its input and
    builds the stage's graph (abar^l); F_ck^l runs without a graph and keeps
    its input; F_null^l runs without a graph and frees its input; B^l
    back-propagates delta^l through the stage's graph, frees it and consumes
    a^{l-1} when present (DESIGN Q18).  Parameter gradients accumulate in
    `.grad` exactly as with a plain backward: each B^l runs once.
  * `RotorSequential` ties the three together for a training step, the way
    `torch.utils.checkpoint.checkpoint_sequential` is used.

`stages` is a list of L callables (the nn.Sequential children) followed by the
loss callable `loss(out, target)`.  The DP arithmetic is not here: solving goes
through the C ABI (`paper_1911_13214_b200.solve`).
"""
from __future__ import annotations

import statistics
import time

import numpy as np
import torch

from .strategies import BWD, FALL, FCK, FNULL


def _nbytes(t) -> int:
    return int(t.numel() * t.element_size()) if isinstance(t, torch.Tensor) else 0


class _Timer:
    def __init__(self, device):
        self.cuda = device.type == "cuda"

    def __enter__(self):
        if self.cuda:
            self.e0 = torch.cuda.Event(enable_timing=True)
            self.e1 = torch.cuda.Event(enable_timing=True)
            self.e0.record()
        else:
            self.t0 = time.perf_counter()
        return self

    def __exit__(self, *exc):
        if self.cuda:
            self.e1.record()
            self.e1.synchronize()
            self.seconds = self.e0.elapsed_time(self.e1) / 1e3
        else:
            self.seconds = time.perf_counter() - self.t0


def _saved_bytes(fn, inp, params):
    """Run fn(inp) with autograd and sum the bytes of the non-parameter tensors it
    saves for backward (deduplicated by storage), together with its output."""
    seen = {}
    pids = {p.data_ptr() for p in params}

    def pack(t):
        if t.data_ptr() not in pids:
            seen[t.data_ptr()] = max(seen.get(t.data_ptr(), 0), _nbytes(t))
        return t

    with torch.enable_grad(), torch.autograd.graph.saved_tensors_hooks(pack, lambda t: t):
        out = fn(inp)
    seen[out.data_ptr()] = max(seen.get(out.data_ptr(), 0), _nbytes(out))
    if inp.data_ptr() in seen:  # the input is a^{l-1}: kept apart from abar^l (Table 1)
        del seen[inp.data_ptr()]
    return out, sum(seen.values())


class ProfiledChain:
    """A measured chain, laid out as `rotor_chain` (include/rotor.h)."""

    def __init__(self, L, uf, ub, wx, wbx, wy, of, ob):
        self.L = int(L)
        self.uf = np.ascontiguousarray(uf, dtype=np.float64)
        self.ub = np.ascontiguousarray(ub, dtype=np.float64)
        self.wx, self.wbx, self.wy, self.of, self.ob = (np.ascontiguousarray(v, dtype=np.uint64)
                                                        for v in (wx, wbx, wy, of, ob))
        self.name = "profiled"


def profile(stages, x, target, repeat: int = 3) -> ProfiledChain:
    """Parameter estimation on the sample (x, target); see the module doc."""
    dev = x.device
    cuda = dev.type == "cuda"
    L = len(stages) - 1
    n = L + 1
    if cuda:  # one untimed iteration first: library autotuning / lazy init stay out of the times
        with torch.enable_grad():
            y = x.detach()
            for f in stages[:-1]:
                y = f(y)
            stages[-1](y, target).backward()
        for f in stages:
            for p in (f.parameters() if isinstance(f, torch.nn.Module) else []):
                p.grad = None
        del y
    uf, ub, wx, wbx, wy, of, ob = [], [], [_nbytes(x)], [], [], [], []
    a = x.detach()
    for l in range(1, n + 1):
        f = stages[l - 1]
        fn = (lambda inp, f=f: f(inp, target)) if l == n else f
        params = list(f.parameters()) if isinstance(f, torch.nn.Module) else []
        inp = a.detach().requires_grad_(l > 1 or x.requires_grad)
        # forward: time (no graph) and overhead beyond the output
        ts = []
        for _ in range(repeat):
            if cuda:
                torch.cuda.synchronize(dev)
                base = torch.cuda.memory_allocated(dev)
                torch.cuda.reset_peak_memory_stats(dev)
            with torch.no_grad(), _Timer(dev) as tm:
                y = fn(inp)
            ts.append(tm.seconds)
            o_f = max(0, torch.cuda.max_memory_allocated(dev) - base - _nbytes(y)) if cuda else 0
            del y
        uf.append(statistics.median(ts))
        of.append(o_f)
        # abar^l and backward: time and overhead beyond the input gradient
        ts = []
        for _ in range(repeat):
            inp.grad = None
            out, sb = _saved_bytes(fn, inp, params)
            d = torch.ones_like(out) if l == n else torch.randn_like(out)
            if cuda:
                torch.cuda.synchronize(dev)
                base = torch.cuda.memory_allocated(dev)
                torch.cuda.reset_peak_memory_stats(dev)
            with _Timer(dev) as tm:
                torch.autograd.backward(out, d)
            ts.append(tm.seconds)
            g = _nbytes(inp.grad) if inp.requires_grad else 0
            o_b = max(0, torch.cuda.max_memory_allocated(dev) - base - g) if cuda else 0
            del out, d
        for p in params:
            p.grad = None
        ub.append(statistics.median(ts))
        ob.append(o_b)
        wbx.append(sb)
        if l < n:
            with torch.no_grad():
                a = f(a)
            wx.append(_nbytes(a))
    wy = list(wx) + [_nbytes(torch.ones((), dtype=x.dtype))]  # delta^l has the shape of a^l; delta^{L+1} scalar
    return ProfiledChain(L, uf, ub, wx, wbx, wy, of, ob)


def execute(stages, ops, x, target):
    """Sequence processing (Table 1); returns the loss (detached).

    Parameter gradients accumulate in `.grad`; a^0 = x (its gradient lands in
    x.grad when x requires grad)."""
    L = len(stages) - 1
    n = L + 1
    a = {0: x.detach()}  # a^l without graph
    ab = {}  # abar^l: (input leaf, output with the stage's graph)
    delta = None
    loss = None
    for op, l in ops:
        op, l = int(op), int(l)
        f = stages[l - 1]
        fn = (lambda inp, f=f: f(inp, target)) if l == n else f
        if op in (FALL, FCK):
            src = a[l - 1] if (l - 1) in a else ab[l - 1][1].detach()
            if op == FALL:
                inp = x if l == 1 and x.requires_grad else src.detach().requires_grad_(l > 1)
                with torch.enable_grad():
                    out = fn(inp)
                ab[l] = (inp, out)
                if l == n:
                    loss = out.detach()
            else:
                with torch.no_grad():
                    a[l] = fn(src)
        elif op == FNULL:
            src = a.pop(l - 1)
            with torch.no_grad():
                a[l] = fn(src)
        elif op == BWD:
            inp, out = ab.pop(l)
            torch.autograd.backward(out, None if l == n else delta)
            delta = inp.grad if l > 1 else None
            a.pop(l - 1, None)  # B^l consumes a^{l-1} when present (Q18)
            del inp, out
        else:
            raise ValueError(f"opcode {op}")
    return loss


class RotorSequential:
    """Optimal persistent checkpointing of an nn.Sequential + loss.

    model = RotorSequential(seq, loss_fn, sample_x, sample_target, mem_limit)
    loss = model.step(x, target)      # forward + backward of one iteration
    """

    def __init__(self, seq, loss_fn, sample_x, sample_target, mem_limit: int | None = None, slots: int = 500,
                 restricted: bool = False, chain: ProfiledChain | None = None):
        from . import solve

        self.stages = list(seq.children()) + [loss_fn]
        self.chain = chain if chain is not None else profile(self.stages, sample_x, sample_target)
        from .strategies import pytorch_schedule, replay

        self.store_all = replay(pytorch_schedule(self.chain.L), self.chain)
        self.mem_limit = int(mem_limit if mem_limit is not None else self.store_all.peak)
        self.slots = slots
        self.result = solve(self.chain, self.mem_limit, slots, restricted=restricted)
        self.ops = [tuple(o) for o in self.result.op_list()] if self.result.status == 0 else None
        if self.ops is None:
            raise ValueError(f"no schedule fits {self.mem_limit} bytes (status {self.result.status})")
        self.predicted = replay(self.ops, self.chain)

    def step(self, x, target):
        return execute(self.stages, self.ops, x, target)


__all__ = ["ProfiledChain", "profile", "execute", "RotorSequential"]
