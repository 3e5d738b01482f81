"""The nn.Sequential tool (§4).

CPU: executing any valid schedule — store-all, checkpoint_sequential, and the
DP-optimal schedules the oracle reconstructs at several budgets — yields the
loss and parameter/input gradients of a plain backward bit for bit (fp64 MLP:
recomputed forwards are deterministic); the profiler's sizes follow the
tensors.  GPU: RotorSequential on a CNN, solved by the library, against
plain autograd, with the measured peak memory of the schedules.
"""
import numpy as np
import pytest
import torch

import paper_1911_13214_b200.executor as E
import paper_1911_13214_b200.strategies as ST


def mlp(width=24, depth=5, dtype=torch.float64, seed=0):
    torch.manual_seed(seed)
    mods = []
    for i in range(depth):
        mods += [torch.nn.Linear(width, width).to(dtype), torch.nn.Tanh() if i % 2 else torch.nn.ReLU()]
    mods.append(torch.nn.LayerNorm(width).to(dtype))
    return torch.nn.Sequential(*mods)


def mse(out, tgt):
    return ((out - tgt) ** 2).mean()


def plain_grads(seq, x, tgt):
    for p in seq.parameters():
        p.grad = None
    xx = x.detach().clone().requires_grad_(x.requires_grad)
    loss = mse(seq(xx), tgt)
    loss.backward()
    return loss.detach(), [p.grad.clone() for p in seq.parameters()], (xx.grad.clone() if x.requires_grad else None)


def run(seq, ops, x, tgt):
    for p in seq.parameters():
        p.grad = None
    xx = x.detach().clone().requires_grad_(x.requires_grad)
    loss = E.execute(list(seq.children()) + [mse], ops, xx, tgt)
    return loss, [p.grad.clone() for p in seq.parameters()], (xx.grad.clone() if x.requires_grad else None)


@pytest.mark.parametrize("input_grad", [False, True])
def test_execute_matches_plain_backward(oracle_mod, input_grad):
    O = oracle_mod
    seq = mlp()
    x = torch.randn(8, 24, dtype=torch.float64)
    tgt = torch.randn(8, 24, dtype=torch.float64)
    x.requires_grad_(input_grad)
    ref = plain_grads(seq, x, tgt)
    stages = list(seq.children()) + [mse]
    ch = E.profile(stages, x.detach(), tgt, repeat=1)
    L = ch.L
    schedules = [ST.pytorch_schedule(L)] + [ST.sequential_schedule(L, k) for k in (2, 3, 5)]
    peak = ST.replay(ST.pytorch_schedule(L), ch).peak
    S = 200
    for f in (0.25, 0.4, 0.6, 1.0):  # DP-optimal schedules (oracle) at several budgets
        o = O.OracleSolve(ch, int(peak * f), S)
        if np.isfinite(o.cost):
            schedules.append(o.reconstruct())
    assert len(schedules) >= 6
    assert any(op == ST.FNULL for s in schedules for op, _ in s) and any(op == ST.FCK for s in schedules for op, _ in s)
    for ops in schedules:
        assert ST.replay(ops, ch).valid
        got = run(seq, ops, x, tgt)
        assert torch.equal(got[0], ref[0])
        assert all(torch.equal(a, b) for a, b in zip(got[1], ref[1]))
        if input_grad:
            assert torch.equal(got[2], ref[2])


def test_profile_sizes():
    seq = mlp(width=16, depth=2, dtype=torch.float32)
    x = torch.randn(4, 16)
    tgt = torch.randn(4, 16)
    stages = list(seq.children()) + [mse]
    ch = E.profile(stages, x, tgt, repeat=1)
    n = ch.L + 1
    assert ch.L == len(list(seq.children()))
    assert list(ch.wx) == [4 * 16 * 4] * (ch.L + 1)  # every activation is 4 x 16 fp32
    assert list(ch.wy[:-1]) == list(ch.wx) and ch.wy[-1] == 4  # delta^l like a^l; scalar loss gradient
    assert len(ch.wbx) == n and all(int(b) >= int(a) for a, b in zip(ch.wx[1:], ch.wbx[:-1]))  # abar includes a
    assert np.all(ch.uf > 0) and np.all(ch.ub > 0)


def test_execute_rejects_missing_inputs():
    seq = mlp(width=8, depth=1)
    x = torch.randn(2, 8, dtype=torch.float64)
    with pytest.raises(KeyError):
        E.execute(list(seq.children()) + [mse], [(ST.FNULL, 1), (ST.FNULL, 1)], x, x)


@pytest.mark.gpu
def test_rotor_sequential_cnn_on_gpu():
    """Profile a CNN on the GPU, solve with the library at limits from 30% of the
    store-all peak up, run one training step with the lowest feasible, a middle and the
    100% schedule: gradients equal plain autograd (same deterministic kernels, up to
    fp32 summation-order noise), and the measured peak of the lowest is well below
    that of the 100% one."""
    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.benchmark = False
    dev = torch.device("cuda")
    torch.manual_seed(0)
    layers = []
    c = 3
    for i, co in enumerate([32, 32, 64, 64, 64, 128, 128]):
        layers += [torch.nn.Conv2d(c, co, 3, padding=1), torch.nn.ReLU()]
        c = co
    layers += [torch.nn.AdaptiveAvgPool2d(4), torch.nn.Flatten(), torch.nn.Linear(c * 16, 10)]
    seq = torch.nn.Sequential(*layers).to(dev)
    ce = lambda out, t: torch.nn.functional.cross_entropy(out, t)
    x = torch.randn(32, 3, 64, 64, device=dev)
    tgt = torch.randint(0, 10, (32,), device=dev)

    for p in seq.parameters():
        p.grad = None
    loss0 = ce(seq(x), tgt)
    loss0.backward()
    ref = [p.grad.clone() for p in seq.parameters()]

    peaks = {}
    base = E.RotorSequential(seq, ce, x, tgt, mem_limit=None)
    feasible = []
    for f in (0.3, 0.4, 0.5, 0.6, 0.75, 0.9):
        try:
            feasible.append((f, E.RotorSequential(seq, ce, x, tgt, mem_limit=int(base.store_all.peak * f),
                                                  chain=base.chain)))
        except ValueError:  # below the chain's minimal memory (o_b of a convolution, ...)
            pass
    assert len(feasible) >= 2, "expected feasible limits below the store-all peak"
    for f, rs in [feasible[0], feasible[len(feasible) // 2], (1.0, base)]:
        assert rs.predicted.peak <= rs.mem_limit
        for p in seq.parameters():
            p.grad = None
        torch.cuda.synchronize()
        m0 = torch.cuda.memory_allocated()
        torch.cuda.reset_peak_memory_stats()
        loss = rs.step(x, tgt)
        torch.cuda.synchronize()
        peaks[f] = torch.cuda.max_memory_allocated() - m0
        assert torch.allclose(loss, loss0.detach(), rtol=0, atol=1e-6)
        for a, b in zip(seq.parameters(), ref):
            assert torch.allclose(a.grad, b, rtol=1e-5, atol=1e-6)
    lo = feasible[0][0]
    assert peaks[lo] < 0.9 * peaks[1.0], peaks
