"""The nn.Sequential tool end to end on the GPU (§4): profile a CNN,
solve at several memory limits, run training steps with each schedule and
compare the measured peak memory / step time with the model's prediction
(replay of the schedule on the profiled chain), next to store-all and
checkpoint_sequential.  Random weights, synthetic batch.

  python scripts/executor_demo.py [--batch 64] [--size 128]
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1911_13214_b200.executor as E  # noqa: E402
import paper_1911_13214_b200.strategies as ST  # noqa: E402


def cnn(dev):
    torch.manual_seed(0)
    layers, c = [], 3
    for co in [64, 64, 128, 128, 128, 256, 256, 256, 256, 512, 512]:
        layers += [torch.nn.Conv2d(c, co, 3, padding=1), torch.nn.BatchNorm2d(co), torch.nn.ReLU()]
        c = co
    layers += [torch.nn.AdaptiveAvgPool2d(2), torch.nn.Flatten(), torch.nn.Linear(c * 4, 100)]
    return torch.nn.Sequential(*layers).to(dev)


def measure(stages, ops, x, tgt, params, iters=5):
    times, peak = [], 0
    for i in range(iters + 1):
        for p in params:
            p.grad = None
        torch.cuda.synchronize()
        m0 = torch.cuda.memory_allocated()
        torch.cuda.reset_peak_memory_stats()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        E.execute(stages, ops, x, tgt)
        e1.record()
        e1.synchronize()
        if i:
            times.append(e0.elapsed_time(e1) / 1e3)
            peak = max(peak, torch.cuda.max_memory_allocated() - m0)
    return peak, statistics.median(times)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--size", type=int, default=128)
    args = ap.parse_args()
    dev = torch.device("cuda")
    seq = cnn(dev)
    params = list(seq.parameters())
    ce = lambda out, t: torch.nn.functional.cross_entropy(out, t)
    x = torch.randn(args.batch, 3, args.size, args.size, device=dev)
    tgt = torch.randint(0, 100, (args.batch,), device=dev)
    stages = list(seq.children()) + [ce]
    ch = E.profile(stages, x, tgt)
    L = ch.L
    sa = ST.replay(ST.pytorch_schedule(L), ch)
    rows = []
    pk, tm = measure(stages, ST.pytorch_schedule(L), x, tgt, params)
    rows.append(("pytorch (store all)", sa.peak, sa.time, pk, tm))
    for k in ST.sequential_segment_counts(L)[::3]:
        ops = ST.sequential_schedule(L, k)
        pr = ST.replay(ops, ch)
        pk, tm = measure(stages, ops, x, tgt, params)
        rows.append((f"sequential {k} segments", pr.peak, pr.time, pk, tm))
    for f in (0.2, 0.3, 0.4, 0.6, 0.8, 1.0):
        try:
            rs = E.RotorSequential(seq, ce, x, tgt, mem_limit=int(sa.peak * f), chain=ch)
        except ValueError:
            rows.append((f"optimal M = {f:.1f} x store-all", None, None, None, None))
            continue
        pk, tm = measure(stages, rs.ops, x, tgt, params)
        rows.append((f"optimal M = {f:.1f} x store-all", rs.predicted.peak, rs.predicted.time, pk, tm))
    print(f"CNN: {L} stages + loss, batch {args.batch} x 3 x {args.size}^2, fp32; profiled store-all peak "
          f"{sa.peak / 2**20:.0f} MiB, model step {sa.time * 1e3:.2f} ms\n")
    print("| schedule | predicted peak MiB | measured peak MiB | predicted step ms | measured step ms |")
    print("|---|---|---|---|---|")
    for name, pp, pt, mp, mt in rows:
        if pp is None:
            print(f"| {name} | infeasible | | | |")
            continue
        print(f"| {name} | {pp / 2**20:.0f} | {mp / 2**20:.0f} | {pt * 1e3:.2f} | {mt * 1e3:.2f} |")


if __name__ == "__main__":
    main()
