"""The §5.2 strategy comparison on the synthetic chains: pytorch
(store all), sequential (2..2·sqrt(L) segments), revolve and optimal (GPU DP
at 10 limits between 0 and the pytorch peak), every schedule replayed under
Table 1.  Prints a markdown table per chain (time per iteration, throughput
relative to pytorch, peak memory relative to pytorch) and the Pareto envelope.

  python scripts/compare_strategies.py [--slots 500] [--json out.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import chaingen as G  # noqa: E402
import paper_1911_13214_b200.strategies as ST  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--slots", type=int, default=500)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    chains, _, _ = G.config5(n_limits=1)
    todo = [("cfg2 ResNet-101-shaped L=100", G.config2().chain), ("cfg3 DenseNet-shaped L=300", G.config3().chain)]
    todo += [(f"cfg5 chain {i} (L={c.L})", c) for i, c in enumerate(chains)]
    out = []
    for name, ch in todo:
        t0 = time.perf_counter()
        pts = ST.compare(ch, slots=args.slots)
        dt = time.perf_counter() - t0
        base = next(p for p in pts if p.strategy == "pytorch")
        print(f"\n### {name}  (sweep {dt:.2f} s incl. 20 GPU solves)\n")
        print("| strategy | param | peak / pytorch | time / pytorch | throughput / pytorch |")
        print("|---|---|---|---|---|")
        for p in pts:
            par = f"{int(p.param)} seg" if p.strategy == "sequential" else (
                f"M = {p.param / base.peak:.1f} x" if p.strategy in ("optimal", "revolve") else "-")
            if not p.feasible:
                print(f"| {p.strategy} | {par} | - | infeasible | 0 |")
                continue
            print(f"| {p.strategy} | {par} | {p.peak / base.peak:.3f} | {p.time / base.time:.4f} | "
                  f"{base.time / p.time:.4f} |")
        env = ST.pareto(pts)
        print("\nPareto envelope (peak / pytorch -> throughput / pytorch, strategy): " + ", ".join(
            f"{p.peak / base.peak:.2f} -> {base.time / p.time:.3f} {p.strategy}" for p in env))
        out.append({"chain": name, "points": [p.__dict__ for p in pts], "sweep_s": dt})
    if args.json:
        with open(args.json, "w") as f:
            json.dump(out, f, indent=1, default=float)


if __name__ == "__main__":
    main()
