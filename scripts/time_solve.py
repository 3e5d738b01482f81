"""Wall time of K config-4 solves through the library's host API (quick A/B of
schedules / env switches; bench.py is the measurement of record).
Usage: python scripts/time_solve.py [dag|diagonal] [K]"""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as ge  # noqa: E402

ge.build_library()
import chaingen as G  # noqa: E402
import paper_1911_13214_b200 as R  # noqa: E402

schedule = sys.argv[1] if len(sys.argv) > 1 else "dag"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 5
p = G.config4()
R.solve(p.chain, p.mem_limit, p.slots, schedule=schedule)  # warm-up (workspace, streams)
ts = []
for _ in range(K):
    t0 = time.perf_counter()
    r = R.solve(p.chain, p.mem_limit, p.slots, schedule=schedule)
    ts.append((time.perf_counter() - t0) * 1e3)
print(f"{schedule} {os.environ.get('ROTOR_DIAG_SKIP', '0')} median {statistics.median(ts):.2f} ms  min {min(ts):.2f}  cost {r.cost!r}")
