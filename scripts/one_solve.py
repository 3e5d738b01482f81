"""One config-4 solve through the library (for ncu launch lists: exactly one
solve's launches).  Usage: python scripts/one_solve.py [dag|diagonal] [config]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as ge  # noqa: E402

ge.build_library()
import chaingen as G  # noqa: E402
import paper_1911_13214_b200 as R  # noqa: E402

schedule = sys.argv[1] if len(sys.argv) > 1 else "dag"
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 4
p = {4: G.config4, 3: G.config3, 2: G.config2}[cfg]()
r = R.solve(p.chain, p.mem_limit, p.slots, schedule=schedule)
print(schedule, p.name, r.status, r.cost, r.n_ops)
