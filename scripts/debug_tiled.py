"""Run one config through the tiled path (used under compute-sanitizer on the GPU box)."""
import sys
sys.path.insert(0, ".")
import chaingen as G
import paper_1911_13214_b200 as R
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
p = {1: G.config1, 2: G.config2, 3: G.config3}[cfg]()
r = R.solve(p.chain, p.mem_limit, p.slots, kernel="tiled")
print("status", r.status, "cost", r.cost, "n_ops", r.n_ops)
