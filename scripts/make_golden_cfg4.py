"""Write tests/golden/cfg4_L1000_S4000.txt from the ORACLE's full config-4 fill.

Config 4 of BASELINE.json (long heterogeneous chain, L=1000, S=4000, M = 0.25
budget_ref) is the headline workload.  Its whole table —
Theorem 1 filled by Algorithm 1 (Q3 order), 501,501
rows of 4,001 fp64 values — is computed here by the plain C oracle (OpenMP
over the cells of each diagonal, bit-identical to the single-thread fill, see
tests/test_oracle_pins.py), once, and recorded as:

  cost          the fp64 bits of C[1, L+1, S - slots(a^0)] (Alg. 1 return)
  list:top      the whole top row C[1, L+1, m], m = 0..S (fp64 bits)
  list:H / G    per-s and per-d checksums of every row (tests/table_hash.py)
  list:ops      Algorithm 2's schedule from the top cell (Q4/Q11),
                each op as (opcode << 32 | stage)

This script calls only `oracle/`, `chaingen/` (inputs) and the test-side
checksum module; it never touches the CUDA product.
Usage: python scripts/make_golden_cfg4.py [threads]   (~10 min on 8 cores, 16 GB RAM)
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import chaingen as G  # noqa: E402
import oracle as O  # noqa: E402
import table_hash as TH  # noqa: E402


def main():
    threads = int(sys.argv[1]) if len(sys.argv) > 1 else O.max_threads()
    p = G.config4()
    ch = p.chain
    n = ch.L + 1
    t0 = time.time()
    o = O.OracleSolve(ch, p.mem_limit, p.slots, threads=threads, keep_d=False)
    t_fill = time.time() - t0
    C = o.table_view()
    hs = TH.hash_canonical_table(C, n)
    assert hs.complete()
    top = C[TH.cell_index(n, 1, n)].copy()
    cost = o.cost
    ops = o.reconstruct()
    t_all = time.time() - t0
    out = os.path.join(ROOT, "tests", "golden", "cfg4_L1000_S4000.txt")
    with open(out, "w") as f:
        f.write("# Config 4 (BASELINE.json configs[3]): chaingen.config4(), L=1000, S=4000, M=0.25*budget_ref.\n")
        f.write("# Written by scripts/make_golden_cfg4.py from the oracle only (oracle/rotor_oracle.c,\n")
        f.write(f"# OpenMP fill with {threads} threads: {t_fill:.0f} s fill, {t_all:.0f} s total).\n")
        f.write("# Theorem 1 P:717-739 / Algorithm 1 P:809-826 (fill), P:824 (top query), Algorithm 2 P:829-847.\n")
        f.write("# Checksums: tests/table_hash.py (row hash over fp64 bits, combined per s and per d).\n")
        f.write(f"L {ch.L}\nS {p.slots}\nM {p.mem_limit}\nm_top {o.m_top}\n")
        f.write(f"cost {np.float64(cost).view(np.uint64):016x}\n")
        f.write(f"cost_float {cost!r}\n")
        f.write(f"n_ops {len(ops)}\n")
        TH.write_hex(f, "top", top.view(np.uint64))
        TH.write_hex(f, "H", hs.H[1:])
        TH.write_hex(f, "G", hs.G)
        TH.write_hex(f, "ops", [(a << 32) | b for a, b in ops])
    print(f"wrote {out}: cost={cost!r} ops={len(ops)} fill {t_fill:.0f}s total {t_all:.0f}s")


if __name__ == "__main__":
    main()
