"""Write tests/golden/cfg1_unit_L10.txt from the ORACLE's exhaustive search only.

The fixture pins the DP on config 1 (unit chain L=10, u_f=u_b=1, every size 1
slot, overheads 0): for each budget m (slots, a^0 not
counted, Theorem 1) the optimal persistent makespan found by
Dijkstra over Table-1 memory states (oracle.brute_force, §4.1 persistency),
and the restricted ("revolve") optimum from the Griewank-Walther
binomial formula (see tests/test_oracle_pins.py for the
mapping C_restricted[1,l,c+2] = l*u_f + t(l,c) + l*u_b).

This script calls only `oracle/` and `chaingen/`; it never touches the CUDA
product.  Usage: python scripts/make_golden.py [max_m]
"""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import chaingen as G  # noqa: E402
import oracle as O  # noqa: E402


def main():
    max_m = int(sys.argv[1]) if len(sys.argv) > 1 else 12
    p = G.config1()
    o = O.OracleSolve(p.chain, p.mem_limit, p.slots, fill=False)  # only for the discretised sizes
    sz = o.sizes()
    n = sz.n
    rows = []
    for m in range(0, max_m + 1):
        t0 = time.time()
        c, ops = O.brute_force(sz, m + sz.wx[0], max_states=200_000_000)
        # restricted optimum from the closed form: c = m - 2 extra checkpoints (see tests)
        cres = math.inf if m < 3 else n * 1.0 + O.griewank_t(n, m - 2) + n * 1.0
        rows.append((m, c, cres))
        print(f"m={m} brute={c} restricted_closed_form={cres} ({time.time() - t0:.1f}s)", flush=True)
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                       "cfg1_unit_L10.txt")
    with open(out, "w") as f:
        f.write("# config 1: unit chain L=10 (n=11 stages), u_f=u_b=1, wx=wbx=wy=1, of=ob=0, M=S=50\n")
        f.write("# m = DP budget in slots (a^0 not counted, P:698-700); top cell C[1,11,m]\n")
        f.write("# persistent = exhaustive Dijkstra over Table-1 memory states (oracle.brute_force)\n")
        f.write("# restricted = revolve optimum n*u_f + t(n, m-2) + n*u_b (Griewank-Walther, P:45-47)\n")
        f.write("# written by scripts/make_golden.py (calls oracle/ only)\n")
        f.write("m persistent restricted\n")
        for m, c, cr in rows:
            f.write(f"{m} {c} {cr}\n")
    print("wrote", out)


if __name__ == "__main__":
    main()
