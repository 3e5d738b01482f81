"""Host-side pieces of bench.py (no GPU): the reference arm's JSON line and the
algorithmic-bytes model of the wavefront roofline."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_transitions_formula():
    # nominal transitions: every cell of diagonal d has d F_ck candidates + 1 F_all candidate
    L, S = 7, 11
    n = L + 1
    brute = sum((d + 1) * (S + 1) for d in range(1, L + 1) for s in range(1, n - d + 1))
    assert bench.n_transitions(L, S) == brute


def test_middle_transitions_bruteforce():
    """The middle kernel's candidates: every split s' of a cell (s,t) that lies in a
    32-stage block strictly between the blocks of s and t (enumerated cell by cell),
    at every m; a subset of the nominal transitions."""
    TB = 32
    for L, S in ((70, 3), (96, 5), (130, 2)):
        n = L + 1
        brute = 0
        for s in range(1, n + 1):
            for t in range(s + 1, n + 1):
                bs, bt = (s - 1) // TB, (t - 1) // TB
                brute += sum(1 for sp in range(s + 1, t + 1) if bs < (sp - 1) // TB < bt)
        assert bench.middle_transitions(L, S, TB) == brute * (S + 1)
        assert bench.middle_transitions(L, S, TB) < bench.n_transitions(L, S)


def test_middle_alg_bytes_bruteforce():
    """fp32 operand reads (one per real row / column, split and m) and their quad
    minima (one per group of 4 real rows / columns), enumerated tile by tile."""
    TB = 32
    for L, S in ((70, 3), (130, 2)):
        n = L + 1
        nb = (n + TB - 1) // TB
        brute = 0
        for I in range(nb):
            rows = [s for s in range(TB * I + 1, TB * I + TB + 1) if s <= n]
            for J in range(I + 2, nb):
                cols = [t for t in range(TB * J + 1, TB * J + TB + 1) if t <= n]
                splits = range(TB * (I + 1) + 1, TB * J + 1)
                groups = len({(s - 1) // 4 for s in rows}) + len({(t - 1) // 4 for t in cols})
                brute += sum(4 * len(rows) + 4 * len(cols) + 4 * groups for _ in splits)
        assert bench.middle_alg_bytes(L, S, TB) == brute * (S + 1)


def test_alg_bytes_wavefront_bruteforce():
    """Distinct rows read per diagonal, by enumerating the cells each candidate touches."""
    L, S = 9, 3
    n = L + 1
    rows = 0
    for d in range(1, L + 1):
        touched = set()
        for s in range(1, n - d + 1):
            t = s + d
            for k in range(1, d + 1):
                touched.add((s, s + k - 1))  # prefix row C[s, s'-1]
                touched.add((s + k, t))  # suffix row C[s', t]
            touched.add((s + 1, t))  # F_all row (also a suffix row)
        rows += len(touched)
    cells = n * (n + 1) // 2
    assert bench.alg_bytes_wavefront(L, S) == 8.0 * (S + 1) * (rows + cells)


def test_reference_arm_json_line():
    env = dict(os.environ, ROTOR_REF_WINDOW="30")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, env=env, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "cpu_baseline",
              "e2e", "config"):
        assert k in line
    assert line["value"] > 0 and line["cpu_baseline"]["kind"] == "oracle"
    assert line["e2e"]["h2d_bytes_per_step"] == 0
