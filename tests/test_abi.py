"""C-ABI library checks that need no GPU (`-m "not gpu"`).

The library must load, export every symbol include/rotor.h declares, and
reject bad arguments before touching the device.  No compute call is made.
"""
import ctypes
import os
import re

import numpy as np
import pytest

import chaingen as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def R():
    import __graft_entry__ as ge

    ge.build_library()
    import paper_1911_13214_b200 as R

    return R


def _declared_symbols():
    txt = open(os.path.join(ROOT, "include", "rotor.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(rotor_[a-z_]+)\s*\(", txt)))


def test_header_declares_core_entry_points():
    syms = _declared_symbols()
    for s in ("rotor_solve", "rotor_solve_batch", "rotor_solve_device", "rotor_export_tables"):
        assert s in syms


def test_library_exports_every_declared_symbol(R):
    lib = ctypes.CDLL(R.LIB_PATH)
    syms = _declared_symbols()
    assert syms
    for s in syms:
        assert hasattr(lib, s), f"missing export {s}"
    assert sorted(R.EXPORTS) == syms


def test_sm100a_code_in_library(R):
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", R.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_host_side_helpers(R):
    # nominal transitions: sum_{d=1}^{L} (n-d)(d+1)(S+1)
    assert R.transitions(10, 50) == 14025
    assert R.transitions(1000, 4000) == pytest.approx(6.708e11, rel=1e-3)
    assert R.max_ops(10) == 11 * 12 // 2 + 11
    ws = R.workspace_bytes(1000, 4000)
    assert ws >= 501501 * 4001 * 8  # the C table alone
    wf = R.workspace_bytes(1000, 4000, kernel="wavefront")
    assert ws > wf  # the tiled fill also stores A = U + C
    assert R.workspace_bytes(1000, 4000, kernel="wavefront", keep_argmin=True) > wf


def test_argument_errors_without_device(R):
    ch = G.unit_chain(3)
    for bad in [dict(mem_limit=0, slots=10), dict(mem_limit=10, slots=0)]:
        with pytest.raises(R.RotorError) as e:
            R.solve(ch, **bad)
        assert e.value.status == R.EINPUT
    bad = G.unit_chain(3)
    bad.uf[2] = float("nan")
    with pytest.raises(R.RotorError) as e:
        R.solve(bad, 10, 10)
    assert e.value.status == R.EINPUT
    bad.uf[2] = -1.0
    with pytest.raises(R.RotorError):
        R.solve(bad, 10, 10)
    with pytest.raises(ValueError):
        ch2 = G.unit_chain(3)
        ch2.L = 4
        R.solve(ch2, 10, 10)


def test_partition_lpt(R):
    w = np.array([5.0, 4, 3, 3, 2, 2, 1], dtype=np.float64)
    part = R.partition_lpt(w, 3)
    loads = np.bincount(part, weights=w, minlength=3)
    assert loads.max() - loads.min() <= 1.0
    assert np.array_equal(R.partition_lpt(w, 3), part)  # deterministic
    # LPT bound: makespan <= 4/3 OPT
    rng = G.SplitMix64(3)
    for _ in range(50):
        w = np.array([rng.uniform() * 100 for _ in range(40)])
        k = 1 + rng.randint(0, 7)
        part = R.partition_lpt(w, k)
        assert set(part) <= set(range(k))
        loads = np.bincount(part, weights=w, minlength=k)
        assert loads.max() <= (4.0 / 3.0) * max(w.sum() / k, w.max()) + 1e-9
