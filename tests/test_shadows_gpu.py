"""The invariants the pruned middle's filter relies on (DESIGN.md §5.0/§5.2),
checked on the GPU's own workspace after a tiled solve, against the fp64
table by their definitions:

* C32(s, t) holds rd32(C(s, t, m - wx[s-1])) at column m (+inf for m < wx[s-1]),
  A32(s, c) holds rd32(A(s, c, m)), A = fl(fl(P[c] - P[s-1]) + C(s, c, m));
* every quad minimum the middle reads is the min of its 4 cells' shadows
  (existing cells only; +inf if none).  (The minima of a column group whose
  whole 8-column sub-tile lies past the last stage are never written: every
  cell a lane reading them holds is past the last stage, bound -inf, so they
  never decide anything.)

A quad minimum above its cells would let the middle skip a candidate that is
the minimum — a wrong table that a parity test catches only when it changes
a value; this checks the lower-bound property itself.  The row layout is
re-derived here from DESIGN.md §5.0 (block-major, 40 rows per block column /
row: 32 cells, then 8 quad minima)."""
import numpy as np
import pytest
import torch

import chaingen as G

TB, SR, QUAD = 32, 40, 32


def _rd32(x):
    f = x.astype(np.float32)
    down = f.astype(np.float64) > x
    f[down] = np.nextafter(f[down], np.float32(-np.inf))
    return f


def _slots(x, S, M):
    return min(S + 1, -(-int(x) * S // M))


def _check(p):
    import paper_1911_13214_b200 as R

    ch, S, M = p.chain, p.slots, p.mem_limit
    L, n = ch.L, ch.L + 1
    dev = torch.device("cuda")
    d_chain = {k: torch.from_numpy(np.asarray(getattr(ch, k)).astype(np.float64 if k in ("uf", "ub") else np.int64)).to(dev)
               for k in ("uf", "ub", "wx", "wbx", "wy", "of", "ob")}
    ws = torch.zeros(R.workspace_bytes(L, S, kernel="tiled"), dtype=torch.uint8, device=dev)
    cap = R.max_ops(L)
    out = dict(cost=torch.empty(1, dtype=torch.float64, device=dev), ops=torch.empty((cap, 2), dtype=torch.int32, device=dev),
               n_ops=torch.empty(1, dtype=torch.int64, device=dev), status=torch.empty(1, dtype=torch.int32, device=dev))
    R.solve_device(d_chain, L, M, S, ws, out, kernel="tiled")
    torch.cuda.synchronize()
    lay = R.shadow_layout(L, S, kernel="tiled")
    w = ws.cpu().numpy()
    pitch = lay["pitch"]
    cells = n * (n + 1) // 2

    def cell(s, t):
        r = s - 1
        return r * n - r * (r - 1) // 2 + (t - s)

    Cw = w[lay["c_off"] - 16 * 8: lay["c_off"] - 16 * 8 + cells * pitch * 8].view(np.float64).reshape(cells, pitch)[:, 16:16 + S + 1]
    C32 = w[lay["c32_off"]: lay["c32_off"] + lay["c32_rows"] * pitch * 4].view(np.float32)
    A32 = w[lay["a32_off"]: lay["a32_off"] + lay["a32_rows"] * pitch * 4].view(np.float32)
    ms = np.arange(S + 1)

    def sh(arr, rows, row):  # the shadow row's columns 0..S (m-chunked layout)
        return arr[((ms >> 5) * rows + row) * 32 + (ms & 31)]

    # layout
    def sc_row(J, s):
        return SR * (TB * J * (J + 1) // 2 + (s - 1))

    def srow_c(s, t):
        J = (t - 1) // TB
        return sc_row(J, s) + (t - 1 - TB * J)

    def sa_col(I, c):
        return SR * (I * n - TB * I * (I - 1) // 2 + (c - (TB * I + 1)))

    def srow_a(s, c):
        I = (s - 1) // TB
        return sa_col(I, c) + (s - 1 - TB * I)

    wx = [_slots(x, S, M) for x in ch.wx]
    P = np.concatenate([[0.0], np.cumsum(np.asarray(ch.uf, dtype=np.float64))])
    nb = (n + TB - 1) // TB
    # cell shadows
    for s in range(1, n + 1):
        ws_ = wx[s - 1]
        for t in range(s, n + 1):
            c = Cw[cell(s, t)]
            exp = np.full(S + 1, np.inf, dtype=np.float32)
            if ws_ <= S:
                exp[ws_:] = _rd32(c[: S + 1 - ws_])
            got = sh(C32, lay["c32_rows"], srow_c(s, t))
            assert np.array_equal(got.view(np.uint32), exp.view(np.uint32)), ("C32", s, t)
            if t < n:
                a = (P[t] - P[s - 1]) + c
                got = sh(A32, lay["a32_rows"], srow_a(s, t))
                assert np.array_equal(got.view(np.uint32), _rd32(a).view(np.uint32)), ("A32", s, t)
    # quad minima the middle reads: C32 rows s of blocks K < J, A32 columns of blocks J > I and c = i0 + 31
    for J in range(1, nb):
        for s in range(1, TB * J + 1):
            for g in range(8):
                if TB * J + 1 + 8 * (g // 2) > n:
                    continue  # its 8-column sub-tile has no cell: no leaf writes it, no middle lane reads it
                ts = [t for t in range(TB * J + 1 + 4 * g, TB * J + 5 + 4 * g) if t <= n]
                exp = np.full(S + 1, np.inf, dtype=np.float32)
                for t in ts:
                    exp = np.minimum(exp, sh(C32, lay["c32_rows"], srow_c(s, t)))
                got = sh(C32, lay["c32_rows"], sc_row(J, s) + QUAD + g)
                assert np.array_equal(got.view(np.uint32), exp.view(np.uint32)), ("QC", J, s, g)
    for I in range(nb):
        i0 = TB * I + 1
        if i0 + TB - 1 > n:
            continue  # a partial last block is never a middle's row block
        cols = [i0 + TB - 1] + list(range(i0 + TB, n))
        for c in cols:
            for g in range(8):
                exp = np.full(S + 1, np.inf, dtype=np.float32)
                for s in range(i0 + 4 * g, i0 + 4 * g + 4):
                    exp = np.minimum(exp, sh(A32, lay["a32_rows"], srow_a(s, c)))
                got = sh(A32, lay["a32_rows"], sa_col(I, c) + QUAD + g)
                assert np.array_equal(got.view(np.uint32), exp.view(np.uint32)), ("QA", I, c, g)


@pytest.mark.gpu
@pytest.mark.parametrize("which", ["cfg2", "random130"])
def test_shadows_and_quad_minima_gpu(which):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge

    ge.build_library()
    if which == "cfg2":
        p = G.config2()
    else:  # n = 131: a partial last tile block, large shifts
        rng = G.SplitMix64(77)
        ch = G.random_chain(rng, 130, real_times=True, big=True)
        p = G.Problem(ch, mem_limit=int(sum(int(x) for x in ch.wbx) * 0.25), slots=300, name="random130")
    _check(p)
