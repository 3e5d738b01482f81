"""B200-native solver for the optimal persistent checkpointing DP of arXiv 1911.13214.

Thin Python binding over the C ABI of `include/rotor.h` (ctypes, argument
marshalling only).  Every step of the path — discretisation (§5.2),
limits, the Theorem 1 table fill (Algorithm 1
P:809-826) and the Algorithm 2 reconstruction — runs in the
sm_100a kernels of `librotor_b200.so`.  There is no CPU fallback: importing
this package without the built library raises.

A chain is any object with attributes L, uf, ub, wx, wbx, wy, of, ob laid out
as `rotor_chain` in include/rotor.h (e.g. `chaingen.Chain`).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "librotor_b200.so")

FALL, FCK, FNULL, BWD = 0, 1, 2, 3
OK, EINPUT, INFEASIBLE, EINVALID, EDEVICE, ENOMEM, ETRUNC = range(7)
STATUS = {0: "OK", 1: "EINPUT", 2: "INFEASIBLE", 3: "EINVALID", 4: "EDEVICE", 5: "ENOMEM", 6: "ETRUNC"}
KERNELS = {"auto": 0, "wavefront": 1, "tiled": 2}

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback for the solver)"
    )


class rotor_chain(ctypes.Structure):
    _fields_ = [
        ("uf", ctypes.c_void_p), ("ub", ctypes.c_void_p), ("wx", ctypes.c_void_p), ("wbx", ctypes.c_void_p),
        ("wy", ctypes.c_void_p), ("of", ctypes.c_void_p), ("ob", ctypes.c_void_p),
    ]


class rotor_op(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("stage", ctypes.c_int32)]


class rotor_options(ctypes.Structure):
    _fields_ = [
        ("restricted", ctypes.c_int32), ("kernel", ctypes.c_int32), ("keep_argmin", ctypes.c_int32),
        ("profile", ctypes.c_int32), ("counters", ctypes.c_int32), ("schedule", ctypes.c_int32),
        ("reserved", ctypes.c_int32 * 2),
    ]


class rotor_timings(ctypes.Structure):
    _fields_ = [
        ("pre_ms", ctypes.c_double), ("fill_ms", ctypes.c_double), ("reconstruct_ms", ctypes.c_double),
        ("fill_launches", ctypes.c_int32), ("total_launches", ctypes.c_int32),
        ("middle_ms", ctypes.c_double), ("middle_launches", ctypes.c_int32),
    ]


class rotor_counters(ctypes.Structure):
    _fields_ = [
        ("nominal", ctypes.c_double), ("middle_nominal", ctypes.c_double), ("dependent_nominal", ctypes.c_double),
        ("middle_split_visits", ctypes.c_uint64), ("coarse_pass", ctypes.c_uint64),
        ("quadrant_compares", ctypes.c_uint64), ("exact_splits", ctypes.c_uint64), ("evaluated", ctypes.c_double),
        ("middle_wait_cycles", ctypes.c_uint64), ("middle_init_cycles", ctypes.c_uint64),
        ("middle_loop_cycles", ctypes.c_uint64), ("middle_flush_cycles", ctypes.c_uint64),
        ("middle_warp_imbalance", ctypes.c_double), ("middle_slot_cycles", ctypes.c_uint64 * 16),
        ("leaf_ctas", ctypes.c_uint64), ("leaf_setup_ns", ctypes.c_uint64), ("leaf_wait_ns", ctypes.c_uint64),
        ("leaf_work_ns", ctypes.c_uint64), ("leaf_sync_ns", ctypes.c_uint64), ("leaf_pass1_ns", ctypes.c_uint64),
    ]


_lib = ctypes.CDLL(LIB_PATH)
_c = ctypes
_vp, _i32, _i64, _u64, _d = _c.c_void_p, _c.c_int32, _c.c_int64, _c.c_uint64, _c.c_double
_P = _c.POINTER

_lib.rotor_solve.argtypes = [_P(rotor_chain), _i32, _u64, _i32, _P(_d), _vp, _i64, _P(_i64)]
_lib.rotor_solve_ex.argtypes = [_P(rotor_chain), _i32, _u64, _i32, _P(rotor_options), _vp, _u64, _vp, _P(_d), _vp,
                                _i64, _P(_i64)]
_lib.rotor_solve_device.argtypes = [_P(rotor_chain), _i32, _u64, _i32, _P(rotor_options), _vp, _u64, _vp, _vp, _vp,
                                    _i64, _vp, _vp]
_lib.rotor_workspace_bytes.argtypes = [_i32, _i32, _P(rotor_options), _P(_u64)]
_lib.rotor_shadow_layout.argtypes = [_i32, _i32, _P(rotor_options), _P(_i64)]
_lib.rotor_max_ops.argtypes = [_i32]
_lib.rotor_max_ops.restype = _i64
_lib.rotor_solve_batch.argtypes = [_P(rotor_chain), _P(_i32), _i32, _P(_u64), _i32, _i32, _P(rotor_options), _P(_i32),
                                   _i32, _vp, _P(_d), _vp, _P(_i64), _P(_i64), _P(_i64), _P(_i32)]
_lib.rotor_solve_sharded.argtypes = [_P(rotor_chain), _i32, _u64, _i32, _P(rotor_options), _P(_i32), _i32, _i32,
                                     _P(_d), _vp, _i64, _P(_i64)]
_lib.rotor_partition_lpt.argtypes = [_P(_d), _i32, _i32, _P(_i32)]
_lib.rotor_transitions.argtypes = [_i32, _i32]
_lib.rotor_transitions.restype = _d
_lib.rotor_export_tables.argtypes = [_vp, _vp, _i64]
_lib.rotor_last_timings.argtypes = [_P(rotor_timings)]
_lib.rotor_last_counters.argtypes = [_P(rotor_counters)]
_lib.rotor_export_rows.argtypes = [_vp, _vp, _i64, _vp]
_lib.rotor_tile_blocks.argtypes = [_i32]
_lib.rotor_tile_blocks.restype = _i32
_lib.rotor_tile_bytes.argtypes = [_i32, _P(_u64)]
_lib.rotor_sharded_begin.argtypes = [_P(rotor_chain), _i32, _u64, _i32, _P(rotor_options), _vp, _u64, _vp, _P(_vp)]
_lib.rotor_sharded_step.argtypes = [_vp, _i32, _i32, _i32, _vp]
_lib.rotor_sharded_pack.argtypes = [_vp, _i32, _i32, _i32, _vp, _u64, _i32, _vp]
_lib.rotor_sharded_finish.argtypes = [_vp, _vp, _vp, _vp, _i64, _vp, _vp]
_lib.rotor_sharded_free.argtypes = [_vp]
_lib.rotor_sharded_launches.argtypes = [_vp, _P(_i64)]
_lib.rotor_release.argtypes = []
_lib.rotor_last_error.restype = _c.c_char_p
_lib.rotor_version.restype = _i32

# every symbol include/rotor.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "rotor_solve", "rotor_solve_ex", "rotor_solve_device", "rotor_workspace_bytes", "rotor_shadow_layout",
    "rotor_max_ops",
    "rotor_solve_batch", "rotor_solve_sharded", "rotor_partition_lpt", "rotor_transitions", "rotor_export_tables", "rotor_export_rows",
    "rotor_last_timings", "rotor_last_counters",
    "rotor_release", "rotor_last_error", "rotor_version",
    "rotor_tile_blocks", "rotor_tile_bytes", "rotor_sharded_begin", "rotor_sharded_step", "rotor_sharded_pack",
    "rotor_sharded_finish", "rotor_sharded_free", "rotor_sharded_launches",
)


class RotorError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def last_error() -> str:
    return (_lib.rotor_last_error() or b"").decode()


def _check(r: int, allow=(OK,)):
    if r not in allow:
        raise RotorError(r, last_error())
    return r


SCHEDULES = {"dag": 0, "diagonal": 1}


def _options(restricted=False, kernel="auto", keep_argmin=False, profile=False, counters=False,
             schedule="dag") -> rotor_options:
    o = rotor_options()
    o.schedule = SCHEDULES[schedule] if isinstance(schedule, str) else int(schedule)
    o.counters = 1 if counters else 0
    o.restricted = 1 if restricted else 0
    o.kernel = KERNELS[kernel] if isinstance(kernel, str) else int(kernel)
    o.keep_argmin = 1 if keep_argmin else 0
    o.profile = 1 if profile else 0
    return o


def _host_chain(ch):
    """Keep contiguous numpy copies alive and build the rotor_chain view."""
    arrs = dict(
        uf=np.ascontiguousarray(ch.uf, dtype=np.float64), ub=np.ascontiguousarray(ch.ub, dtype=np.float64),
        wx=np.ascontiguousarray(ch.wx, dtype=np.uint64), wbx=np.ascontiguousarray(ch.wbx, dtype=np.uint64),
        wy=np.ascontiguousarray(ch.wy, dtype=np.uint64), of=np.ascontiguousarray(ch.of, dtype=np.uint64),
        ob=np.ascontiguousarray(ch.ob, dtype=np.uint64),
    )
    n = int(ch.L) + 1
    for k, a in arrs.items():
        want = n + 1 if k == "wy" else n
        if a.shape != (want,):
            raise ValueError(f"chain.{k} must have {want} entries, got {a.shape}")
    c = rotor_chain(*(a.ctypes.data for a in (arrs["uf"], arrs["ub"], arrs["wx"], arrs["wbx"], arrs["wy"],
                                               arrs["of"], arrs["ob"])))
    return c, arrs


@dataclass
class Result:
    status: int
    cost: float
    ops: np.ndarray  # (n_ops, 2) int32: opcode, stage
    n_ops: int

    @property
    def feasible(self) -> bool:
        return self.status in (OK, ETRUNC)

    def op_list(self):
        return [(int(a), int(b)) for a, b in self.ops]


def max_ops(L: int) -> int:
    return int(_lib.rotor_max_ops(int(L)))


def transitions(L: int, slots: int) -> float:
    return float(_lib.rotor_transitions(int(L), int(slots)))


def workspace_bytes(L: int, slots: int, **opts) -> int:
    b = _u64()
    o = _options(**opts)
    _check(_lib.rotor_workspace_bytes(int(L), int(slots), _c.byref(o), _c.byref(b)))
    return int(b.value)


def solve(chain, mem_limit: int, slots: int, *, ops_cap: int | None = None, stream=None, workspace=None, **opts) -> Result:
    """rotor_solve_ex: host chain in, cost + Algorithm-2 schedule out (blocking).

    stream: a torch.cuda.Stream / raw cudaStream_t int / None (legacy stream).
    workspace: a device tensor (uint8) of >= workspace_bytes(), or None (library cache).
    """
    c, keep = _host_chain(chain)
    L = int(chain.L)
    cap = max_ops(L) if ops_cap is None else int(ops_cap)
    ops = np.zeros((max(cap, 1), 2), dtype=np.int32)
    cost = _d()
    n_ops = _i64(0)
    o = _options(**opts)
    ws_ptr, ws_bytes = _ws(workspace)
    r = _lib.rotor_solve_ex(_c.byref(c), L, int(mem_limit), int(slots), _c.byref(o), ws_ptr, ws_bytes,
                            _stream_ptr(stream), _c.byref(cost), ops.ctypes.data if cap > 0 else None, cap,
                            _c.byref(n_ops))
    _check(r, allow=(OK, INFEASIBLE, ETRUNC))
    del keep
    k = int(n_ops.value) if r != INFEASIBLE else 0
    return Result(r, float(cost.value), ops[: min(k, cap)].copy(), k)


def _stream_ptr(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)


def _ws(workspace):
    if workspace is None:
        return None, 0
    return int(workspace.data_ptr()), int(workspace.numel() * workspace.element_size())


def shadow_layout(L: int, slots: int, **opts) -> dict:
    """rotor_shadow_layout: byte offsets / row counts of the tiled fill's fp32 shadows in a workspace."""
    arr = (_i64 * 6)()
    o = _options(**opts)
    _check(_lib.rotor_shadow_layout(int(L), int(slots), _c.byref(o), arr))
    return dict(c32_off=arr[0], c32_rows=arr[1], a32_off=arr[2], a32_rows=arr[3], c_off=arr[4], pitch=arr[5])


def solve_device(d_chain: dict, L: int, mem_limit: int, slots: int, workspace, out: dict, stream=None, **opts) -> int:
    """rotor_solve_device: all arguments are CUDA tensors (no host sync).

    d_chain: dict of device tensors uf, ub (float64), wx, wbx, wy, of, ob (int64 holding uint64 bytes).
    out: dict of device tensors cost (float64[1]), ops (int32[cap,2]), n_ops (int64[1]), status (int32[1]).
    """
    c = rotor_chain(*(int(d_chain[k].data_ptr()) for k in ("uf", "ub", "wx", "wbx", "wy", "of", "ob")))
    o = _options(**opts)
    ws_ptr, ws_bytes = _ws(workspace)
    cap = int(out["ops"].shape[0])
    r = _lib.rotor_solve_device(_c.byref(c), int(L), int(mem_limit), int(slots), _c.byref(o), ws_ptr, ws_bytes,
                                _stream_ptr(stream), int(out["cost"].data_ptr()), int(out["ops"].data_ptr()), cap,
                                int(out["n_ops"].data_ptr()), int(out["status"].data_ptr()))
    return _check(r)


def export_tables(n: int, slots: int, C: bool = True, D: bool = True):
    """Tables of the last solve on this thread, canonical layout (cells, S+1)."""
    cells = n * (n + 1) // 2
    Ca = np.empty((cells, slots + 1), dtype=np.float64) if C else None
    Da = np.empty((cells, slots + 1), dtype=np.uint16) if D else None
    _check(_lib.rotor_export_tables(Ca.ctypes.data if C else None, Da.ctypes.data if D else None,
                                    cells * (slots + 1)))
    return Ca, Da


def export_rows(cells, slots: int) -> np.ndarray:
    """C rows of the last solve for the listed (s, t) cells: array (len(cells), S+1)."""
    s = np.ascontiguousarray([c[0] for c in cells], dtype=np.int32)
    t = np.ascontiguousarray([c[1] for c in cells], dtype=np.int32)
    out = np.empty((len(cells), slots + 1), dtype=np.float64)
    _check(_lib.rotor_export_rows(s.ctypes.data, t.ctypes.data, len(cells), out.ctypes.data))
    return out


def last_timings() -> dict:
    t = rotor_timings()
    _check(_lib.rotor_last_timings(_c.byref(t)))
    return dict(pre_ms=t.pre_ms, fill_ms=t.fill_ms, reconstruct_ms=t.reconstruct_ms,
                fill_launches=t.fill_launches, total_launches=t.total_launches,
                middle_ms=t.middle_ms, middle_launches=t.middle_launches)


def last_counters() -> dict:
    """Work counters of the last solve (options counters=True; include/rotor.h rotor_counters)."""
    c = rotor_counters()
    _check(_lib.rotor_last_counters(_c.byref(c)))
    out = {k: getattr(c, k) for k, _ in rotor_counters._fields_}
    out["middle_slot_cycles"] = list(c.middle_slot_cycles)
    return out


def _devices(devices):
    """None -> (NULL, 0): the current device; "all" -> (NULL, -1); a list -> (int32 array, len)."""
    if devices is None:
        return None, 0
    if isinstance(devices, str) and devices == "all":
        return None, -1
    d = np.ascontiguousarray(list(devices), dtype=np.int32)
    return d, len(d)


def solve_batch(chains, limits, slots: int, *, with_ops: bool = False, stream=None, devices=None, **opts):
    """rotor_solve_batch: len(chains) x len(limits[i]) independent solves.

    devices: None (the current device, on `stream`), "all", or a list of CUDA
    ordinals (repeats allowed) the problems are LPT-split over.
    Returns (costs [n_chains, n_limits], status, n_ops, ops list-of-arrays or None).
    """
    nc = len(chains)
    nl = len(limits[0]) if nc else 0
    keep = [_host_chain(ch) for ch in chains]
    arr = (rotor_chain * max(nc, 1))(*[k[0] for k in keep])
    Ls = np.array([int(ch.L) for ch in chains], dtype=np.int32)
    lim = np.ascontiguousarray(np.array(limits, dtype=np.uint64).reshape(nc, nl))
    costs = np.zeros((nc, nl), dtype=np.float64)
    status = np.zeros((nc, nl), dtype=np.int32)
    n_ops = np.zeros((nc, nl), dtype=np.int64)
    o = _options(**opts)
    ops = offs = caps = None
    if with_ops:
        caps = np.repeat(np.array([max_ops(int(ch.L)) for ch in chains], dtype=np.int64), nl)
        offs = np.concatenate([[0], np.cumsum(caps)[:-1]]).astype(np.int64)
        ops = np.empty((int(caps.sum()), 2), dtype=np.int32)
    P = lambda a, t: a.ctypes.data_as(_P(t)) if a is not None else None
    dv, nd = _devices(devices)
    r = _lib.rotor_solve_batch(arr, P(Ls, _i32), nc, P(lim, _u64), nl, int(slots), _c.byref(o), P(dv, _i32), nd,
                               _stream_ptr(stream), P(costs, _d), ops.ctypes.data if ops is not None else None,
                               P(offs, _i64), P(caps, _i64), P(n_ops, _i64), P(status, _i32))
    _check(r)
    return costs, status, n_ops, (BatchOps(ops, offs, n_ops.reshape(-1)) if with_ops else None)


class BatchOps:
    """The schedules of a solve_batch call as a read-only sequence: item p (problem
    chain p // n_limits, limit p % n_limits) is an [n_ops, 2] int32 view into one
    array, made on access (no per-call Python loop over the problems)."""

    def __init__(self, ops, offs, n_ops):
        self._ops, self._offs, self._n = ops, offs, n_ops

    def __len__(self):
        return len(self._n)

    def __getitem__(self, p):
        if isinstance(p, slice):
            return [self[i] for i in range(*p.indices(len(self)))]
        if p < 0:
            p += len(self)
        if not 0 <= p < len(self):
            raise IndexError(p)
        o = int(self._offs[p])
        return self._ops[o: o + max(int(self._n[p]), 0)]

    def __iter__(self):
        return (self[i] for i in range(len(self)))


def solve_sharded(chain, mem_limit: int, slots: int, devices, *, halo_mode: int = 1, ops_cap: int | None = None,
                  **opts) -> Result:
    """rotor_solve_sharded: ONE table sharded over `devices` (list of CUDA ordinals,
    repeats allowed; "all"; or an int k: ordinals 0..k-1) from this process,
    tiles exchanged per tile diagonal by peer pull (halo_mode 1) or pack + peer
    copy (halo_mode 0).  Bit-identical to solve()."""
    c, keep = _host_chain(chain)
    L = int(chain.L)
    if isinstance(devices, int):
        dv, nd = None, int(devices)
    else:
        dv, nd = _devices(devices)
    cap = max_ops(L) if ops_cap is None else int(ops_cap)
    ops = np.zeros((max(cap, 1), 2), dtype=np.int32)
    cost = _d()
    n_ops = _i64(0)
    o = _options(**opts)
    r = _lib.rotor_solve_sharded(_c.byref(c), L, int(mem_limit), int(slots), _c.byref(o),
                                 dv.ctypes.data_as(_P(_i32)) if dv is not None else None, nd, int(halo_mode),
                                 _c.byref(cost), ops.ctypes.data if cap > 0 else None, cap, _c.byref(n_ops))
    _check(r, allow=(OK, INFEASIBLE, ETRUNC))
    del keep
    k = int(n_ops.value) if r != INFEASIBLE else 0
    return Result(r, float(cost.value), ops[: min(k, cap)].copy(), k)


def partition_lpt(weights, n_parts: int) -> np.ndarray:
    w = np.ascontiguousarray(weights, dtype=np.float64)
    out = np.zeros(len(w), dtype=np.int32)
    _check(_lib.rotor_partition_lpt(w.ctypes.data_as(_P(_d)), len(w), int(n_parts), out.ctypes.data_as(_P(_i32))))
    return out


def tile_blocks(L: int) -> int:
    """Number of 32-stage blocks of the tiled fill: tile diagonals are 0 .. tile_blocks(L)-1."""
    return int(_lib.rotor_tile_blocks(int(L)))


def tile_bytes(slots: int) -> int:
    b = _u64()
    _check(_lib.rotor_tile_bytes(int(slots), _c.byref(b)))
    return int(b.value)


class Shard:
    """One rank's sharded single-table solve (rotor_sharded_* of include/rotor.h).

    d_chain: dict of device tensors as for solve_device; workspace: device uint8
    tensor of >= workspace_bytes(L, slots, kernel="tiled").
    """

    def __init__(self, d_chain: dict, L: int, mem_limit: int, slots: int, workspace, stream=None, **opts):
        self.L, self.S = int(L), int(slots)
        self._keep = (d_chain, workspace)
        c = rotor_chain(*(int(d_chain[k].data_ptr()) for k in ("uf", "ub", "wx", "wbx", "wy", "of", "ob")))
        o = _options(**opts)
        ws_ptr, ws_bytes = _ws(workspace)
        h = _vp()
        _check(_lib.rotor_sharded_begin(_c.byref(c), self.L, int(mem_limit), self.S, _c.byref(o), ws_ptr, ws_bytes,
                                        _stream_ptr(stream), _c.byref(h)))
        self.h = h.value

    def step(self, delta: int, lo: int, hi: int, stream=None):
        _check(_lib.rotor_sharded_step(self.h, int(delta), int(lo), int(hi), _stream_ptr(stream)))

    def pack(self, delta: int, lo: int, hi: int, buf, unpack: bool = False, stream=None):
        nbytes = int(buf.numel() * buf.element_size())
        _check(_lib.rotor_sharded_pack(self.h, int(delta), int(lo), int(hi), int(buf.data_ptr()), nbytes,
                                       1 if unpack else 0, _stream_ptr(stream)))

    def finish(self, out: dict, stream=None):
        cap = int(out["ops"].shape[0])
        _check(_lib.rotor_sharded_finish(self.h, _stream_ptr(stream), int(out["cost"].data_ptr()),
                                         int(out["ops"].data_ptr()), cap, int(out["n_ops"].data_ptr()),
                                         int(out["status"].data_ptr())))

    def launches(self) -> int:
        n = _i64()
        _check(_lib.rotor_sharded_launches(self.h, _c.byref(n)))
        return int(n.value)

    def close(self):
        if getattr(self, "h", None):
            _lib.rotor_sharded_free(self.h)
            self.h = None

    def __del__(self):
        self.close()


def release():
    _lib.rotor_release()


def version() -> int:
    return int(_lib.rotor_version())
