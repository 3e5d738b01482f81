/*
 * rotor.h — C ABI of the B200 (sm_100a) solver for the optimal persistent
 * checkpointing DP of arXiv 1911.13214 ("Rotor").
 *
 * The library computes, on the GPU, the table C(s,t,m) of Theorem 1
 * (PAPER.md P:717-739): the optimal time to process stages s..t of a chain
 * within m memory slots, assuming a^{s-1} and delta^t are stored and a^{s-1}
 * is not counted in m.  It then reconstructs the optimal operation
 * sequence with Algorithm 2.  Sizes are discretised into S slots
 * of M/S bytes, each rounded up (§5.2).  The readings of the paper
 * it implements (fill order, tie rule, fp64 association, …) are listed in
 * DESIGN.md §3; they are part of this contract.
 *
 * Conventions for every entry point
 *   - Plain C types only; no exception or C++ type crosses the boundary.
 *   - All output buffers are caller-owned.  Input buffers are read-only and
 *     only read during the call (or, for the *_device variants, until the
 *     work enqueued on `stream` completes).
 *   - A `stream` argument is a cudaStream_t passed as void*; NULL means the
 *     legacy default stream.  Device pointers must belong to the current
 *     device of the calling thread.
 *   - Every function returns a rotor_status.  On error, rotor_last_error()
 *     returns a thread-local message.  Calls are thread-compatible, not
 *     re-entrant on the same workspace.
 */
#ifndef ROTOR_H
#define ROTOR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------------------
 * The chain (§3.1; Table 1).
 * n = L+1 stages; stage L+1 is the loss.  Arrays are 0-based
 * storage of the paper's 1-based indices:
 *   uf[l-1], ub[l-1]  time of F^l / B^l, l = 1..L+1        (finite, >= 0)
 *   wx[l]             size of a^l, l = 0..L                 (bytes)
 *   wbx[l-1]          size of abar^l, l = 1..L+1            (bytes)
 *   wy[l]             size of delta^l, l = 0..L+1 (L+2 values)
 *   of[l-1], ob[l-1]  memory overhead of F^l / B^l           (bytes)
 * Host pointers for rotor_solve / rotor_solve_ex / rotor_solve_batch; device
 * pointers for rotor_solve_device.
 * ------------------------------------------------------------------------- */
typedef struct {
    const double *uf, *ub;
    const uint64_t *wx;
    const uint64_t *wbx;
    const uint64_t *wy;
    const uint64_t *of, *ob;
} rotor_chain;

/* Schedule operations (Table 1): F_all, F_ck, F_null, B. */
typedef enum { ROTOR_FALL = 0, ROTOR_FCK = 1, ROTOR_FNULL = 2, ROTOR_BWD = 3 } rotor_opcode;
typedef struct {
    int32_t op;    /* rotor_opcode */
    int32_t stage; /* 1..L+1 */
} rotor_op;

typedef enum {
    ROTOR_OK = 0,
    ROTOR_EINPUT = 1,      /* bad argument: L < 1, S < 1, M = 0, NaN/negative time, NULL array */
    ROTOR_INFEASIBLE = 2,  /* no valid persistent schedule within M: cost = +inf, n_ops = 0 */
    ROTOR_EINVALID = 3,    /* internal consistency failure (reconstruction could not follow C) */
    ROTOR_EDEVICE = 4,     /* CUDA error (message in rotor_last_error) */
    ROTOR_ENOMEM = 5,      /* workspace too small / device allocation failed */
    ROTOR_ETRUNC = 6       /* cost valid; ops truncated to ops_cap (n_ops holds the full count) */
} rotor_status;

/* Fill kernels. */
typedef enum {
    ROTOR_KERNEL_AUTO = 0,
    ROTOR_KERNEL_WAVEFRONT = 1, /* one launch per diagonal d, one thread per (s,m) cell, k-loop */
    ROTOR_KERNEL_TILED = 2      /* blocked (s,t)-tile min-plus evaluation (fast path) */
} rotor_kernel;

typedef struct {
    int32_t restricted;  /* 1: F_all only at s = t — the paper's "revolve" baseline */
    int32_t kernel;      /* rotor_kernel */
    int32_t keep_argmin; /* 1: record D (uint16 argmin) during the fill (wavefront kernel only) */
    int32_t profile;     /* 1: time the phases with CUDA events (see rotor_last_timings) */
    int32_t counters;    /* 1: count the pruned middle kernel's work (see rotor_last_counters) */
    int32_t schedule;    /* tiled fill: 0 = tile DAG over several streams (default),
                            1 = diagonal by diagonal on the caller's stream (middle launches timed) */
    int32_t reserved[2];
} rotor_options;

/* Default options: all zero (unrestricted, auto kernel, no D, no profiling). */

/* ---------------------------------------------------------------------------
 * rotor_solve — Algorithm 1 + Algorithm 2 for one chain and one memory limit.
 *   chain, L   : host chain (above), L >= 1
 *   mem_limit  : M in bytes (> 0); slots: S >= 1 (the paper uses 500)
 *   cost_out   : C[1, L+1, S - slots(wx[0])] (Alg. 1 return); +inf when infeasible
 *   ops        : caller buffer of ops_cap entries, or NULL for a size query
 *   n_ops_out  : number of ops of the optimal sequence (written even when truncated)
 * Uses a library-owned, per-device cached workspace and the legacy stream;
 * blocks until the result is on the host.
 * Returns ROTOR_OK, ROTOR_INFEASIBLE, ROTOR_ETRUNC or an error.
 * ------------------------------------------------------------------------- */
int rotor_solve(const rotor_chain *chain, int32_t L, uint64_t mem_limit, int32_t slots, double *cost_out,
                rotor_op *ops, int64_t ops_cap, int64_t *n_ops_out);

/* rotor_solve with options, an explicit stream and optionally a caller-owned
 * device workspace (e.g. torch-allocated) of workspace_bytes >=
 * rotor_workspace_bytes(); d_workspace == NULL uses the library cache.
 * Copies the (host) chain to the device and the cost/ops back inside the call
 * (the end-to-end path); blocks until done. */
int rotor_solve_ex(const rotor_chain *chain, int32_t L, uint64_t mem_limit, int32_t slots,
                   const rotor_options *opt, void *d_workspace, uint64_t workspace_bytes, void *stream,
                   double *cost_out, rotor_op *ops, int64_t ops_cap, int64_t *n_ops_out);

/* Device-resident solve: d_chain holds DEVICE pointers; results are written to
 * device memory: *d_cost (double), d_ops[0..ops_cap), *d_n_ops (int64: op
 * count, -1 if infeasible), *d_status (int32 rotor_status of the device
 * phase).  Fully asynchronous on `stream` (no host synchronisation); host-side
 * argument errors are returned immediately.  d_workspace is required. */
int rotor_solve_device(const rotor_chain *d_chain, int32_t L, uint64_t mem_limit, int32_t slots,
                       const rotor_options *opt, void *d_workspace, uint64_t workspace_bytes, void *stream,
                       double *d_cost, rotor_op *d_ops, int64_t ops_cap, int64_t *d_n_ops, int32_t *d_status);

/* Device workspace bytes needed for (L, S, options). */
int rotor_workspace_bytes(int32_t L, int32_t slots, const rotor_options *opt, uint64_t *bytes);

/* Test / debug aid: where the tiled fill keeps its fp32 round-down shadows in
 * a workspace of rotor_workspace_bytes, so a caller holding
 * the workspace (rotor_solve_device) can check them against the fp64 table.
 * out[0] byte offset of C32, out[1] rows of C32 (scrows), out[2] byte offset
 * of A32, out[3] rows of A32 (sarows), out[4] byte offset of C (the cell
 * (1,1) at m = 0), out[5] doubles per C row (pitch).  C32 / A32 are float
 * arrays in the m-chunked layout: element (row, m) at ((m / 32) * rows + row)
 * * 32 + m % 32; rows follow srow_c / srow_a / sc_row / sa_col of
 * rotor_common.cuh (block-major, 32 cells then 8 quad minima per block
 * column / row).  Shadows exist only for the tiled kernel (ROTOR_EINPUT for
 * an options set without them). */
int rotor_shadow_layout(int32_t L, int32_t slots, const rotor_options *opt, int64_t out[6]);

/* Upper bound on the op count of any schedule Algorithm 2 can return for L:
 * n(n+1)/2 forwards + n backwards, n = L+1 (a node (s,t) split at s' emits
 * s'-s forwards; by induction an interval of len stages emits at most
 * len(len+1)/2) — a safe ops_cap. */
int64_t rotor_max_ops(int32_t L);

/* ---------------------------------------------------------------------------
 * Batched multi-limit solve ("Algorithm 1 for 10 different memory
 * limits"): n_chains chains x n_limits limits, each pair its own table with
 * slot size limits[i*n_limits+j]/S (§5.2).  SURVEY.md §8(e) 1: the problems
 * are independent, so they are spread over a device list with no exchange.
 *   chains[i], Ls[i]          : host chains
 *   limits[i*n_limits + j]    : bytes
 *   devices, n_devices        : where to run.  devices == NULL && n_devices == 0:
 *                               the current device, on `stream`.  A list of
 *                               n_devices >= 1 CUDA ordinals (an ordinal may
 *                               repeat): the problems are split by LPT on their
 *                               nominal transitions (rotor_partition_lpt), one
 *                               host thread per entry, each with its own stream
 *                               and library workspace on its device; `stream`
 *                               is then unused.  devices == NULL && n_devices < 0:
 *                               every visible device.
 *   costs[i*n_limits + j]     : out
 *   ops + ops_offsets[p]      : out, problem p = i*n_limits + j writes at most ops_caps[p]
 *                               ops at ops + ops_offsets[p] (ops may be NULL: costs only)
 *   n_ops[p]                  : out (-1 if infeasible); may be NULL
 *   status[p]                 : out rotor_status per problem (OK, INFEASIBLE,
 *                               ETRUNC when ops[] was too short); may be NULL
 * Blocks until every result is on the host.  Returns ROTOR_OK if every
 * problem ran (individual infeasibility is reported in status[]), else the
 * first error (with the failing device in rotor_last_error()).
 * ------------------------------------------------------------------------- */
int rotor_solve_batch(const rotor_chain *chains, const int32_t *Ls, int32_t n_chains, const uint64_t *limits,
                      int32_t n_limits, int32_t slots, const rotor_options *opt, const int32_t *devices,
                      int32_t n_devices, void *stream, double *costs, rotor_op *ops, const int64_t *ops_offsets,
                      const int64_t *ops_caps, int64_t *n_ops, int32_t *status);

/* ---------------------------------------------------------------------------
 * One table sharded over a device list, driven from ONE process (SURVEY.md
 * §8(e) 2).  The tiled fill's 32 x 32-stage tiles of tile diagonal delta
 * depend only on tiles of smaller delta (Theorem 1 reads strictly shorter
 * intervals), so per delta every device computes a contiguous,
 * balanced range of the tiles, and the finished tiles travel to the others
 * before delta + 1:
 *   halo_mode 0: the owner packs its tiles' C rows into a staging buffer, each
 *                other device pulls the buffer with a peer copy
 *                (cudaMemcpyPeerAsync over NVLink) and unpacks it;
 *   halo_mode 1: fused peer pull — each other device's unpack kernel reads the
 *                owner's C rows directly through peer memory (P2P loads over
 *                NVLink), no staging buffer (needs peer access; falls back to
 *                mode 0 where a pair has none).
 * Receivers rebuild the A rows and the fp32 shadows from C with the fill's own
 * association (Q12), so results are bit-identical to rotor_solve.  Devices
 * synchronise by CUDA events only; the host thread only enqueues.  The first
 * device runs Algorithm 2 on its complete table.
 *   chain, L, mem_limit, slots, opt : as rotor_solve_ex (host chain; the fill is the tiled one)
 *   devices, n_devices : CUDA ordinals (an ordinal may repeat: several shards on
 *                        one device, each with its own workspace); devices ==
 *                        NULL: ordinals 0..n_devices-1 (n_devices < 0: every
 *                        visible device)
 *   cost_out, ops, ops_cap, n_ops_out : as rotor_solve
 * Library workspaces (one per entry, rotor_workspace_bytes each) are leased
 * for the call; the first entry's table is this thread's "last solve"
 * (rotor_export_*).  Blocks until the result is on the host.
 * ------------------------------------------------------------------------- */
int rotor_solve_sharded(const rotor_chain *chain, int32_t L, uint64_t mem_limit, int32_t slots,
                        const rotor_options *opt, const int32_t *devices, int32_t n_devices, int32_t halo_mode,
                        double *cost_out, rotor_op *ops, int64_t ops_cap, int64_t *n_ops_out);

/* ---------------------------------------------------------------------------
 * Sharded single-table solve, for one process per GPU
 * (the building blocks rotor_solve_sharded drives itself in one process).
 * The tiled fill cuts the (s,t) triangle into 32x32-stage tiles processed by
 * tile diagonal delta = 0 .. rotor_tile_blocks(L)-1; every tile of one delta
 * depends only on tiles of smaller delta (Theorem 1 reads strictly shorter
 * intervals).  Each rank keeps a full workspace; per delta it
 * computes its share of the tiles (rotor_sharded_step), packs them
 * (rotor_sharded_pack), the caller all-gathers the packed buffers (NCCL), and
 * every rank unpacks the other ranks' tiles (rotor_sharded_pack, unpack = 1).
 * All calls enqueue on `stream` and return immediately.  A handle owns the
 * state of one sharded solve (several handles may coexist, e.g. to emulate
 * ranks on one GPU).  The result equals rotor_solve's bit for bit (the same
 * kernels compute every tile).
 * ------------------------------------------------------------------------- */
typedef struct rotor_shard rotor_shard;
int32_t rotor_tile_blocks(int32_t L);                 /* ceil((L+1)/32) */
int rotor_tile_bytes(int32_t slots, uint64_t *bytes); /* packed bytes per tile (its C rows, all m) */
/* discretise + limits + leaf diagonal + setup; d_chain and the workspace as in
 * rotor_solve_device (options: kernel forced to TILED).  *out: new handle. */
int rotor_sharded_begin(const rotor_chain *d_chain, int32_t L, uint64_t mem_limit, int32_t slots,
                        const rotor_options *opt, void *d_workspace, uint64_t workspace_bytes, void *stream,
                        rotor_shard **out);
/* middle + dependent phase of the tiles I in [tile_lo, tile_hi) of diagonal delta
 * (0 <= tile_lo <= tile_hi <= rotor_tile_blocks(L) - delta) */
int rotor_sharded_step(rotor_shard *h, int32_t delta, int32_t tile_lo, int32_t tile_hi, void *stream);
/* copy those tiles' C rows to (unpack = 0) or from (unpack = 1) d_buf, layout
 * [tile][32 s][32 t][S+1] fp64, buf_bytes >= count * rotor_tile_bytes; unpack
 * also rebuilds the A rows, A(s,t,m) = fl(fl(P[t] - P[s-1]) + C(s,t,m)) (the
 * fill's own association, Q12: bit-identical), so only C travels */
int rotor_sharded_pack(rotor_shard *h, int32_t delta, int32_t tile_lo, int32_t tile_hi, void *d_buf,
                       uint64_t buf_bytes, int32_t unpack, void *stream);
/* Algorithm 2 on the completed table; outputs as in rotor_solve_device.  Also
 * makes this table the "last solve" of the thread for rotor_export_*. */
int rotor_sharded_finish(rotor_shard *h, void *stream, double *d_cost, rotor_op *d_ops, int64_t ops_cap,
                         int64_t *d_n_ops, int32_t *d_status);
int rotor_sharded_free(rotor_shard *h);
/* Kernels this shard has launched since rotor_sharded_begin (begin, steps,
 * packs / unpacks, finish); host-side counter, no synchronisation. */
int rotor_sharded_launches(const rotor_shard *h, int64_t *launches);

/* Longest-processing-time partition of n_items weighted items over n_parts
 * parts (host helper for sharding independent solves across GPUs/ranks).
 * part_of[i] in 0..n_parts-1; deterministic (ties -> lowest part index). */
int rotor_partition_lpt(const double *weights, int32_t n_items, int32_t n_parts, int32_t *part_of);

/* Nominal DP transitions of one table: sum_{d=1}^{L} (L+1-d)(d+1)(S+1)
 * (every cell of diagonal d has d F_ck candidates + 1 F_all candidate). */
double rotor_transitions(int32_t L, int32_t slots);

/* ---------------------------------------------------------------------------
 * Parity / debug: copy the tables of the LAST solve made by this thread
 * (rotor_solve / rotor_solve_ex / rotor_solve_device) to host memory, in the
 * canonical layout
 *     cell(s,t) = (s-1)*n - (s-1)*(s-2)/2 + (t-s), n = L+1   (s-major)
 *     C_host[cell*(S+1) + m], m = 0..S      (fp64; +inf = infeasible)
 *     D_host[cell*(S+1) + m]                (uint16: k = s'-s for an F_ck split,
 *                                            0 for F_all / leaf, 0xFFFF if C = +inf)
 * n_values must equal n(n+1)/2*(S+1).  Either pointer may be NULL.  D is
 * derived on the device from C by Algorithm 2's test (smallest s' with
 * C = C_ck) unless it was recorded during the fill.  The workspace of
 * that solve must still be alive.  Synchronous.
 * ------------------------------------------------------------------------- */
int rotor_export_tables(double *C_host, uint16_t *D_host, int64_t n_values);

/* Sampled export of the last solve: for r = 0..n_rows-1, copies the S+1 values
 * C[s[r], t[r], 0..S] to C_host[r*(S+1) ...] (1 <= s[r] <= t[r] <= L+1).
 * Used for parity at sizes whose full table does not fit host memory. */
int rotor_export_rows(const int32_t *s, const int32_t *t, int64_t n_rows, double *C_host);

/* Phase timings of the last solve on this thread (options.profile = 1). */
typedef struct {
    double pre_ms;         /* discretise + prefix sums + limits + leaf diagonal */
    double fill_ms;        /* all diagonals d = 1..L (the dominant phase) */
    double reconstruct_ms; /* Algorithm 2 walk */
    int32_t fill_launches; /* kernels launched for the fill */
    int32_t total_launches;/* kernels launched by the solve */
    double middle_ms;      /* tiled fill: the middle-kernel launches alone (events on the launch stream) */
    int32_t middle_launches;
} rotor_timings;
int rotor_last_timings(rotor_timings *out);

/* Work counters of the last solve on this thread (options.counters = 1, tiled
 * fill).  Every cell of diagonal d >= 1 has d + 1 candidates (Eq. (2),
 * P:723-737); the nominal count is independent of gating and pruning.  The
 * tiled fill's middle kernel (splits s' in the tile blocks strictly between
 * the cell's row and column blocks) filters its candidates
 * with exact fp32 lower bounds; what it did is counted per (warp, split)
 * visit, a warp covering an 8 x 8 cell tile x 32 m (2048 candidates):
 *   middle_split_visits : (warp, split) visits            (x 2048 candidates)
 *   coarse_pass         : visits whose whole-tile bound did not reject the split
 *   quadrant_compares   : 4 x 4 quadrants compared cell by cell (x 512 fp32 compares)
 *   exact_splits        : visits recomputed in fp64        (x 2048 candidates)
 * Everything else (the dependent phase: splits inside the cell's own tile
 * blocks, F_all, the gates) is evaluated exactly, candidate by candidate.
 * Synchronous. */
typedef struct {
    double nominal;                 /* sum_{d=1}^{L} (n-d)(d+1)(S+1) */
    double middle_nominal;          /* candidates of the middle ranges (existing cells, m = 0..S) */
    double dependent_nominal;       /* nominal - middle_nominal */
    uint64_t middle_split_visits;
    uint64_t coarse_pass;
    uint64_t quadrant_compares;
    uint64_t exact_splits;
    double evaluated;               /* 512 quadrant_compares + 2048 exact_splits + dependent_nominal */
    /* clock cycles of the middle's warps, summed over warps (where its time goes) */
    uint64_t middle_wait_cycles;    /* waiting for operand boxes (the bulk-copy ring) */
    uint64_t middle_init_cycles;    /* item setup (gates, bounds) */
    uint64_t middle_loop_cycles;    /* the filter over the splits */
    uint64_t middle_flush_cycles;   /* the exact fp64 pass of the fired splits */
    double middle_warp_imbalance;   /* max / mean over the 16 warp slots of (loop + flush) cycles */
    uint64_t middle_slot_cycles[16];/* (loop + flush) cycles per warp slot = 8 x 8 sub-tile position in the tile */
    /* where the off-diagonal leaves' time goes (ns of GPU global timer, summed
     * over CTAs, thread 0 of each): setup (arrival ticket, sub-tile tables,
     * staged operands), waiting for the lower m-chunks' rows (look-back
     * flags), the rows' own work, the per-row barrier + release */
    uint64_t leaf_ctas;
    uint64_t leaf_setup_ns;
    uint64_t leaf_wait_ns;
    uint64_t leaf_work_ns;          /* the rows after pass 1: right range, F_all, stores (+ the next row's early loads) */
    uint64_t leaf_sync_ns;
    uint64_t leaf_pass1_ns;         /* the rows' pass 1: the rows-below / F_all loads and the left range */
} rotor_counters;
int rotor_last_counters(rotor_counters *out);

/* Release the library-owned cached workspaces (all devices). */
int rotor_release(void);

const char *rotor_last_error(void);
int32_t rotor_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ROTOR_H */
