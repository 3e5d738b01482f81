// Host side of the C ABI declared in include/rotor.h: argument validation,
// workspace layout, launch sequencing, caching, export and timing.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <map>
#include <thread>
#include <mutex>
#include <numeric>
#include <vector>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "rotor.h"
#include "rotor_common.cuh"
#include "rotor_kernels.cuh"

namespace {

// NVTX ranges around the host-side phases of every entry point (no-ops unless a
// profiler such as Nsight Systems is attached): a timeline of a solve is
// segmented into precompute / fill / reconstruct, per tile diagonal and per
// sharded rank.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

thread_local std::string g_err;

int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) return fail(ROTOR_EDEVICE, "%s: %s", #x, cudaGetErrorString(e_)); \
    } while (0)

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

// Workspace layout of one problem (all offsets 256-byte aligned).
struct Layout {
    int L = 0, n = 0, S = 0;
    int64_t pitch = 0, cells = 0;
    int stack_cap = 0;
    int64_t ops_cap = 0;
    size_t off_wx, off_wbx, off_wy, off_of, off_ob, off_P, off_w, off_mnull, off_stack, off_res;
    size_t off_chain, off_ops, off_C, off_D, off_A, off_C32, off_A32, off_tiled, off_ctr;
    int64_t sarows = 0, scrows = 0;
    size_t total = 0;
    bool has_D = false;
    bool has_A = false;
};

// The tiled fill is the default (AUTO); the wavefront kernel is used when
// requested explicitly or when the argmin table D is recorded during the fill.
bool uses_tiled(const rotor_options &o) {
    if (o.kernel == ROTOR_KERNEL_TILED) return true;
    if (o.kernel == ROTOR_KERNEL_WAVEFRONT) return false;
    return o.keep_argmin == 0;
}

int64_t max_ops(int L) {
    int64_t n = (int64_t)L + 1;
    return n * (n + 1) / 2 + n;
}

Layout make_layout(int L, int S, const rotor_options &o) {
    Layout y;
    y.L = L;
    y.n = L + 1;
    y.S = S;
    y.pitch = ((int64_t)rotor::kPad + S + 1 + 31) / 32 * 32;  // 256-byte aligned rows, left pad
    y.cells = (int64_t)y.n * (y.n + 1) / 2;
    y.stack_cap = 4 * y.n + 64;
    y.ops_cap = max_ops(L);
    const size_t n2 = (size_t)y.n + 2;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t r = off;
        off += al(bytes);
        return r;
    };
    y.off_wx = take(n2 * 4);
    y.off_wbx = take(n2 * 4);
    y.off_wy = take(n2 * 4);
    y.off_of = take(n2 * 4);
    y.off_ob = take(n2 * 4);
    y.off_P = take(n2 * 8);
    y.off_w = take(n2 * 8);
    y.off_mnull = take((size_t)y.n * y.n * 4);
    y.off_stack = take((size_t)y.stack_cap * sizeof(int4));
    y.off_res = take(64);
    y.off_ctr = take(256);
    y.off_chain = take(7 * al(n2 * 8));
    y.off_ops = take((size_t)y.ops_cap * sizeof(rotor_op));
    y.off_C = take((size_t)(y.cells + rotor::kPadRows) * y.pitch * 8);
    y.has_D = o.keep_argmin != 0;
    y.off_D = y.has_D ? take((size_t)y.cells * y.pitch * 2) : 0;
    y.has_A = uses_tiled(o);
    y.off_A = y.has_A ? take((size_t)(y.cells + rotor::kPadRows) * y.pitch * 8) : 0;
    y.scrows = rotor::shadow_rows_c(y.n);
    y.sarows = rotor::shadow_rows_a(y.n);
    y.off_C32 = y.has_A ? take((size_t)y.scrows * y.pitch * 4) : 0;
    y.off_A32 = y.has_A ? take((size_t)y.sarows * y.pitch * 4) : 0;
    y.off_tiled = take(rotor::tiled_extra_bytes(L, S));
    y.total = off;
    return y;
}

rotor::Problem make_problem(const Layout &y, char *ws, const rotor_options &o) {
    rotor::Problem p{};
    p.L = y.L;
    p.n = y.n;
    p.S = y.S;
    p.restricted = o.restricted ? 1 : 0;
    p.pitch = y.pitch;
    p.wx = (int32_t *)(ws + y.off_wx);
    p.wbx = (int32_t *)(ws + y.off_wbx);
    p.wy = (int32_t *)(ws + y.off_wy);
    p.of = (int32_t *)(ws + y.off_of);
    p.ob = (int32_t *)(ws + y.off_ob);
    p.P = (double *)(ws + y.off_P);
    p.w = (double *)(ws + y.off_w);
    p.mnullT = (int32_t *)(ws + y.off_mnull);
    p.stack = (int4 *)(ws + y.off_stack);
    p.stack_cap = y.stack_cap;
    p.C = (double *)(ws + y.off_C) + rotor::kPad;  // column m = 0 of row 0
    p.D = y.has_D ? (uint16_t *)(ws + y.off_D) + rotor::kPad : nullptr;
    p.A = y.has_A ? (double *)(ws + y.off_A) + rotor::kPad : nullptr;
    p.C32 = y.has_A ? (float *)(ws + y.off_C32) : nullptr;
    p.A32 = y.has_A ? (float *)(ws + y.off_A32) : nullptr;
    p.sarows = y.sarows;
    p.scrows = y.scrows;
    p.counters = (y.has_A && o.counters) ? (unsigned long long *)(ws + y.off_ctr) : nullptr;
    p.flags = y.has_A ? (int *)(ws + y.off_tiled) : nullptr;
    p.mlist = y.has_A ? (uint16_t *)(ws + y.off_tiled + rotor::tiled_list_offset(y.L, y.S)) : nullptr;
    p.res_cost = (double *)(ws + y.off_res);
    p.res_nops = (int64_t *)(ws + y.off_res + 8);
    p.res_status = (int32_t *)(ws + y.off_res + 16);
    p.ops = (rotor_op *)(ws + y.off_ops);
    p.ops_cap = y.ops_cap;
    return p;
}

rotor_options opts_or_default(const rotor_options *o) {
    rotor_options r;
    memset(&r, 0, sizeof r);
    if (o) r = *o;
    return r;
}

int check_args(int32_t L, uint64_t M, int32_t S) {
    if (L < 1) return fail(ROTOR_EINPUT, "L must be >= 1 (got %d)", L);
    if (L > 65000) return fail(ROTOR_EINPUT, "L must be <= 65000 (argmin codes are uint16)");
    if (S < 1) return fail(ROTOR_EINPUT, "slots must be >= 1 (got %d)", S);
    if (S > (1 << 28)) return fail(ROTOR_EINPUT, "slots too large");
    if (M == 0) return fail(ROTOR_EINPUT, "mem_limit must be > 0");
    return ROTOR_OK;
}

int check_host_chain(const rotor_chain *c, int L) {
    if (!c || !c->uf || !c->ub || !c->wx || !c->wbx || !c->wy || !c->of || !c->ob)
        return fail(ROTOR_EINPUT, "chain has a NULL array");
    for (int i = 0; i <= L; i++) {
        double a = c->uf[i], b = c->ub[i];
        if (!(a >= 0.0 && a < INFINITY) || !(b >= 0.0 && b < INFINITY))
            return fail(ROTOR_EINPUT, "times must be finite and >= 0 (stage %d)", i + 1);
    }
    return ROTOR_OK;
}

// ---- library-owned cached workspaces ----
// One entry per (device, kind): kind 0 = rotor_solve / rotor_solve_ex, kind
// kBatchKind + w = batch worker w, kShardKind + r = sharded rank r.  A call
// LEASES its entry for its whole duration (the entry's mutex), so two threads
// never share a workspace; a call that grows an entry frees the old buffer.
// `gen` counts the solves an entry has served: the last-solve record keeps it,
// and the export calls refuse to read an entry a later call has reused.
constexpr int kBatchKind = 16, kShardKind = 4096;
struct CacheEntry {
    std::mutex mu;
    void *ptr = nullptr;
    size_t bytes = 0;
    std::atomic<uint64_t> gen{0};
};
std::mutex g_cache_mu;
std::map<std::pair<int, int>, std::unique_ptr<CacheEntry>> g_cache;

struct Lease {
    CacheEntry *e = nullptr;
    std::unique_lock<std::mutex> lk;
};

int lease_workspace(int kind, size_t bytes, Lease &l, void **out) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CacheEntry *e;
    {
        std::lock_guard<std::mutex> g(g_cache_mu);
        auto &slot = g_cache[{dev, kind}];
        if (!slot) slot.reset(new CacheEntry());
        e = slot.get();
    }
    l.lk = std::unique_lock<std::mutex>(e->mu);
    l.e = e;
    if (e->bytes < bytes) {
        if (e->ptr) {
            cudaDeviceSynchronize();
            cudaFree(e->ptr);
            e->ptr = nullptr;
            e->bytes = 0;
        }
        void *p = nullptr;
        cudaError_t err = cudaMalloc(&p, bytes);
        if (err != cudaSuccess) {
            cudaGetLastError();
            return fail(ROTOR_ENOMEM, "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(err));
        }
        e->ptr = p;
        e->bytes = bytes;
    }
    e->gen++;
    *out = e->ptr;
    return ROTOR_OK;
}

// ---- per-thread record of the last solve (export / timings) ----
struct LastSolve {
    bool valid = false;
    Layout y;
    rotor::Problem p;
    int device = 0;
    cudaStream_t stream = nullptr;
    bool profiled = false;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    int fill_launches = 0, total_launches = 0;
    std::vector<cudaEvent_t> mid_ev;  // pairs around the tiled fill's middle launches
    int mid_n = 0;
    bool counted = false;  // options.counters: p.counters holds this solve's middle counters
    CacheEntry *cache = nullptr;  // the library workspace the tables live in (nullptr: caller-owned)
    uint64_t cache_gen = 0;
};
thread_local LastSolve g_last;

// The tables of the last solve are still readable: a library workspace may
// have been reused by a later call (of any thread) since.
int check_last_alive() {
    if (!g_last.valid) return fail(ROTOR_EINPUT, "no solve on this thread");
    if (g_last.cache && g_last.cache->gen.load() != g_last.cache_gen)
        return fail(ROTOR_EINVALID, "the library workspace of the last solve was reused by a later call");
    return ROTOR_OK;
}

int ensure_events() {
    for (auto &e : g_last.ev)
        if (!e) CK(cudaEventCreate(&e));
    return ROTOR_OK;
}

// Enqueue the whole device path for one problem (no host synchronisation).
// Results go to the workspace's own result/ops areas unless `redirect` is given.
struct Outputs {
    double *cost;
    int64_t *nops;
    int32_t *status;
    rotor_op *ops;
    int64_t ops_cap;
};

int enqueue_solve(const rotor_chain &dch, uint64_t M, const Layout &y, char *ws, const rotor_options &o,
                  cudaStream_t st, const Outputs *redirect) {
    rotor::Problem p = make_problem(y, ws, o);
    if (redirect) {
        p.res_cost = redirect->cost;
        p.res_nops = redirect->nops;
        p.res_status = redirect->status;
        p.ops = redirect->ops;
        p.ops_cap = redirect->ops_cap;
    }
    int dev = 0;
    CK(cudaGetDevice(&dev));
    g_last.valid = true;
    g_last.y = y;
    g_last.p = p;
    g_last.device = dev;
    g_last.stream = st;
    g_last.profiled = o.profile != 0;
    g_last.counted = p.counters != nullptr;
    g_last.cache = nullptr;
    if (p.counters) CK(cudaMemsetAsync(p.counters, 0, 256, st));
    if (o.profile) {
        int r = ensure_events();
        if (r) return r;
        CK(cudaEventRecord(g_last.ev[0], st));
    }
    int launches = 0;
    NvtxRange nv_solve("rotor.solve");
    {
        NvtxRange nv("rotor.precompute+leaf");
        rotor::launch_precompute(dch, M, p, st);
        rotor::launch_leaf(p, st);
    }
    launches += 2;
    CK(cudaGetLastError());
    if (o.profile) CK(cudaEventRecord(g_last.ev[1], st));
    int fill = 0;
    if (y.has_A) {
        g_last.mid_n = 0;
        int cap = 0;
        if (o.profile) {
            const int nb = rotor::tiled_nb(y.n);
            cap = nb * (nb - 1) / 2;  // middle launches: one per diagonal, or one per tile (DAG schedule)
            while ((int)g_last.mid_ev.size() < 2 * cap) {
                cudaEvent_t e;
                CK(cudaEventCreate(&e));
                g_last.mid_ev.push_back(e);
            }
        }
        {
            NvtxRange nv("rotor.fill.tiled");
            fill = rotor::launch_fill_tiled(p, st, o.schedule, cap ? g_last.mid_ev.data() : nullptr, cap, &g_last.mid_n);
        }
        if (fill < 0) {
            cudaError_t e = cudaGetLastError();
            return fail(ROTOR_EDEVICE, "tiled fill launch failed: %s", cudaGetErrorString(e));
        }
    } else {
        NvtxRange nv("rotor.fill.wavefront");
        for (int d = 1; d <= y.L; d++) rotor::launch_diag_wavefront(p, d, st);
        fill = y.L;
    }
    CK(cudaGetLastError());
    launches += fill;
    if (o.profile) CK(cudaEventRecord(g_last.ev[2], st));
    NvtxRange nv_rec("rotor.reconstruct");
    rotor::launch_reconstruct(p, st);
    launches += 1;
    CK(cudaGetLastError());
    if (o.profile) CK(cudaEventRecord(g_last.ev[3], st));
    g_last.fill_launches = fill;
    g_last.total_launches = launches;
    return ROTOR_OK;
}

// ---- batched independent solves (rotor_solve_batch) ----
struct BatchIn {
    const rotor_chain *chains;
    const int32_t *Ls;
    int32_t n_chains;
    const uint64_t *limits;
    int32_t n_limits, slots;
    rotor_options o;
    rotor_op *ops;
    const int64_t *ops_offsets, *ops_caps;
};
struct BatchOut {
    double *costs;
    int64_t *n_ops;
    int32_t *status;
};

// Per-thread pinned host staging (grown, never shrunk) for device-to-host result copies.
rotor_op *pinned_staging(size_t bytes) {
    static thread_local void *buf = nullptr;
    static thread_local size_t cap = 0;
    if (cap < bytes) {
        if (buf) cudaFreeHost(buf);
        buf = nullptr;
        cap = 0;
        if (cudaMallocHost(&buf, bytes) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        cap = bytes;
    }
    return (rotor_op *)buf;
}

// The problems idx (global index q = chain * n_limits + limit) on the current
// device: one fused k_batch launch on `st`, results scattered to the caller's
// arrays at their global indices (distinct workers write disjoint entries).
int batch_on_device(const BatchIn &in, const std::vector<int64_t> &idx, int kind, cudaStream_t st,
                    const BatchOut &out) {
    NvtxRange nv("rotor.batch");
    const int64_t P = (int64_t)idx.size();
    if (P == 0) return ROTOR_OK;
    const int n_chains = in.n_chains, slots = in.slots;
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    int L_max = 0;
    for (int i = 0; i < n_chains; i++) L_max = std::max(L_max, (int)in.Ls[i]);

    // host staging: chains padded to a common stride, problem descriptors
    const int64_t stride = L_max + 2;
    std::vector<double> h_d(2 * n_chains * stride, 0.0);
    std::vector<uint64_t> h_u(5 * n_chains * stride, 0);
    for (int i = 0; i < n_chains; i++) {
        const int n1 = in.Ls[i] + 1;
        memcpy(&h_d[(0 * n_chains + i) * stride], in.chains[i].uf, n1 * 8);
        memcpy(&h_d[(1 * n_chains + i) * stride], in.chains[i].ub, n1 * 8);
        memcpy(&h_u[(0 * n_chains + i) * stride], in.chains[i].wx, n1 * 8);
        memcpy(&h_u[(1 * n_chains + i) * stride], in.chains[i].wbx, n1 * 8);
        memcpy(&h_u[(2 * n_chains + i) * stride], in.chains[i].wy, (n1 + 1) * 8);
        memcpy(&h_u[(3 * n_chains + i) * stride], in.chains[i].of, n1 * 8);
        memcpy(&h_u[(4 * n_chains + i) * stride], in.chains[i].ob, n1 * 8);
    }
    std::vector<int32_t> h_pc(P), h_L(in.Ls, in.Ls + n_chains);
    std::vector<uint64_t> h_lim(P);
    std::vector<int64_t> h_off(P, 0), h_cap(P, 0);
    int64_t total_ops = 0;
    for (int64_t k = 0; k < P; k++) {
        const int64_t q = idx[k];
        h_pc[k] = (int32_t)(q / in.n_limits);
        h_lim[k] = in.limits[q];
        if (in.ops) {
            h_cap[k] = std::max<int64_t>(0, in.ops_caps[q]);
            h_off[k] = total_ops;
            total_ops += h_cap[k];
        }
    }
    // queue order: the longest chains first (cost ~ L^3 at a common S): the
    // short tables fill the tail instead of a long one starting last
    std::vector<int32_t> h_order(P);
    for (int64_t k = 0; k < P; k++) h_order[k] = (int32_t)k;
    std::stable_sort(h_order.begin(), h_order.end(),
                     [&](int32_t x, int32_t y) { return in.Ls[h_pc[x]] > in.Ls[h_pc[y]]; });
    // persistent k_batch CTAs (512 threads): batch_ctas_per_sm() resident per SM
    // (rotor_batch.cu; before the pruning, config 5: 1 per SM 86.4 ms, 2 59.0, 3 50.0 at 40
    // registers / 47.5 at 32, 4 44.6; 256 threads x 6 62.6, x 7 60.6; 384 x 4
    // 50.6; 128 x 12 91.2)
    const int n_slots = (int)std::min<int64_t>(P, rotor::batch_ctas_per_sm() * (int64_t)sms);
    const size_t slot = rotor::batch_slot_bytes(L_max, slots);
    // one device allocation (a leased library workspace): descriptors, outputs, ops, then the slot pool
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t r = off;
        off += al(bytes);
        return r;
    };
    const size_t o_d = take(h_d.size() * 8), o_u = take(h_u.size() * 8), o_pc = take(P * 4), o_L = take(n_chains * 4),
                 o_lim = take(P * 8), o_off = take(P * 8), o_cap = take(P * 8), o_cost = take(P * 8),
                 o_nops = take(P * 8), o_st = take(P * 4), o_ops = take((size_t)std::max<int64_t>(total_ops, 1) * 8),
                 o_ctr = take(8), o_ord = take(P * 4), o_pool = take((size_t)n_slots * slot),
                 o_cmp = take((size_t)std::max<int64_t>(total_ops, 1) * 8);  // compacted ops
    void *wsv = nullptr;
    Lease lease;
    int r = lease_workspace(kind, off, lease, &wsv);
    if (r) return r;
    char *w = (char *)wsv;
    CK(cudaMemcpyAsync(w + o_d, h_d.data(), h_d.size() * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(w + o_u, h_u.data(), h_u.size() * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(w + o_pc, h_pc.data(), P * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(w + o_L, h_L.data(), n_chains * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(w + o_lim, h_lim.data(), P * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(w + o_off, h_off.data(), P * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(w + o_cap, h_cap.data(), P * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(w + o_ord, h_order.data(), P * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(w + o_ctr, 0, 8, st));
    rotor::BatchArgs b{};
    b.n_problems = (int)P;
    b.S = slots;
    b.restricted = in.o.restricted ? 1 : 0;
    b.L_max = L_max;
    b.prob_chain = (const int32_t *)(w + o_pc);
    b.limits = (const uint64_t *)(w + o_lim);
    b.chain_L = (const int32_t *)(w + o_L);
    b.chain_stride = stride;
    b.uf = (const double *)(w + o_d);
    b.ub = (const double *)(w + o_d) + n_chains * stride;
    b.wx = (const uint64_t *)(w + o_u);
    b.wbx = (const uint64_t *)(w + o_u) + 1 * n_chains * stride;
    b.wy = (const uint64_t *)(w + o_u) + 2 * n_chains * stride;
    b.of = (const uint64_t *)(w + o_u) + 3 * n_chains * stride;
    b.ob = (const uint64_t *)(w + o_u) + 4 * n_chains * stride;
    b.pool = w + o_pool;
    b.cost = (double *)(w + o_cost);
    b.nops = (int64_t *)(w + o_nops);
    b.status = (int32_t *)(w + o_st);
    b.ops = in.ops ? (rotor_op *)(w + o_ops) : nullptr;
    b.ops_off = (const int64_t *)(w + o_off);
    b.ops_cap = (const int64_t *)(w + o_cap);
    b.counter = (int *)(w + o_ctr);
    b.order = (const int32_t *)(w + o_ord);
    // ROTOR_BATCH_MC: m-chunk of k_batch's fill order (config 5, ms per sweep,
    // every candidate: whole rows 31.6, 16 m 31.8, 32 m 32.7, 64 m 30.8, 128 m
    // 29.2; pruned: whole rows 26.9, 64 m 18.5, 128 m 19.6, 256 m 21.3)
    static const int batch_mc = [] {
        const char *e = getenv("ROTOR_BATCH_MC");
        return e ? atoi(e) : 64;
    }();
    b.mc = batch_mc;
    // ROTOR_BATCH_PRUNE: 1 (default) the monotone-in-m bound per warp of 32 m,
    // 2/4 per 16/8 m (config 5: 18.9 / 22.3 / 23.4 ms), 0 every candidate of
    // every cell (wavefront_cell, 26.2 ms)
    static const int batch_prune = [] {
        const char *e = getenv("ROTOR_BATCH_PRUNE");
        return e ? atoi(e) : 1;
    }();
    b.prune = batch_prune;
    rotor::launch_batch(b, n_slots, st);
    CK(cudaGetLastError());
    std::vector<double> h_c(P);
    std::vector<int64_t> h_n(P);
    std::vector<int32_t> h_s(P);
    CK(cudaMemcpyAsync(h_c.data(), w + o_cost, P * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(h_n.data(), w + o_nops, P * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(h_s.data(), w + o_st, P * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    // the ops: compacted on the device (problem k's min(n_k, cap_k) ops after
    // the previous problems'), ONE copy into pinned staging, then scattered on
    // the host into the caller's buffer
    std::vector<int64_t> h_cnt(P, 0), h_dst(P, 0);
    int64_t n_copy = 0;
    if (in.ops) {
        for (int64_t k = 0; k < P; k++) {
            h_cnt[k] = h_n[k] > 0 ? std::min(h_n[k], h_cap[k]) : 0;
            h_dst[k] = n_copy;
            n_copy += h_cnt[k];
        }
    }
    rotor_op *staged = nullptr;
    if (n_copy > 0) {
        // reuse the offsets area of the descriptors: o_off (src offsets), o_cap
        // (counts) and o_nops (destination offsets) are no longer needed
        CK(cudaMemcpyAsync(w + o_cap, h_cnt.data(), P * 8, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(w + o_nops, h_dst.data(), P * 8, cudaMemcpyHostToDevice, st));
        rotor_op *dev_dst = (rotor_op *)(w + o_cmp);
        rotor::launch_compact_ops((const rotor_op *)(w + o_ops), (const int64_t *)(w + o_off),
                                  (const int64_t *)(w + o_cap), (const int64_t *)(w + o_nops), dev_dst, (int)P, st);
        CK(cudaGetLastError());
        staged = pinned_staging((size_t)n_copy * sizeof(rotor_op));
        if (!staged) return fail(ROTOR_ENOMEM, "pinned staging of %lld ops failed", (long long)n_copy);
        CK(cudaMemcpyAsync(staged, dev_dst, (size_t)n_copy * sizeof(rotor_op), cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    int first_err = ROTOR_OK;
    for (int64_t k = 0; k < P; k++) {
        const int64_t q = idx[k];
        int sq = h_s[k];
        // costs-only mode (ops == NULL): the device reports ETRUNC for every
        // feasible problem (no op buffer) — that is a plain success here
        if (sq == ROTOR_ETRUNC && !in.ops) sq = ROTOR_OK;
        if (sq == ROTOR_OK && in.ops && h_n[k] > h_cap[k]) sq = ROTOR_ETRUNC;
        if (out.status) out.status[q] = sq;
        if (out.n_ops) out.n_ops[q] = (sq == ROTOR_OK || sq == ROTOR_ETRUNC) ? h_n[k] : -1;
        out.costs[q] = sq == ROTOR_INFEASIBLE ? INFINITY : h_c[k];
        if (sq != ROTOR_OK && sq != ROTOR_INFEASIBLE && sq != ROTOR_ETRUNC && !first_err) first_err = sq;
        if (h_cnt[k] > 0) memcpy(in.ops + in.ops_offsets[q], staged + h_dst[k], (size_t)h_cnt[k] * sizeof(rotor_op));
    }
    if (first_err) return fail(first_err, "batched solve: a problem failed with status %d", first_err);
    return ROTOR_OK;
}

}  // namespace

extern "C" {

int32_t rotor_version(void) { return 1; }

const char *rotor_last_error(void) { return g_err.c_str(); }

int64_t rotor_max_ops(int32_t L) { return L < 1 ? 0 : max_ops(L); }

double rotor_transitions(int32_t L, int32_t slots) {
    double n = (double)L + 1, tot = 0;
    for (int d = 1; d <= L; d++) tot += (n - d) * (d + 1) * ((double)slots + 1);
    return tot;
}

int rotor_workspace_bytes(int32_t L, int32_t slots, const rotor_options *opt, uint64_t *bytes) {
    int r = check_args(L, 1, slots);
    if (r) return r;
    if (!bytes) return fail(ROTOR_EINPUT, "bytes is NULL");
    *bytes = make_layout(L, slots, opts_or_default(opt)).total;
    return ROTOR_OK;
}

int rotor_shadow_layout(int32_t L, int32_t slots, const rotor_options *opt, int64_t out[6]) {
    int r = check_args(L, 1, slots);
    if (r) return r;
    if (!out) return fail(ROTOR_EINPUT, "out is NULL");
    const Layout y = make_layout(L, slots, opts_or_default(opt));
    if (!y.has_A) return fail(ROTOR_EINPUT, "these options use no shadows (not the tiled kernel)");
    out[0] = (int64_t)y.off_C32;
    out[1] = y.scrows;
    out[2] = (int64_t)y.off_A32;
    out[3] = y.sarows;
    out[4] = (int64_t)y.off_C + (int64_t)rotor::kPad * 8;
    out[5] = y.pitch;
    return ROTOR_OK;
}

int rotor_solve_device(const rotor_chain *d_chain, int32_t L, uint64_t mem_limit, int32_t slots,
                       const rotor_options *opt, void *d_workspace, uint64_t workspace_bytes, void *stream,
                       double *d_cost, rotor_op *d_ops, int64_t ops_cap, int64_t *d_n_ops, int32_t *d_status) {
    int r = check_args(L, mem_limit, slots);
    if (r) return r;
    if (!d_chain || !d_chain->uf || !d_chain->ub || !d_chain->wx || !d_chain->wbx || !d_chain->wy || !d_chain->of ||
        !d_chain->ob)
        return fail(ROTOR_EINPUT, "chain has a NULL array");
    if (!d_cost || !d_n_ops || !d_status) return fail(ROTOR_EINPUT, "result pointers must be non-NULL");
    if (ops_cap > 0 && !d_ops) return fail(ROTOR_EINPUT, "d_ops is NULL with ops_cap > 0");
    const rotor_options o = opts_or_default(opt);
    Layout y = make_layout(L, slots, o);
    if (!d_workspace) return fail(ROTOR_EINPUT, "d_workspace is required");
    if (workspace_bytes < y.total)
        return fail(ROTOR_ENOMEM, "workspace too small: %llu < %zu", (unsigned long long)workspace_bytes, y.total);
    Outputs out{d_cost, d_n_ops, d_status, d_ops, ops_cap < 0 ? 0 : ops_cap};
    return enqueue_solve(*d_chain, mem_limit, y, (char *)d_workspace, o, (cudaStream_t)stream, &out);
}

int rotor_solve_ex(const rotor_chain *chain, int32_t L, uint64_t mem_limit, int32_t slots, const rotor_options *opt,
                   void *d_workspace, uint64_t workspace_bytes, void *stream, double *cost_out, rotor_op *ops,
                   int64_t ops_cap, int64_t *n_ops_out) {
    int r = check_args(L, mem_limit, slots);
    if (r) return r;
    r = check_host_chain(chain, L);
    if (r) return r;
    const rotor_options o = opts_or_default(opt);
    Layout y = make_layout(L, slots, o);
    void *ws = d_workspace;
    Lease lease;
    if (!ws) {
        r = lease_workspace(0, y.total, lease, &ws);
        if (r) return r;
    } else if (workspace_bytes < y.total) {
        return fail(ROTOR_ENOMEM, "workspace too small: %llu < %zu", (unsigned long long)workspace_bytes, y.total);
    }
    cudaStream_t st = (cudaStream_t)stream;
    char *w = (char *)ws;
    const size_t n1 = (size_t)L + 1;
    const size_t seg = al(((size_t)y.n + 2) * 8);
    char *stage = w + y.off_chain;
    rotor_chain dch;
    dch.uf = (const double *)(stage + 0 * seg);
    dch.ub = (const double *)(stage + 1 * seg);
    dch.wx = (const uint64_t *)(stage + 2 * seg);
    dch.wbx = (const uint64_t *)(stage + 3 * seg);
    dch.wy = (const uint64_t *)(stage + 4 * seg);
    dch.of = (const uint64_t *)(stage + 5 * seg);
    dch.ob = (const uint64_t *)(stage + 6 * seg);
    CK(cudaMemcpyAsync((void *)dch.uf, chain->uf, n1 * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync((void *)dch.ub, chain->ub, n1 * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync((void *)dch.wx, chain->wx, n1 * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync((void *)dch.wbx, chain->wbx, n1 * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync((void *)dch.wy, chain->wy, (n1 + 1) * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync((void *)dch.of, chain->of, n1 * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync((void *)dch.ob, chain->ob, n1 * 8, cudaMemcpyHostToDevice, st));
    r = enqueue_solve(dch, mem_limit, y, w, o, st, nullptr);
    if (r) return r;
    if (lease.e) {
        g_last.cache = lease.e;
        g_last.cache_gen = lease.e->gen.load();
    }
    struct {
        double cost;
        int64_t nops;
        int32_t status;
    } res;
    CK(cudaMemcpyAsync(&res.cost, w + y.off_res, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&res.nops, w + y.off_res + 8, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&res.status, w + y.off_res + 16, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (cost_out) *cost_out = res.cost;
    if (res.status == ROTOR_INFEASIBLE) {
        if (n_ops_out) *n_ops_out = 0;
        if (cost_out) *cost_out = INFINITY;
        return fail(ROTOR_INFEASIBLE, "infeasible: no persistent schedule within the memory limit");
    }
    if (res.status != ROTOR_OK && res.status != ROTOR_ETRUNC)
        return fail(res.status, "device phase failed with status %d", res.status);
    if (n_ops_out) *n_ops_out = res.nops;
    if (ops && ops_cap > 0) {
        int64_t cnt = std::min<int64_t>(res.nops, ops_cap);
        if (cnt > 0) {
            CK(cudaMemcpyAsync(ops, w + y.off_ops, (size_t)cnt * sizeof(rotor_op), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
        }
    }
    if (ops && res.nops > ops_cap) return fail(ROTOR_ETRUNC, "ops truncated: %lld > cap %lld", (long long)res.nops,
                                               (long long)ops_cap);
    return ROTOR_OK;
}

int rotor_solve(const rotor_chain *chain, int32_t L, uint64_t mem_limit, int32_t slots, double *cost_out,
                rotor_op *ops, int64_t ops_cap, int64_t *n_ops_out) {
    return rotor_solve_ex(chain, L, mem_limit, slots, nullptr, nullptr, 0, nullptr, cost_out, ops, ops_cap,
                          n_ops_out);
}

int rotor_solve_batch(const rotor_chain *chains, const int32_t *Ls, int32_t n_chains, const uint64_t *limits,
                      int32_t n_limits, int32_t slots, const rotor_options *opt, const int32_t *devices,
                      int32_t n_devices, void *stream, double *costs, rotor_op *ops, const int64_t *ops_offsets,
                      const int64_t *ops_caps, int64_t *n_ops, int32_t *status) {
    if (!chains || !Ls || !limits || !costs || n_chains < 0 || n_limits < 0)
        return fail(ROTOR_EINPUT, "bad batch arguments");
    if (ops && (!ops_offsets || !ops_caps)) return fail(ROTOR_EINPUT, "ops requires ops_offsets and ops_caps");
    const int64_t P = (int64_t)n_chains * n_limits;
    for (int i = 0; i < n_chains; i++) {
        int r = check_args(Ls[i], 1, slots);
        if (r) return r;
        r = check_host_chain(&chains[i], Ls[i]);
        if (r) return r;
    }
    for (int64_t q = 0; q < P; q++)
        if (limits[q] == 0) return fail(ROTOR_EINPUT, "mem_limit must be > 0 (problem %lld)", (long long)q);
    if (devices && n_devices < 1) return fail(ROTOR_EINPUT, "n_devices must be >= 1 with a device list");
    // the workers: one per device-list entry (a device may be listed twice)
    std::vector<int> workers;
    int cur = 0;
    CK(cudaGetDevice(&cur));
    if (devices) {
        int nvis = 0;
        CK(cudaGetDeviceCount(&nvis));
        for (int i = 0; i < n_devices; i++) {
            if (devices[i] < 0 || devices[i] >= nvis) return fail(ROTOR_EINPUT, "bad device %d", devices[i]);
            workers.push_back(devices[i]);
        }
    } else if (n_devices < 0) {
        int nvis = 0;
        CK(cudaGetDeviceCount(&nvis));
        for (int i = 0; i < nvis; i++) workers.push_back(i);
    }
    const BatchIn in{chains, Ls, n_chains, limits, n_limits, slots, opts_or_default(opt), ops, ops_offsets, ops_caps};
    BatchOut out{costs, n_ops, status};
    if (P == 0) return ROTOR_OK;
    if (workers.empty()) {  // the current device, the caller's stream
        std::vector<int64_t> idx(P);
        std::iota(idx.begin(), idx.end(), 0);
        return batch_on_device(in, idx, kBatchKind, (cudaStream_t)stream, out);
    }
    // LPT over the workers by nominal transitions; one host thread per worker,
    // each with its own stream and (leased) workspace on its device
    std::vector<double> wgt(P);
    for (int64_t q = 0; q < P; q++) wgt[q] = rotor_transitions(Ls[q / n_limits], slots);
    std::vector<int32_t> part(P);
    rotor_partition_lpt(wgt.data(), (int32_t)P, (int32_t)workers.size(), part.data());
    std::vector<std::vector<int64_t>> idx(workers.size());
    for (int64_t q = 0; q < P; q++) idx[part[q]].push_back(q);
    std::vector<int> rc(workers.size(), ROTOR_OK);
    std::vector<std::string> msg(workers.size());
    std::vector<std::thread> th;
    for (size_t w = 0; w < workers.size(); w++) {
        th.emplace_back([&, w]() {
            if (idx[w].empty()) return;
            cudaStream_t st = nullptr;
            if (cudaSetDevice(workers[w]) != cudaSuccess ||
                cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
                rc[w] = fail(ROTOR_EDEVICE, "device %d: cannot create a stream", workers[w]);
            } else {
                rc[w] = batch_on_device(in, idx[w], kBatchKind + (int)w, st, out);
                cudaStreamDestroy(st);
            }
            if (rc[w]) msg[w] = g_err;
        });
    }
    for (auto &t : th) t.join();
    for (size_t w = 0; w < workers.size(); w++)
        if (rc[w]) return fail(rc[w], "device %d: %s", workers[w], msg[w].c_str());
    return ROTOR_OK;
}

int rotor_partition_lpt(const double *weights, int32_t n_items, int32_t n_parts, int32_t *part_of) {
    if (n_items < 0 || n_parts < 1 || (n_items > 0 && (!weights || !part_of)))
        return fail(ROTOR_EINPUT, "bad partition arguments");
    std::vector<int> idx(n_items);
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return weights[a] > weights[b]; });
    std::vector<double> load(n_parts, 0.0);
    for (int i : idx) {
        int best = 0;
        for (int q = 1; q < n_parts; q++)
            if (load[q] < load[best]) best = q;
        part_of[i] = best;
        load[best] += weights[i];
    }
    return ROTOR_OK;
}

int rotor_export_tables(double *C_host, uint16_t *D_host, int64_t n_values) {
    if (int r = check_last_alive()) return r;
    const Layout &y = g_last.y;
    const int64_t want = y.cells * (y.S + 1);
    if (n_values != want) return fail(ROTOR_EINPUT, "n_values %lld != %lld", (long long)n_values, (long long)want);
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (dev != g_last.device) CK(cudaSetDevice(g_last.device));
    CK(cudaStreamSynchronize(g_last.stream));
    const size_t row = (size_t)(y.S + 1);
    if (C_host)
        CK(cudaMemcpy2D(C_host, row * 8, g_last.p.C, (size_t)y.pitch * 8, row * 8, (size_t)y.cells,
                        cudaMemcpyDeviceToHost));
    if (D_host) {
        if (g_last.p.D) {
            CK(cudaMemcpy2D(D_host, row * 2, g_last.p.D, (size_t)y.pitch * 2, row * 2, (size_t)y.cells,
                            cudaMemcpyDeviceToHost));
        } else {
            uint16_t *tmp = nullptr;
            CK(cudaMalloc(&tmp, (size_t)y.cells * row * 2));
            for (int d = 0; d <= y.L; d++) rotor::launch_derive_argmin(g_last.p, d, tmp, (int64_t)row, 0);
            cudaError_t e = cudaGetLastError();
            if (e == cudaSuccess) e = cudaDeviceSynchronize();
            if (e == cudaSuccess) e = cudaMemcpy(D_host, tmp, (size_t)y.cells * row * 2, cudaMemcpyDeviceToHost);
            cudaFree(tmp);
            if (e != cudaSuccess) return fail(ROTOR_EDEVICE, "derive argmin: %s", cudaGetErrorString(e));
        }
    }
    if (dev != g_last.device) CK(cudaSetDevice(dev));
    return ROTOR_OK;
}

// ---- sharded single-table solve (one process per GPU; see include/rotor.h) ----
struct rotor_shard {
    Layout y;
    rotor::Problem p;
    rotor::TiledCtx ctx;
    int device;
    cudaStream_t stream;
    int64_t launches = 0;
};

int32_t rotor_tile_blocks(int32_t L) { return L < 1 ? 0 : rotor::tiled_nb(L + 1); }

int rotor_tile_bytes(int32_t slots, uint64_t *bytes) {
    if (slots < 1 || !bytes) return fail(ROTOR_EINPUT, "bad arguments");
    *bytes = rotor::tiled_tile_bytes(slots);
    return ROTOR_OK;
}

int rotor_sharded_begin(const rotor_chain *d_chain, int32_t L, uint64_t mem_limit, int32_t slots,
                        const rotor_options *opt, void *d_workspace, uint64_t workspace_bytes, void *stream,
                        rotor_shard **out) {
    if (!out) return fail(ROTOR_EINPUT, "out is NULL");
    *out = nullptr;
    int r = check_args(L, mem_limit, slots);
    if (r) return r;
    if (!d_chain || !d_chain->uf || !d_chain->ub || !d_chain->wx || !d_chain->wbx || !d_chain->wy || !d_chain->of ||
        !d_chain->ob)
        return fail(ROTOR_EINPUT, "chain has a NULL array");
    rotor_options o = opts_or_default(opt);
    o.kernel = ROTOR_KERNEL_TILED;
    o.keep_argmin = 0;
    Layout y = make_layout(L, slots, o);
    if (!d_workspace) return fail(ROTOR_EINPUT, "d_workspace is required");
    if (workspace_bytes < y.total)
        return fail(ROTOR_ENOMEM, "workspace too small: %llu < %zu", (unsigned long long)workspace_bytes, y.total);
    cudaStream_t st = (cudaStream_t)stream;
    rotor::Problem p = make_problem(y, (char *)d_workspace, o);
    rotor::launch_precompute(*d_chain, mem_limit, p, st);
    rotor::launch_leaf(p, st);
    CK(cudaGetLastError());
    rotor_shard *h = new rotor_shard();
    if (rotor::tiled_prepare(p, &h->ctx, st)) {
        delete h;
        return fail(ROTOR_EDEVICE, "tiled setup failed");
    }
    h->y = y;
    h->p = p;
    h->stream = st;
    h->launches = 2;  // precompute, leaf
    CK(cudaGetDevice(&h->device));
    *out = h;
    return ROTOR_OK;
}

int rotor_sharded_step(rotor_shard *h, int32_t delta, int32_t tile_lo, int32_t tile_hi, void *stream) {
    if (!h) return fail(ROTOR_EINPUT, "NULL shard handle");
    const int nb = rotor::tiled_nb(h->p.n);
    if (delta < 0 || delta >= nb || tile_lo < 0 || tile_hi > nb - delta || tile_lo > tile_hi)
        return fail(ROTOR_EINPUT, "bad tile range [%d,%d) at delta %d", tile_lo, tile_hi, delta);
    const int nl = rotor::tiled_delta(h->p, &h->ctx, delta, tile_lo, tile_hi, (cudaStream_t)stream);
    if (nl < 0) return fail(ROTOR_EDEVICE, "tiled step failed");
    h->launches += nl;
    CK(cudaGetLastError());
    return ROTOR_OK;
}

int rotor_sharded_pack(rotor_shard *h, int32_t delta, int32_t tile_lo, int32_t tile_hi, void *d_buf,
                       uint64_t buf_bytes, int32_t unpack, void *stream) {
    if (!h) return fail(ROTOR_EINPUT, "NULL shard handle");
    const int nb = rotor::tiled_nb(h->p.n);
    if (delta < 0 || delta >= nb || tile_lo < 0 || tile_hi > nb - delta || tile_lo > tile_hi || !d_buf)
        return fail(ROTOR_EINPUT, "bad pack arguments");
    if (buf_bytes < (uint64_t)(tile_hi - tile_lo) * rotor::tiled_tile_bytes(h->p.S))
        return fail(ROTOR_ENOMEM, "pack buffer too small");
    h->launches += rotor::tiled_pack(h->p, delta, tile_lo, tile_hi, (double *)d_buf, unpack ? 1 : 0,
                                     (cudaStream_t)stream);
    CK(cudaGetLastError());
    return ROTOR_OK;
}

int rotor_sharded_launches(const rotor_shard *h, int64_t *launches) {
    if (!h || !launches) return fail(ROTOR_EINPUT, "NULL argument");
    *launches = h->launches;
    return ROTOR_OK;
}

int rotor_sharded_free(rotor_shard *h) {
    delete h;
    return ROTOR_OK;
}

int rotor_sharded_finish(rotor_shard *h, void *stream, double *d_cost, rotor_op *d_ops, int64_t ops_cap,
                         int64_t *d_n_ops, int32_t *d_status) {
    if (!h) return fail(ROTOR_EINPUT, "NULL shard handle");
    if (!d_cost || !d_n_ops || !d_status || (ops_cap > 0 && !d_ops)) return fail(ROTOR_EINPUT, "bad outputs");
    g_last.valid = true;
    g_last.y = h->y;
    g_last.p = h->p;
    g_last.device = h->device;
    g_last.stream = (cudaStream_t)stream;
    g_last.profiled = false;
    g_last.counted = false;
    g_last.cache = nullptr;  // the caller owns this workspace
    rotor::Problem p = h->p;
    // the precompute wrote its status into the workspace's result slot: carry it over
    CK(cudaMemcpyAsync(d_status, p.res_status, 4, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    p.res_cost = d_cost;
    p.res_nops = d_n_ops;
    p.res_status = d_status;
    p.ops = d_ops;
    p.ops_cap = ops_cap < 0 ? 0 : ops_cap;
    rotor::launch_reconstruct(p, (cudaStream_t)stream);
    h->launches += 1;
    CK(cudaGetLastError());
    return ROTOR_OK;
}

// ---- one table sharded over a device list from one process (rotor_solve_sharded) ----
namespace {
// contiguous balanced ranges [lo, hi) of n items over k parts (the first n % k get one more)
void tile_ranges(int n, int k, std::vector<int> &lo, std::vector<int> &hi) {
    lo.resize(k);
    hi.resize(k);
    int a = 0;
    for (int r = 0; r < k; r++) {
        lo[r] = a;
        a += n / k + (r < n % k ? 1 : 0);
        hi[r] = a;
    }
}

struct ShardRank {
    int dev = 0;
    Lease lease;
    char *ws = nullptr;
    cudaStream_t st = nullptr;
    cudaEvent_t ev_step = nullptr, ev_pack = nullptr, ev_copied = nullptr;
    cudaStream_t xs = nullptr;         // exchange stream: this rank's receives of other ranks' tiles
    cudaEvent_t ev_recv = nullptr;     // recorded on xs after a diagonal's foreign tiles landed
    rotor::Problem p{};
    rotor::TiledCtx ctx{};
    double *send[2] = {nullptr, nullptr}, *recv = nullptr;
};

// host chain -> the staging area of a workspace (as rotor_solve_ex)
int stage_chain(const rotor_chain *chain, int L, const Layout &y, char *w, cudaStream_t st, rotor_chain &dch) {
    const size_t n1 = (size_t)L + 1;
    const size_t seg = al(((size_t)y.n + 2) * 8);
    char *stage = w + y.off_chain;
    dch.uf = (const double *)(stage + 0 * seg);
    dch.ub = (const double *)(stage + 1 * seg);
    dch.wx = (const uint64_t *)(stage + 2 * seg);
    dch.wbx = (const uint64_t *)(stage + 3 * seg);
    dch.wy = (const uint64_t *)(stage + 4 * seg);
    dch.of = (const uint64_t *)(stage + 5 * seg);
    dch.ob = (const uint64_t *)(stage + 6 * seg);
    CK(cudaMemcpyAsync((void *)dch.uf, chain->uf, n1 * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync((void *)dch.ub, chain->ub, n1 * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync((void *)dch.wx, chain->wx, n1 * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync((void *)dch.wbx, chain->wbx, n1 * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync((void *)dch.wy, chain->wy, (n1 + 1) * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync((void *)dch.of, chain->of, n1 * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync((void *)dch.ob, chain->ob, n1 * 8, cudaMemcpyHostToDevice, st));
    return ROTOR_OK;
}

int sharded_run(const rotor_chain *chain, int L, uint64_t M, int S, const rotor_options &o, std::vector<ShardRank> &rk,
                int halo_mode, double *cost_out, rotor_op *ops, int64_t ops_cap, int64_t *n_ops_out) {
    const int R = (int)rk.size();
    const Layout y = make_layout(L, S, o);
    const int nb = rotor::tiled_nb(y.n);
    const int cap = (nb + R - 1) / R;  // most tiles one rank computes on one tile diagonal
    const size_t tb = rotor::tiled_tile_bytes(S);
    const size_t stage_bytes = halo_mode == 0 && R > 1 ? 3 * cap * tb : 0;
    // per rank: device, leased workspace (+ the staging buffers of halo mode 0), stream, events, setup
    for (int r = 0; r < R; r++) {
        ShardRank &q = rk[r];
        CK(cudaSetDevice(q.dev));
        void *w = nullptr;
        int e = lease_workspace(kShardKind + r, y.total + stage_bytes, q.lease, &w);
        if (e) return e;
        q.ws = (char *)w;
        CK(cudaStreamCreateWithFlags(&q.st, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&q.ev_step, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&q.ev_pack, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&q.ev_copied, cudaEventDisableTiming));
        CK(cudaStreamCreateWithFlags(&q.xs, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&q.ev_recv, cudaEventDisableTiming));
        if (stage_bytes) {
            q.send[0] = (double *)(q.ws + y.total);
            q.send[1] = (double *)(q.ws + y.total + cap * tb);
            q.recv = (double *)(q.ws + y.total + 2 * cap * tb);
        }
        rotor_chain dch;
        if ((e = stage_chain(chain, L, y, q.ws, q.st, dch))) return e;
        q.p = make_problem(y, q.ws, o);
        rotor::launch_precompute(dch, M, q.p, q.st);
        rotor::launch_leaf(q.p, q.st);
        CK(cudaGetLastError());
        if (rotor::tiled_prepare(q.p, &q.ctx, q.st)) return fail(ROTOR_EDEVICE, "tiled setup failed on device %d", q.dev);
        CK(cudaEventRecord(q.ev_copied, q.st));
    }
    // Pipelined per tile diagonal: a rank first computes the tiles whose two
    // neighbours on the previous diagonal (tiles I and I+1) it computed itself
    // — they overlap the previous diagonal's exchange, which runs on the
    // rank's exchange stream xs — then waits for that exchange (ev_recv) and
    // computes its edge tiles.  Every tile reads whole rows / columns of the
    // diagonals before the previous one, which the wait of the previous
    // iteration ordered in (Theorem 1 reads strictly shorter intervals,
    // P:733-737; the same schedule as dist.solve_sharded).
    std::vector<int> lo, hi, plo, phi;
    NvtxRange nv_fill("rotor.sharded.fill");
    for (int delta = 0; delta < nb; delta++) {
        char nm[48];
        snprintf(nm, sizeof nm, "rotor.sharded.delta=%d", delta);
        NvtxRange nv_d(nm);
        tile_ranges(nb - delta, R, lo, hi);
        for (int r = 0; r < R; r++) {  // every rank: its share of the tiles of this diagonal
            ShardRank &q = rk[r];
            CK(cudaSetDevice(q.dev));
            int a = lo[r], b = hi[r];  // the local span
            if (delta > 0 && R > 1) {
                a = std::max(lo[r], plo[r]);
                b = std::min(hi[r], phi[r] - 1);
                if (a >= b) a = b = lo[r];
            }
            auto step = [&](int l, int h) -> int {
                if (h <= l) return ROTOR_OK;
                if (rotor::tiled_delta(q.p, &q.ctx, delta, l, h, q.st) < 0)
                    return fail(ROTOR_EDEVICE, "tiled step failed on device %d", q.dev);
                CK(cudaGetLastError());
                return ROTOR_OK;
            };
            int e = step(a, b);
            if (e) return e;
            if (delta > 0 && R > 1) CK(cudaStreamWaitEvent(q.st, q.ev_recv, 0));  // the previous diagonal's foreign tiles
            if ((e = step(lo[r], a)) || (e = step(std::max(b, lo[r]), hi[r]))) return e;
            CK(cudaEventRecord(q.ev_step, q.st));
        }
        plo = lo;
        phi = hi;
        if (R == 1) continue;
        if (halo_mode == 0) {  // pack -> peer copy -> unpack
            const int b = delta & 1;
            for (int r = 0; r < R; r++) {
                ShardRank &q = rk[r];
                if (hi[r] <= lo[r]) continue;
                CK(cudaSetDevice(q.dev));
                // send[b] was last read by the copies of delta - 2, which every
                // receiver's exchange stream ordered before its copies of delta - 1
                for (int x = 0; x < R; x++)
                    if (x != r) CK(cudaStreamWaitEvent(q.st, rk[x].ev_copied, 0));
                rotor::tiled_pack(q.p, delta, lo[r], hi[r], q.send[b], 0, q.st);
                CK(cudaGetLastError());
                CK(cudaEventRecord(q.ev_pack, q.st));
            }
            for (int r = 0; r < R; r++) {
                ShardRank &q = rk[r];
                CK(cudaSetDevice(q.dev));
                for (int x = 0; x < R; x++) {
                    if (x == r || hi[x] <= lo[x]) continue;
                    CK(cudaStreamWaitEvent(q.xs, rk[x].ev_pack, 0));
                    CK(cudaMemcpyPeerAsync(q.recv, q.dev, rk[x].send[b], rk[x].dev, (size_t)(hi[x] - lo[x]) * tb, q.xs));
                    rotor::tiled_pack(q.p, delta, lo[x], hi[x], q.recv, 1, q.xs);
                    CK(cudaGetLastError());
                }
                CK(cudaEventRecord(q.ev_copied, q.xs));
                CK(cudaEventRecord(q.ev_recv, q.xs));
            }
        } else {  // fused P2P halo: each rank pulls the owners' tiles through peer memory
            for (int r = 0; r < R; r++) {
                ShardRank &q = rk[r];
                CK(cudaSetDevice(q.dev));
                for (int x = 0; x < R; x++) {
                    if (x == r || hi[x] <= lo[x]) continue;
                    CK(cudaStreamWaitEvent(q.xs, rk[x].ev_step, 0));
                    rotor::tiled_pull(q.p, rk[x].p.C, delta, lo[x], hi[x], q.xs);
                    CK(cudaGetLastError());
                }
                CK(cudaEventRecord(q.ev_recv, q.xs));
            }
        }
    }
    for (int r = 0; r < R && R > 1; r++) {  // the last diagonal's exchange
        CK(cudaSetDevice(rk[r].dev));
        CK(cudaStreamWaitEvent(rk[r].st, rk[r].ev_recv, 0));
    }
    // Algorithm 2 on the first rank's complete table
    ShardRank &q0 = rk[0];
    CK(cudaSetDevice(q0.dev));
    rotor::launch_reconstruct(q0.p, q0.st);
    CK(cudaGetLastError());
    g_last.valid = true;
    g_last.y = y;
    g_last.p = q0.p;
    g_last.device = q0.dev;
    g_last.stream = q0.st;  // synchronised below; not used after the call
    g_last.profiled = false;
    g_last.counted = false;
    g_last.cache = q0.lease.e;
    g_last.cache_gen = q0.lease.e->gen.load();
    struct {
        double cost;
        int64_t nops;
        int32_t status;
    } res;
    CK(cudaMemcpyAsync(&res, q0.ws + y.off_res, 20, cudaMemcpyDeviceToHost, q0.st));
    for (int r = 0; r < R; r++) {
        CK(cudaSetDevice(rk[r].dev));
        CK(cudaStreamSynchronize(rk[r].st));
    }
    CK(cudaSetDevice(q0.dev));
    g_last.stream = nullptr;
    if (cost_out) *cost_out = res.cost;
    if (res.status == ROTOR_INFEASIBLE) {
        if (n_ops_out) *n_ops_out = 0;
        if (cost_out) *cost_out = INFINITY;
        return fail(ROTOR_INFEASIBLE, "infeasible: no persistent schedule within the memory limit");
    }
    if (res.status != ROTOR_OK && res.status != ROTOR_ETRUNC)
        return fail(res.status, "device phase failed with status %d", res.status);
    if (n_ops_out) *n_ops_out = res.nops;
    if (ops && ops_cap > 0 && res.nops > 0)
        CK(cudaMemcpy(ops, q0.ws + y.off_ops, (size_t)std::min<int64_t>(res.nops, ops_cap) * sizeof(rotor_op),
                      cudaMemcpyDeviceToHost));
    if (ops && res.nops > ops_cap)
        return fail(ROTOR_ETRUNC, "ops truncated: %lld > cap %lld", (long long)res.nops, (long long)ops_cap);
    return ROTOR_OK;
}
}  // namespace

int rotor_solve_sharded(const rotor_chain *chain, int32_t L, uint64_t mem_limit, int32_t slots,
                        const rotor_options *opt, const int32_t *devices, int32_t n_devices, int32_t halo_mode,
                        double *cost_out, rotor_op *ops, int64_t ops_cap, int64_t *n_ops_out) {
    int r = check_args(L, mem_limit, slots);
    if (r) return r;
    if ((r = check_host_chain(chain, L))) return r;
    if (halo_mode != 0 && halo_mode != 1) return fail(ROTOR_EINPUT, "halo_mode must be 0 or 1");
    int nvis = 0, dev0 = 0;
    CK(cudaGetDeviceCount(&nvis));
    CK(cudaGetDevice(&dev0));
    std::vector<int> devs;
    if (devices) {
        if (n_devices < 1) return fail(ROTOR_EINPUT, "n_devices must be >= 1 with a device list");
        for (int i = 0; i < n_devices; i++) {
            if (devices[i] < 0 || devices[i] >= nvis) return fail(ROTOR_EINPUT, "bad device %d", devices[i]);
            devs.push_back(devices[i]);
        }
    } else {
        const int k = n_devices < 0 ? nvis : n_devices;
        if (k < 1 || k > nvis) return fail(ROTOR_EINPUT, "n_devices %d with %d visible devices", n_devices, nvis);
        for (int i = 0; i < k; i++) devs.push_back(i);
    }
    // peer access between distinct devices (mode 1 needs it everywhere, else mode 0)
    for (size_t i = 0; i < devs.size(); i++)
        for (size_t j = 0; j < devs.size(); j++) {
            if (devs[i] == devs[j]) continue;
            int can = 0;
            CK(cudaDeviceCanAccessPeer(&can, devs[i], devs[j]));
            if (!can) {
                halo_mode = 0;
                continue;
            }
            CK(cudaSetDevice(devs[i]));
            cudaError_t e = cudaDeviceEnablePeerAccess(devs[j], 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            else if (e != cudaSuccess) {
                cudaSetDevice(dev0);
                return fail(ROTOR_EDEVICE, "peer access %d -> %d: %s", devs[i], devs[j], cudaGetErrorString(e));
            }
        }
    rotor_options o = opts_or_default(opt);
    o.kernel = ROTOR_KERNEL_TILED;
    o.keep_argmin = 0;
    o.counters = 0;
    o.profile = 0;
    std::vector<ShardRank> rk(devs.size());
    for (size_t i = 0; i < devs.size(); i++) rk[i].dev = devs[i];
    r = sharded_run(chain, L, mem_limit, slots, o, rk, halo_mode, cost_out, ops, ops_cap, n_ops_out);
    for (auto &q : rk) {  // on error too: wait for the work in flight, then free the streams / events
        cudaSetDevice(q.dev);
        if (q.st) cudaStreamSynchronize(q.st);
        if (q.ev_step) cudaEventDestroy(q.ev_step);
        if (q.ev_pack) cudaEventDestroy(q.ev_pack);
        if (q.ev_copied) cudaEventDestroy(q.ev_copied);
        if (q.xs) cudaStreamSynchronize(q.xs);
        if (q.ev_recv) cudaEventDestroy(q.ev_recv);
        if (q.xs) cudaStreamDestroy(q.xs);
        if (q.st) cudaStreamDestroy(q.st);
    }
    cudaSetDevice(dev0);
    return r;
}

int rotor_export_rows(const int32_t *s, const int32_t *t, int64_t n_rows, double *C_host) {
    if (int r = check_last_alive()) return r;
    if (n_rows < 0 || (n_rows > 0 && (!s || !t || !C_host))) return fail(ROTOR_EINPUT, "bad export_rows arguments");
    const Layout &y = g_last.y;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (dev != g_last.device) CK(cudaSetDevice(g_last.device));
    CK(cudaStreamSynchronize(g_last.stream));
    const size_t row = (size_t)(y.S + 1);
    for (int64_t r = 0; r < n_rows; r++)
        if (s[r] < 1 || t[r] < s[r] || t[r] > y.n) return fail(ROTOR_EINPUT, "bad cell (%d,%d)", s[r], t[r]);
    // runs of consecutive cells (e.g. (s, t..t+k) in the s-major order) go in one 2-D copy
    for (int64_t r = 0; r < n_rows;) {
        const int64_t c0 = rotor::cell_index(y.n, s[r], t[r]);
        int64_t k = 1;
        while (r + k < n_rows && rotor::cell_index(y.n, s[r + k], t[r + k]) == c0 + k) k++;
        CK(cudaMemcpy2D(C_host + r * row, row * 8, g_last.p.C + c0 * y.pitch, (size_t)y.pitch * 8, row * 8,
                        (size_t)k, cudaMemcpyDeviceToHost));
        r += k;
    }
    if (dev != g_last.device) CK(cudaSetDevice(dev));
    return ROTOR_OK;
}

int rotor_last_timings(rotor_timings *out) {
    if (!out) return fail(ROTOR_EINPUT, "out is NULL");
    if (int r = check_last_alive()) return r;
    if (!g_last.profiled) return fail(ROTOR_EINPUT, "last solve was not profiled");
    CK(cudaEventSynchronize(g_last.ev[3]));
    float a = 0, b = 0, c = 0;
    CK(cudaEventElapsedTime(&a, g_last.ev[0], g_last.ev[1]));
    CK(cudaEventElapsedTime(&b, g_last.ev[1], g_last.ev[2]));
    CK(cudaEventElapsedTime(&c, g_last.ev[2], g_last.ev[3]));
    out->pre_ms = a;
    out->fill_ms = b;
    out->reconstruct_ms = c;
    out->fill_launches = g_last.fill_launches;
    out->total_launches = g_last.total_launches;
    double mid = 0;
    for (int i = 0; i < g_last.mid_n; i++) {
        float x = 0;
        CK(cudaEventElapsedTime(&x, g_last.mid_ev[2 * i], g_last.mid_ev[2 * i + 1]));
        mid += x;
    }
    out->middle_ms = mid;
    out->middle_launches = g_last.mid_n;
    return ROTOR_OK;
}

int rotor_last_counters(rotor_counters *out) {
    if (!out) return fail(ROTOR_EINPUT, "out is NULL");
    if (int r = check_last_alive()) return r;
    if (!g_last.counted) return fail(ROTOR_EINPUT, "last solve did not count (options.counters)");
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (dev != g_last.device) CK(cudaSetDevice(g_last.device));
    unsigned long long c[32];
    CK(cudaStreamSynchronize(g_last.stream));
    CK(cudaMemcpy(c, g_last.p.counters, sizeof c, cudaMemcpyDeviceToHost));
    if (dev != g_last.device) CK(cudaSetDevice(dev));
    const Layout &y = g_last.y;
    out->nominal = rotor_transitions(y.L, y.S);
    out->middle_nominal = (double)rotor::tiled_middle_candidates(y.n) * (y.S + 1);
    out->dependent_nominal = out->nominal - out->middle_nominal;
    out->middle_split_visits = c[0];
    out->coarse_pass = c[1];
    out->quadrant_compares = c[2];
    out->exact_splits = c[3];
    out->evaluated = 512.0 * (double)c[2] + 2048.0 * (double)c[3] + out->dependent_nominal;
    out->middle_wait_cycles = c[4];
    out->middle_init_cycles = c[5];
    out->middle_loop_cycles = c[6];
    out->middle_flush_cycles = c[7];
    unsigned long long mx = 0, sum = 0;
    for (int w = 0; w < 16; w++) {
        mx = std::max(mx, c[8 + w]);
        sum += c[8 + w];
        out->middle_slot_cycles[w] = c[8 + w];
    }
    out->middle_warp_imbalance = sum ? mx * 16.0 / (double)sum : 0.0;
    out->leaf_ctas = c[24];
    out->leaf_setup_ns = c[25];
    out->leaf_wait_ns = c[26];
    out->leaf_work_ns = c[27];
    out->leaf_sync_ns = c[28];
    out->leaf_pass1_ns = c[29];
    return ROTOR_OK;
}

int rotor_release(void) {
    std::lock_guard<std::mutex> g(g_cache_mu);
    int dev0 = 0;
    cudaGetDevice(&dev0);
    for (auto &kv : g_cache) {
        CacheEntry *e = kv.second.get();
        std::lock_guard<std::mutex> lk(e->mu);  // waits for a call still using it
        if (e->ptr) {
            cudaSetDevice(kv.first.first);
            cudaDeviceSynchronize();
            cudaFree(e->ptr);
            e->ptr = nullptr;
            e->bytes = 0;
        }
        e->gen++;  // invalidates every last-solve record pointing at it
    }
    cudaSetDevice(dev0);
    g_last.valid = false;
    return ROTOR_OK;
}

}  // extern "C"
