// Tiled fill of the Theorem-1 table — the fast path.
//
// The split candidates of a cell (s,t) are
//     cand(s') = fl( A(s, s'-1, m) + C(s', t, m - wx[s'-1]) ),  s' = s+1..t,
// with A(s,c,m) = fl( fl(P[c] - P[s-1]) + C(s,c,m) ) stored (column-major,
// a_index) when a cell is finalised (Q12 association: fl(fl(U + pre) + suf)).
// For a fixed m this is a min-plus product over s' (the m-shift depends on s'
// only), so the triangle is cut into TB x TB tiles of (s,t), processed by tile
// diagonal Delta = J - I.  For a tile (I,J):
//   * middle (Delta >= 2): s' in blocks I+1..J-1 — every operand is final: a
//     dense min-plus product with TB-fold operand reuse, operands streamed by
//     TMA into shared memory through a full/empty mbarrier ring (k_tile_middle);
//   * dependent: s' in [s+1, i1-1] (C operand in this tile, rows below) and
//     [j0, t] (A operand in this tile, same row), the gates, F_all, and the
//     writes of C and A — a second tiling level of SB x SB sub-tiles
//     (rotor_tiled_dep.cuh): sub-products with SB-fold reuse, then short
//     row-by-row leaves; a row only needs rows below at (shifted) lower m,
//     which are complete, and its own earlier columns at the same m.
// Delta = 1 has no middle; Delta = 0 (diagonal tiles) is a local triangle.
// The min is exact and every candidate has the fixed association above, so the
// table is bit-identical to the wavefront / oracle fill (order-independent).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>
#include <limits.h>

#include <chrono>
#include <map>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "rotor_common.cuh"
#include "rotor_kernels.cuh"

namespace rotor {
namespace tiled {

constexpr int TB = 32;      // tile edge in stages
static_assert(TB == kTB, "the shadow layout's block edge is the tile edge");
constexpr int KC = 8;       // splits per pipeline stage
constexpr int TM = 16;      // m values per CTA (middle kernel)
constexpr int STAGES = 3;   // TMA pipeline depth (2 stages in flight while one is consumed)
// Ring geometry measured at config 4 (same 209 KB of shared memory): KC x STAGES
// = 8 x 3: 268 ms per solve, 4 x 6: 282 ms, 2 x 12: 299 ms — fewer, larger
// stages amortise the per-stage barrier wait / arrive / refill.
constexpr int CONSUMERS = 512;  // 16 warps: two per scheduler slot more than 8 hide the DADD->DSETP->FSEL chain
constexpr int THREADS = CONSUMERS;
// Register tile (s x t) per consumer thread (<= 128 registers).  8 x 4 rather
// than 4 x 8: the two half-warps (adjacent t groups) share the 8 A values, so
// an A load is one shared-memory wavefront and only the 4 C loads are two
// (16 wavefronts per split instead of 20): 217.2 vs 222.0 ms per solve.
constexpr int RS = 8, RT = 4;
static_assert((TB / RS) * (TB / RT) * TM == CONSUMERS, "one thread per (m, register tile)");
// A TMA box must start on a 16-byte boundary of the row (an odd fp64 start
// column faults with "illegal instruction", scripts/tma_probe.cu): the shifted
// C boxes start at the even column below the wanted one and are TMB = TM + 2
// wide; the consumer adds the per-row offset (0 or 1).
constexpr int TMB = TM + 2;
constexpr int A_STAGE = KC * TB * TM;   // doubles [KC][TB s][TM]
constexpr int B_STAGE = KC * TB * TMB;  // doubles [KC][TB t][TMB]
constexpr size_t SMEM_BYTES = (size_t)STAGES * (A_STAGE + B_STAGE) * 8 + 2 * STAGES * 8 + STAGES * KC * 4 + 64;
// The rest of the 227 KB holds a copy of wx (the producer's shift lookups stay
// on chip: a global load there delays every refill by a memory round trip).
constexpr int WX_SMEM_MAX = (int)((226 * 1024 - SMEM_BYTES) / 4);  // 1 KB kept for the static/system share
constexpr size_t ring_bytes(int kc, int stages) {
    return (size_t)stages * kc * TB * (TM + TMB) * 8 + 2 * stages * 8 + stages * kc * 4 + 64;
}
static_assert(ring_bytes(KC, STAGES) == SMEM_BYTES, "ring size");

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// (x0 + y0, x1 + y1) rounded toward -inf, as one packed FADD2.RM (sm_100)
__device__ __forceinline__ float2 fadd2_rd(float2 x, float2 y) {
    unsigned long long r;
    asm("add.rm.f32x2 %0, %1, %2;"
        : "=l"(r)
        : "l"(*reinterpret_cast<unsigned long long *>(&x)), "l"(*reinterpret_cast<unsigned long long *>(&y)));
    return *reinterpret_cast<float2 *>(&r);
}

// non-blocking: true once the phase with this parity has completed (acquire)
__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap *map, int c0, int c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1)
                 : "memory");
}

__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }

// The same exact min on the integer pipe: non-negative doubles (every
// candidate, Q13) order like their int64 bit patterns.  DSETP runs at half the
// DADD rate, so routing a share of the mins through ISETP/SEL looked like a way
// to balance the fp64 and ALU pipes — measured slower on B200 (mixed 17.0 vs
// 18.3 transitions/clk/SM, scripts/microbench_minplus.cu), so it is off.
__device__ __forceinline__ double imin(double a, double b) {
    const long long x = __double_as_longlong(a), y = __double_as_longlong(b);
    return __longlong_as_double(y < x ? y : x);
}
constexpr int INT_MIN_COLS = 0;  // register-tile columns j >= RT - INT_MIN_COLS use imin

// ---------------------------------------------------------------------------
// Middle phase of tile diagonal delta >= 2: partial(s,t,m) = min over s' in
// blocks I+1..J-1 of A(s,s'-1,m) + C(s',t,m-wx[s'-1]); written into C.
// Persistent: one CTA per SM walks the work items (tile, 16-m chunk)
// blockIdx.x, +gridDim.x, ...; the TMA ring runs across item boundaries, so
// the loads of the next item overlap the epilogue of the current one.
// 16 warps (thread = one m, a 4x8 (s,t) register tile); thread 0 also issues
// the 2*KC TMA boxes of each stage (full/empty mbarrier ring).
// ---------------------------------------------------------------------------
// The middle's per-(tile row I, 32-m chunk, warp) fired-split lists, read by
// the sub-product of the dependent phase (the warp's 8 x 8 cells are exactly
// one dependent-phase sub-tile): [0] = count, or MLIST_OVERFLOW when the
// middle evaluated its splits itself and wrote the exact partial; [1..count] =
// split index f (s' = i0 + TB + f).  Per tile ROW: the tiles of one row run
// in order (DAG: one stream per row; diagonal schedule: diagonal by diagonal).
constexpr int MLIST_STRIDE = 32, MLIST_CAP = MLIST_STRIDE - 1;
constexpr uint16_t MLIST_OVERFLOW = 0xFFFF;
__host__ __device__ inline int n_mc32(int S) { return (S + 1 + kSW - 1) / kSW; }
__host__ __device__ inline int64_t mlist_index(int n_mc, int I, int q, int w) {
    return (((int64_t)I * n_mc + q) * (CONSUMERS / 32) + w) * MLIST_STRIDE;
}
inline size_t mlist_bytes(int L, int S) {
    return (size_t)((L + 1 + TB - 1) / TB) * n_mc32(S) * (CONSUMERS / 32) * MLIST_STRIDE * sizeof(uint16_t);
}

template <int KC_, int STAGES_>
__global__ void __launch_bounds__(THREADS, 1)
    k_tile_middle(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmC, Problem p,
                  int delta, int tile_lo, int n_tiles) {
    constexpr int KC = KC_, STAGES = STAGES_;  // ring geometry (KC splits per stage)
    constexpr int A_STAGE = KC * TB * TM, B_STAGE = KC * TB * TMB;
    extern __shared__ __align__(1024) double smem[];  // no static smem: the dynamic base is aligned
    double *As = smem;                     // [STAGES][KC][TB][TM]
    double *Bs = smem + STAGES * A_STAGE;  // [STAGES][KC][TB][TMB]
    uint64_t *full = reinterpret_cast<uint64_t *>(Bs + STAGES * B_STAGE);
    uint64_t *empty = full + STAGES;
    int *soff = reinterpret_cast<int *>(empty + STAGES);  // [STAGES][KC] column offset of each C box
    int *wx_s = soff + STAGES * KC;                       // wx[0..n) when n <= WX_SMEM_MAX

    const int n = p.n;
    const int n_mc = (p.S + 1 + TM - 1) / TM;
    const int n_items = n_tiles * n_mc;
    if ((int)blockIdx.x >= n_items) return;
    const int my_items = (n_items - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
    const int iters = (delta - 1) * TB / KC;
    const int total = my_items * iters;
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int *wxp = p.wx;
    if (n <= WX_SMEM_MAX) {  // ordered before the producer's first use by the __syncthreads below
        for (int i = tid; i < n; i += THREADS) wx_s[i] = p.wx[i];
        wxp = wx_s;
    }

    // TMA producer (no dedicated warp: 16 warps x 128 registers already fill
    // the register file).  Step gi of this CTA's (item, k-step) sequence loads,
    // for k < KC: A cells (i0..i0+TB-1, c = sp0+k-1) and C cells
    // (sp = sp0+k, j0..j0+TB-1) at m - wx[sp-1].  A C window starting below
    // -kPad lies wholly under m = wx[sp-1] <= m_null(s,t): every cell it feeds
    // is gated and the clamped values are never used (DESIGN Q6).
    auto step_coords = [&](int gi, int &m0, int &i0, int &j0, int &sp0) {
        const int item = (int)blockIdx.x + (gi / iters) * (int)gridDim.x;
        const int I = tile_lo + item / n_mc, J = I + delta;
        i0 = I * TB + 1;
        j0 = J * TB + 1;
        m0 = (item % n_mc) * TM;
        sp0 = i0 + TB + (gi % iters) * KC;
    };
    auto issue = [&](int gi) {
        const int st = gi % STAGES;
        int m0, i0, j0, sp0;
        step_coords(gi, m0, i0, j0, sp0);
        // column offsets first: the expect_tx arrive (release) orders them
        // before the consumers' full-barrier wait (acquire)
        for (int k = 0; k < KC; k++) soff[st * KC + k] = (max(m0 - wxp[sp0 + k - 1], -kPad) + kPad) & 1;
        mbar_expect_tx(&full[st], (uint32_t)((A_STAGE + B_STAGE) * 8));
        for (int k = 0; k < KC; k++)
            tma_load_2d(As + st * A_STAGE + k * TB * TM, &tmA, m0 + kPad, (int)a_index(i0, sp0 + k - 1), &full[st]);
        for (int k = 0; k < KC; k++) {
            const int sp = sp0 + k;
            const int c0 = max(m0 - wxp[sp - 1], -kPad) + kPad;
            tma_load_2d(Bs + st * B_STAGE + k * TB * TMB, &tmC, c0 & ~1, (int)cell_index(n, sp, j0), &full[st]);
        }
        // (an L2 prefetch of later steps' boxes, cp.async.bulk.prefetch.tensor,
        // measured slower: 1 or 2 steps ahead 296 vs 265 ms of fill, 6 steps
        // ahead with the 4 x 6 ring 204 vs 164 ms of middle time — not used;
        // so was a non-blocking "lazy" refill by the producer lane, 293 vs 288,
        // and prefetch.global.L2 of the boxes 4-7 steps ahead spread over all
        // 512 threads, 247-251 vs 234 ms of fill)
    };

    if (tid == 0) {
        for (int s = 0; s < STAGES; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CONSUMERS / 32);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    // The producer is lane 0 of the LAST warp: the warp scheduler favours the
    // highest warp id, so the refills are not delayed behind the consumers
    // (with warp 0 as producer ~19% of the warp time was spent waiting for
    // TMA data, profiles/r01_tiled_v4.md).  A dedicated 17th producer warp does
    // not fit: the register file is split per scheduler (16 K registers each),
    // and 5 warps on one scheduler cap every thread at 96 registers.
    constexpr int PRODUCER = CONSUMERS - 32;
    if (tid == PRODUCER)
        for (int gi = 0; gi < STAGES && gi < total; gi++) issue(gi);

    const int mi = tid & 15;
    const int g = tid >> 4;
    const int sg = g / (TB / RT), tg = g % (TB / RT);  // register-tile row / column group
    for (int kl = 0; kl < my_items; kl++) {
    double acc[RS][RT];
#pragma unroll
    for (int i = 0; i < RS; i++)
#pragma unroll
        for (int j = 0; j < RT; j++) acc[i][j] = INFINITY;

    for (int it = 0; it < iters; it++) {
        const int gi = kl * iters + it;
        const int st = gi % STAGES;
        mbar_wait(&full[st], (uint32_t)((gi / STAGES) & 1));
        const double *a_s = As + st * A_STAGE + (sg * RS) * TM + mi;
        const double *b_s = Bs + st * B_STAGE + (tg * RT) * TMB + mi;
#pragma unroll
        for (int k = 0; k < KC; k++) {
            double a[RS], b[RT];
            const double *bk = b_s + k * TB * TMB + soff[st * KC + k];
#pragma unroll
            for (int i = 0; i < RS; i++) a[i] = a_s[k * TB * TM + i * TM];
#pragma unroll
            for (int j = 0; j < RT; j++) b[j] = bk[j * TMB];
#pragma unroll
            for (int i = 0; i < RS; i++)
#pragma unroll
                for (int j = 0; j < RT; j++)
                    acc[i][j] = (j >= RT - INT_MIN_COLS) ? imin(acc[i][j], __dadd_rn(a[i], b[j]))
                                                         : dmin(acc[i][j], __dadd_rn(a[i], b[j]));
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);  // this warp is done reading stage st
        if (tid == PRODUCER && gi + STAGES < total) {  // refill st once every warp released it
            mbar_wait(&empty[st], (uint32_t)((gi / STAGES) & 1));
            issue(gi + STAGES);
        }
    }

    const int item = (int)blockIdx.x + kl * (int)gridDim.x;
    const int I = tile_lo + item / n_mc, J = I + delta;
    const int i0 = I * TB + 1, j0 = J * TB + 1;
    const int m = (item % n_mc) * TM + mi;
    // the partials below are final for the middle range: tell the sub-product
    // (fired-split lists of the pruned kernel) to read them
    if (tid < CONSUMERS / 32) p.mlist[mlist_index(n_mc32(p.S), I, (item % n_mc) * TM / kSW, tid)] = MLIST_OVERFLOW;
    if (m <= p.S) {
#pragma unroll
        for (int i = 0; i < RS; i++) {
            const int s = i0 + sg * RS + i;
#pragma unroll
            for (int j = 0; j < RT; j++) {
                const int t = j0 + tg * RT + j;
                if (t <= n) p.C[cell_index(n, s, t) * p.pitch + m] = acc[i][j];
            }
        }
    }
    }  // items
}

// ---------------------------------------------------------------------------
// Pruned middle (the default, DESIGN 5.2): items of 32 s x 32 t x 32 m; a warp
// = 32 consecutive m of one 8 x 8 (s,t) register tile.  The operands stream as
// fp32 round-down shadows: per split s' one A box A32(i0..i0+31, s'-1, m0..+31)
// and one C box C32(s', j0..j0+31, m0..+31), where C32 is stored pre-shifted by
// wx[s'-1] (store_final_c), so both boxes are 32 consecutive rows x the same
// aligned 32 m — in the m-chunked shadow layout (shadow_index) one contiguous
// 4 KB block each, moved by one bulk copy (cp.async.bulk) into a full/empty
// mbarrier ring.  Each lane keeps only bestf (>= the exact partial minimum)
// for its 64 cells.  Per split: a coarse bound for the whole 8 x 8 tile, then
// per 4 x 4 quadrant, then the per-cell filter fadd_rd(a32, b32) < bestf; the
// splits that can still improve some cell of the warp (mask OR-reduced over
// the warp) are recomputed exactly from the fp64 tables and folded into the
// partial rows of C: the first candidate of a cell is stored, later ones go in
// with a 64-bit atomic min, and the cells that never fired get +inf at the end
// of the item (every partial is written once, no read back).
// ---------------------------------------------------------------------------
constexpr int TMW = kSW, RW = 8;
constexpr int BOX = TB * TMW;                    // floats per operand box (4 KB)
constexpr int FMAX_CAP = 2048;                   // fired splits a warp can record per item (see fmax)


// Exact pass of a warp over the splits it recorded for one item: s' = sp_lo +
// flist[f], f < nf — or, if the list overflowed (nf > fmax), every split
// sp_lo .. sp_lo + n_all - 1.  Every cell's candidates fl(A(s, s'-1, m) +
// C(s', t, m - wx[s'-1])) (Q12) from the fp64 tables are min-ed and the
// partial is stored once (+inf if no candidate).  Each (s, t, m) partial
// belongs to exactly one lane, so nothing is atomic.  Rows in pairs keep the
// running minima in 32 registers.
__device__ __forceinline__ void exact_flush(const Problem &p, const uint16_t *flist, int nf, int fmax, int sp_lo,
                                            int n_all, int s_0, int t_0, int ss, int m, int mc, const int *wxp) {
    // cells (s_0 + ss*i, t_0 + ss*j), i, j < RW
    constexpr int RW = 8, RH = 2, FC = 3;  // rows per pass, splits whose loads are in flight together
    const int n = p.n;
    if (m > p.S) return;
    const bool all = nf > fmax;
    const int cnt = all ? n_all : nf;
    const int64_t sp_pitch = (int64_t)ss * p.pitch;
#pragma unroll 1
    for (int h = 0; h < RW / RH; h++) {
        double acc[RH][RW];
#pragma unroll
        for (int i = 0; i < RH; i++)
#pragma unroll
            for (int j = 0; j < RW; j++) acc[i][j] = INFINITY;
#pragma unroll 1
        for (int f0 = 0; f0 < cnt; f0 += FC) {
            double ad[FC][RH], bd[FC][RW];
#pragma unroll
            for (int u = 0; u < FC; u++) {  // all loads of FC splits first (one memory round trip)
                const bool live = f0 + u < cnt;
                const int sp = sp_lo + (live ? (all ? f0 + u : (int)flist[f0 + u]) : 0);
                const int mm = live ? mc - wxp[sp - 1] : -1;
                // A(s, sp-1): consecutive s are consecutive rows (a_index); C(sp, t): consecutive t too
                const double *ap = p.A + a_index(s_0 + ss * RH * h, live ? sp - 1 : s_0) * p.pitch + mc;
                const double *bp = p.C + cell_index(n, live ? sp : s_0, min(t_0, n)) * p.pitch + mm;
#pragma unroll
                for (int i = 0; i < RH; i++) ad[u][i] = live ? __ldcg(ap + i * sp_pitch) : INFINITY;
#pragma unroll
                for (int j = 0; j < RW; j++)
                    bd[u][j] = (mm >= 0 && t_0 + ss * j <= n) ? __ldcg(bp + j * sp_pitch) : INFINITY;
            }
#pragma unroll
            for (int u = 0; u < FC; u++)
#pragma unroll
                for (int i = 0; i < RH; i++)
#pragma unroll
                    for (int j = 0; j < RW; j++) acc[i][j] = dmin(acc[i][j], __dadd_rn(ad[u][i], bd[u][j]));
        }
#pragma unroll
        for (int i = 0; i < RH; i++) {
            double *crow = p.C + cell_index(n, s_0 + ss * (RH * h + i), min(t_0, n)) * p.pitch + m;
#pragma unroll
            for (int j = 0; j < RW; j++)
                if (t_0 + ss * j <= n) crow[j * sp_pitch] = acc[i][j];
        }
    }
}

constexpr int SBOX = kSR * TMW;  // floats per split and operand: 32 cell rows + 8 quad-minima rows (5 KB)
template <int KC_, int STAGES_>
struct WideRing {
    static constexpr int KC = KC_, STAGES = STAGES_;
    static constexpr int NB = 2;  // bulk copies per stage: the KC splits' A rows, then their C rows
    // floats per stage: [A: KC][kSR rows][TMW], [C: KC][kSR rows][TMW]
    static constexpr int ST = 2 * KC * SBOX;
    // + the fired-split lists: NWARPS x fmax uint16 (wide_list_bytes)
    static constexpr size_t bytes =
        (size_t)STAGES * ST * 4 + 2 * STAGES * 8 + (size_t)STAGES * NB * 8 + 2 * STAGES * 4 + 64;
};
// fired-split list length per warp: every split of the longest item
// ((nb - 2) * TB), capped by FMAX_CAP and by the shared memory left next to
// the ring and wx (a longer list overflows into an all-splits exact pass)
inline int wide_fmax(int n, size_t ring_bytes) {
    const size_t wx_b = n <= 4096 ? (size_t)n * 4 : 0;
    const int room = (int)((227 * 1024 - ring_bytes - wx_b) / ((CONSUMERS / 32) * 2)) & ~7;
    return max(8, min(min(FMAX_CAP, room), max(1, ((n + TB - 1) / TB - 2) * TB)));
}
constexpr int WKC = 8, WSTAGES = 2;  // ring of the wide middle (see tiled_delta)
constexpr int WIDE_WX_MAX = 4096;  // wx staged in shared memory up to this n (wide_fmax agrees)
__host__ __device__ inline bool n_wx_smem(int n) { return n <= WIDE_WX_MAX; }
static_assert((TB / RW) * (TB / RW) * TMW == THREADS, "one lane per (m, 8x8 tile)");

__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// profile counters (Problem::counters, rotor_counters order)
// (COUNT also sums per-warp clock cycles: waiting for stage data, item setup
// (bestf init), filter loop, exact pass)
enum { CTR_SPLITS = 0, CTR_COARSE_PASS = 1, CTR_QUADS = 2, CTR_EXACT = 3, CTR_WAIT = 4, CTR_INIT = 5, CTR_LOOP = 6,
       CTR_FLUSH = 7, CTR_N = 8 };

template <int KCW, int STG, bool COUNT>
__global__ void __launch_bounds__(THREADS, 1)
    k_tile_middle_wide(Problem p, int delta, int tile_lo, int n_tiles, int coarse, int fmax) {
    using R = WideRing<KCW, STG>;
    constexpr int KC = R::KC, STAGES = R::STAGES, ST = R::ST, NB = R::NB;
    constexpr int NWARPS = CONSUMERS / 32;
    extern __shared__ __align__(1024) float fsm[];
    float *ring = fsm;  // [STAGES][A: KC][TB s][TMW] [C: KC][TB t][TMW]
    uint64_t *full = reinterpret_cast<uint64_t *>(ring + STAGES * ST);
    uint64_t *empty = full + STAGES;
    const float **src = reinterpret_cast<const float **>(empty + STAGES);  // [STAGES][NB] next refill's boxes
    int *claim = reinterpret_cast<int *>(src + STAGES * NB);  // step whose refill of the stage is unclaimed
    int *prep = claim + STAGES;                                   // step whose refill addresses are not yet computed
    int *wx_s = prep + STAGES;                                    // wx[0..n) when n <= WIDE_WX_MAX
    uint16_t *fl_s = reinterpret_cast<uint16_t *>(wx_s + (n_wx_smem(p.n) ? p.n : 0));  // [NWARPS][fmax]

    const int n = p.n;
    const int n_mc = (p.S + 1 + TMW - 1) / TMW;
    const int n_items = n_tiles * n_mc;
    if ((int)blockIdx.x >= n_items) return;
    const int my_items = (n_items - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
    const int iters = (delta - 1) * TB / KC;
    const int total = my_items * iters;
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int *wxp = p.wx;
    if (n_wx_smem(n)) {
        for (int i = tid; i < n; i += THREADS) wx_s[i] = p.wx[i];
        wxp = wx_s;
    }
    auto coords = [&](int gi, int &i0, int &j0, int &m0, int &sp0) {
        const int item = (int)blockIdx.x + (gi / iters) * (int)gridDim.x;
        const int I = tile_lo + item / n_mc, J = I + delta;
        i0 = I * TB + 1;
        j0 = J * TB + 1;
        m0 = (item % n_mc) * TMW;
        sp0 = i0 + TB + (gi % iters) * KC;
    };
    // box 0 of a stage: the A32 rows (block I, columns sp0 - 1 .. sp0 + KC - 2),
    // box 1: the C32 rows (block J, rows sp0 .. sp0 + KC - 1) — each split's 32
    // cells + 8 quad minima, and the KC splits consecutive (srow_a / srow_c):
    // one contiguous block each
    auto box_src = [&](int b, int i0, int j0, int m0, int sp0) -> const float * {
        return b == 0 ? p.A32 + shadow_index(p.sarows, sa_col(n, (i0 - 1) / TB, sp0 - 1), m0)
                      : p.C32 + shadow_index(p.scrows, sc_row((j0 - 1) / TB, sp0), m0);
    };
    constexpr uint32_t box_bytes = KC * SBOX * 4;
    auto issue = [&](int gi) {
        const int st = gi % STAGES;
        int i0, j0, m0, sp0;
        coords(gi, i0, j0, m0, sp0);
        mbar_expect_tx(&full[st], (uint32_t)(ST * 4));
        float *dst = ring + st * ST;
        for (int b = 0; b < NB; b++) bulk_load(dst + b * KC * SBOX, box_src(b, i0, j0, m0, sp0), box_bytes, &full[st]);
    };
    // Refills are split in two: the FIRST warp to finish reading a stage
    // computes the source addresses of its next refill (one box per lane,
    // lane < NB) into shared memory; the LAST one issues the copies from
    // them.  The last arriver is the slowest warp; with the whole refill on it
    // (coordinates, 64-bit address arithmetic, copies) it had stayed the
    // slowest for good (the issuing warp at ~1.23x the others' loop cycles).
    // Still true with two copies per stage: the last arriver computing its two
    // addresses itself measured 48.6 vs 46.9 ms of middle per solve.
    static_assert(NB <= 32, "one box per lane");
    auto prepare_warp = [&](int gi, int ln) {  // addresses of step gi's boxes
        int i0, j0, m0, sp0;
        coords(gi, i0, j0, m0, sp0);
        if (ln < NB) src[(gi % STAGES) * NB + ln] = box_src(ln, i0, j0, m0, sp0);
    };
    auto issue_warp = [&](int gi, int ln) {  // lane 0 posts the expected bytes first
        const int st = gi % STAGES;
        if (ln == 0) mbar_expect_tx(&full[st], (uint32_t)(ST * 4));
        __syncwarp();
        if (ln < NB) bulk_load(ring + st * ST + ln * KC * SBOX, src[st * NB + ln], box_bytes, &full[st]);
    };
    if (tid == 0) {
        for (int s = 0; s < STAGES; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CONSUMERS);
            claim[s] = s;
            prep[s] = s;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0)
        for (int gi = 0; gi < STAGES && gi < total; gi++) issue(gi);
    __syncwarp();

    unsigned c_coarse = 0, c_quads = 0, c_exact = 0;  // profile counters (warp-uniform, COUNT only)
    unsigned long long c_wait = 0, c_init = 0, c_loop = 0, c_flush = 0, t_mark = COUNT ? clock64() : 0;
    auto lap = [&](unsigned long long &acc) {
        if (COUNT) {
            const unsigned long long t = clock64();
            acc += t - t_mark;
            t_mark = t;
        }
    };
    const int sg = warp / (TB / RW), tg = warp % (TB / RW);
    uint16_t *flist = fl_s + warp * fmax;  // this warp's fired splits of the current item (s' - sp_lo)
    for (int kl = 0; kl < my_items; kl++) {
        const int item = (int)blockIdx.x + kl * (int)gridDim.x;
        const int I = tile_lo + item / n_mc, J = I + delta;
        // the warp's 8 x 8 cells (s_0 + i, t_0 + j): one contiguous sub-tile = two
        // row groups x two column groups of the quad minima (a warp's cells spread
        // over the tile balanced the warps' work but made the coarse test 2.5x
        // weaker: 81.7 vs 67.4 ms of middle, removed)
        const int s_0 = I * TB + 1 + sg * RW, t_0 = J * TB + 1 + tg * RW;
        const int m = (item % n_mc) * TMW + lane;
        const int mc = min(m, p.S);
        // bestf >= the exact partial minimum; -inf on cells whose partial is
        // never used (gated: m < m_null(s,t), DESIGN Q6; t > n; m > S)
        float bestf[RW][RW];
#pragma unroll
        for (int i = 0; i < RW; i++)
#pragma unroll
            for (int j = 0; j < RW; j++) {
                const int t = t_0 + j;
                bestf[i][j] = (t <= n && m <= p.S && m >= m_null(p, s_0 + i, t)) ? INFINITY : -INFINITY;
            }
        float maxq[2][2];  // >= every bestf of the lane's 4 x 4 quadrants
#pragma unroll
        for (int qa = 0; qa < 2; qa++)
#pragma unroll
            for (int qb = 0; qb < 2; qb++) {
                maxq[qa][qb] = -INFINITY;
#pragma unroll
                for (int i = 4 * qa; i < 4 * qa + 4; i++)
#pragma unroll
                    for (int j = 4 * qb; j < 4 * qb + 4; j++) maxq[qa][qb] = fmaxf(maxq[qa][qb], bestf[i][j]);
            }
        // >= every bestf of the lane's tile (kept with maxq: changes only when a split fires)
        float mall = fmaxf(fmaxf(maxq[0][0], maxq[0][1]), fmaxf(maxq[1][0], maxq[1][1]));
        int nf = 0;  // fired splits of this item (warp-uniform; > fmax: the list overflowed)
        lap(c_init);
        for (int it = 0; it < iters; it++) {
            const int gi = kl * iters + it;
            const int st = gi % STAGES;
            lap(c_loop);
            mbar_wait(&full[st], (uint32_t)((gi / STAGES) & 1));
            lap(c_wait);
            const float *a_f = ring + st * ST + (s_0 - I * TB - 1) * TMW + lane;
            const float *b_f = ring + st * ST + KC * SBOX + (t_0 - J * TB - 1) * TMW + lane;
            // the warp's two row groups / two column groups among the quad minima
            const float *qa_f = ring + st * ST + (kQuad + (s_0 - I * TB - 1) / 4) * TMW + lane;
            const float *qb_f = ring + st * ST + KC * SBOX + (kQuad + (t_0 - J * TB - 1) / 4) * TMW + lane;
            unsigned needk = 0;
#pragma unroll 2
            for (int k = 0; k < KC; k++) {
                // coarse bounds first: per 4 x 4 quadrant (qa, qb) of the lane's
                // tile, fadd_rd(min a over its rows, min b over its columns) is
                // <= every lb of the quadrant (monotone rounding) and maxq >= every
                // bestf of it; a quadrant is compared cell by cell only if that
                // bound is below maxq on some lane of the warp.  The minima come
                // precomputed (QA / QC: 4 loads instead of 16 + 12 FMNMX).
                float ma[2], mb[2];
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    ma[h] = qa_f[k * SBOX + h * TMW];
                    mb[h] = qb_f[k * SBOX + h * TMW];
                }
                bool nk = false;
                if (__any_sync(0xffffffffu, !coarse || __fadd_rd(fminf(ma[0], ma[1]), fminf(mb[0], mb[1])) < mall)) {
                    if (COUNT) c_coarse++;
                    float a[RW], b[RW];
#pragma unroll
                    for (int i = 0; i < RW; i++) a[i] = a_f[k * SBOX + i * TMW];
#pragma unroll
                    for (int j = 0; j < RW; j++) b[j] = b_f[k * SBOX + j * TMW];
#pragma unroll
                    for (int qa = 0; qa < 2; qa++)
#pragma unroll
                        for (int qb = 0; qb < 2; qb++) {
                            const bool maybe = !coarse || __fadd_rd(ma[qa], mb[qb]) < maxq[qa][qb];
                            if (__any_sync(0xffffffffu, maybe)) {
                                if (COUNT) c_quads++;
                                // two cells per packed FADD2.RM (the same rounding per element)
#pragma unroll
                                for (int i = 4 * qa; i < 4 * qa + 4; i++)
#pragma unroll
                                    for (int j = 4 * qb; j < 4 * qb + 4; j += 2) {
                                        const float2 lb = fadd2_rd(make_float2(a[i], a[i]), make_float2(b[j], b[j + 1]));
                                        nk |= (lb.x < bestf[i][j]) | (lb.y < bestf[i][j + 1]);
                                    }
                            }
                        }
                  // (the whole warp is inside the coarse-pass branch: nk is uniform below)
                  if (__any_sync(0xffffffffu, nk)) {
                    // The split may lower some cell: it is recorded for the exact fp64
                    // pass (deferred to the end of the item, so the warp does not stall
                    // on global memory here), and every bestf drops to an fp32 UPPER
                    // bound of the candidate the exact pass will evaluate: a <= nu(a32)
                    // (a32 = rd(a), nu = next float up), so fl64(a + b) <= ru32(nu(a32)
                    // + nu(b32)).  bestf then stays >= the final exact minimum.
                    if (COUNT) c_exact++;
                    const int q = nf + __popc(needk);
                    if (lane == 0 && q < fmax) flist[q] = (uint16_t)(it * KC + k);  // s' - sp_lo
                    float au[RW], bu[RW];
#pragma unroll
                    for (int i = 0; i < RW; i++) au[i] = __int_as_float(__float_as_int(a[i]) + (a[i] < INFINITY));
#pragma unroll
                    for (int j = 0; j < RW; j++) bu[j] = __int_as_float(__float_as_int(b[j]) + (b[j] < INFINITY));
#pragma unroll
                    for (int i = 0; i < RW; i++)
#pragma unroll
                        for (int j = 0; j < RW; j++) bestf[i][j] = fminf(bestf[i][j], __fadd_ru(au[i], bu[j]));
#pragma unroll
                    for (int qa = 0; qa < 2; qa++)
#pragma unroll
                        for (int qb = 0; qb < 2; qb++) {
                            maxq[qa][qb] = -INFINITY;
#pragma unroll
                            for (int i = 4 * qa; i < 4 * qa + 4; i++)
#pragma unroll
                                for (int j = 4 * qb; j < 4 * qb + 4; j++)
                                    maxq[qa][qb] = fmaxf(maxq[qa][qb], bestf[i][j]);
                        }
                    mall = fmaxf(fmaxf(maxq[0][0], maxq[0][1]), fmaxf(maxq[1][0], maxq[1][1]));
                    needk |= 1u << k;
                  }
                }
            }
            nf += __popc(needk);
            // Release stage st (mbarrier arrive: release of the thread's reads); the
            // warp whose arrival completes the phase sees it with a non-blocking
            // test (acquire) and refills the stage at once — no warp ever blocks
            // on slower ones (a dedicated producer warp would not fit the register
            // file).  The CAS hands the refill to exactly one warp.
            // (every thread arrives — count CONSUMERS — rather than lane 0 after a
            // __syncwarp: the same cost here, and compute-sanitizer's racecheck
            // then sees each thread's own release of its reads)
            int first = 0;  // the first warp done with stage st prepares its next refill
            if (lane == 0) first = gi + STAGES < total && atomicCAS(&prep[st], gi, gi + STAGES) == gi;
            if (__shfl_sync(0xffffffffu, first, 0)) prepare_warp(gi + STAGES, lane);
            mbar_arrive(&empty[st]);  // (after the addresses: the arrive releases them too)
            int claimed = 0;
            if (lane == 0)
                claimed = gi + STAGES < total && mbar_test(&empty[st], (uint32_t)((gi / STAGES) & 1)) &&
                          atomicCAS(&claim[st], gi, gi + STAGES) == gi;
            if (__shfl_sync(0xffffffffu, claimed, 0)) issue_warp(gi + STAGES, lane);
        }
        __syncwarp();
        lap(c_loop);
        // the item's fired splits go to the dependent phase's sub-product, which
        // evaluates them exactly with its own splits; only an overflowing list
        // is evaluated here (and its exact partial written)
        uint16_t *gl = p.mlist + mlist_index(n_mc, I, item % n_mc, warp);
        if (nf <= MLIST_CAP) {
            if (lane < nf) gl[1 + lane] = flist[lane];
            if (lane == 0) gl[0] = (uint16_t)nf;
        } else {
            exact_flush(p, flist, nf, fmax, I * TB + 1 + TB, iters * KC, s_0, t_0, 1, m, mc, wxp);
            if (lane == 0) gl[0] = MLIST_OVERFLOW;
        }
        __syncwarp();
        lap(c_flush);
    }
    if (COUNT && lane == 0) {
        atomicAdd(p.counters + CTR_SPLITS, (unsigned long long)my_items * iters * KC);
        atomicAdd(p.counters + CTR_COARSE_PASS, (unsigned long long)c_coarse);
        atomicAdd(p.counters + CTR_QUADS, (unsigned long long)c_quads);
        atomicAdd(p.counters + CTR_EXACT, (unsigned long long)c_exact);
        atomicAdd(p.counters + CTR_WAIT, c_wait);
        atomicAdd(p.counters + CTR_INIT, c_init);
        atomicAdd(p.counters + CTR_LOOP, c_loop);
        atomicAdd(p.counters + CTR_FLUSH, c_flush);
        atomicAdd(p.counters + CTR_N + warp, c_loop + c_flush);  // per warp slot (balance across warps)
    }
}

#include "rotor_tiled_dep.cuh"

// Quad minima of the tiles I in [tile_lo, tile_lo + gridDim.z) of tile
// diagonal delta, rebuilt from their fp32 shadows after a sharded fill unpacked
// them (the leaves write them as they go): y < 256: the column groups of C32
// row s = i0 + y / 8 (min of the 4 shadow rows at the same column: one row s,
// one pre-shift); y >= 256: the row groups of A32 column c = j0 + (y - 256) / 8
// (A(s, c) exists for s <= c, c < n).  Only existing cells enter a minimum; a
// group with none gets +inf.  Thread = one shadow column m <= S.
__global__ void k_tile_quads(Problem p, int delta, int tile_lo) {
    const int n = p.n;
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m > p.S) return;
    const int I = tile_lo + (int)blockIdx.z, J = I + delta;
    const int i0 = I * TB + 1, j0 = J * TB + 1;
    const int y = blockIdx.y & 255, g = y & 7;
    float v = INFINITY;
    if (blockIdx.y < 256) {
        const int s = i0 + (y >> 3), t1 = j0 + 4 * g;
        if (s > n || j0 > n) return;  // no table row
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int t = t1 + k;
            if (t >= s && t <= n) v = fminf(v, p.C32[shadow_index(p.scrows, srow_c(s, t), m)]);
        }
        p.C32[shadow_index(p.scrows, sc_row(J, s) + kQuad + g, m)] = v;
    } else {
        const int c = j0 + (y >> 3), s1 = i0 + 4 * g;
        if (c >= n) return;  // no A column
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int s = s1 + k;
            if (s <= c) v = fminf(v, p.A32[shadow_index(p.sarows, srow_a(n, s, c), m)]);
        }
        p.A32[shadow_index(p.sarows, sa_col(n, I, c) + kQuad + g, m)] = v;
    }
}

inline void launch_quads(const Problem &p, int delta, int tile_lo, int ntiles, cudaStream_t st) {
    dim3 grid((p.S + 1 + 127) / 128, 512, ntiles);
    k_tile_quads<<<grid, 128, 0, st>>>(p, delta, tile_lo);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}

bool make_map(CUtensorMap *map, const double *base, int64_t rows, int64_t pitch, int box_cols, int box_rows) {
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)pitch, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(pitch * 8)};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int KCW, int STG>
bool set_wide_attr() {
    const int b = 227 * 1024;
    const cudaFuncAttribute a = cudaFuncAttributeMaxDynamicSharedMemorySize;
    return cudaFuncSetAttribute(k_tile_middle_wide<KCW, STG, false>, a, b) != cudaSuccess ||
           cudaFuncSetAttribute(k_tile_middle_wide<KCW, STG, true>, a, b) != cudaSuccess;
}

template <int KCW, int STG>
void launch_wide(const Problem &p, int delta, int tile_lo, int nt, int coarse, int grid, size_t wx_b, cudaStream_t st) {
    const int fmax = wide_fmax(p.n, WideRing<KCW, STG>::bytes);
    const size_t smem = WideRing<KCW, STG>::bytes + wx_b + (size_t)(CONSUMERS / 32) * fmax * 2;
    if (p.counters)
        k_tile_middle_wide<KCW, STG, true><<<grid, THREADS, smem, st>>>(p, delta, tile_lo, nt, coarse, fmax);
    else
        k_tile_middle_wide<KCW, STG, false><<<grid, THREADS, smem, st>>>(p, delta, tile_lo, nt, coarse, fmax);
}

}  // namespace tiled

// Scratch of the tiled fill beyond the A table (which is part of the Layout):
// the leaf flags, then (256-byte aligned) the middle's fired-split lists.
size_t tiled_list_offset(int L, int S) { return (tiled::leaf_flag_bytes(L, S) + 255) & ~(size_t)255; }
size_t tiled_extra_bytes(int L, int S) { return tiled_list_offset(L, S) + tiled::mlist_bytes(L, S); }

int tiled_nb(int n) { return (n + tiled::TB - 1) / tiled::TB; }

int64_t tiled_middle_candidates(int n) {
    using tiled::TB;
    const int nb = tiled_nb(n);
    int64_t tot = 0;
    for (int I = 0; I < nb; I++) {
        const int cs = min(n, TB * (I + 1)) - TB * I;
        for (int J = I + 2; J < nb; J++) tot += (int64_t)cs * (min(n, TB * (J + 1)) - TB * J) * (J - I - 1) * TB;
    }
    return tot;
}

// Per-solve setup: kernel attributes, the tensor maps of the exact middle
// (over the whole allocations: left pad columns and spare rows included),
// zeroed leaf flags.  The shared-memory opt-in is a per-device function
// attribute, so it is set on every call (the current device may change
// between solves; the call is cheap).
int tiled_prepare(const Problem &p, TiledCtx *ctx, cudaStream_t st) {
    using namespace tiled;
    static_assert(sizeof(CUtensorMap) <= sizeof(ctx->tmA), "tensor map storage");
    if (cudaFuncSetAttribute(k_tile_middle<KC, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(SMEM_BYTES + (size_t)WX_SMEM_MAX * 4)) != cudaSuccess ||
        set_wide_attr<8, 2>() || set_wide_attr<4, 4>() || set_wide_attr<2, 8>() || set_wide_attr<4, 2>())
        return -1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        return -1;
    const int n = p.n;
    const int64_t rows = (int64_t)n * (n + 1) / 2;
    if (!make_map(reinterpret_cast<CUtensorMap *>(ctx->tmA), p.A - kPad, rows + kPadRows, p.pitch, TM, TB) ||
        !make_map(reinterpret_cast<CUtensorMap *>(ctx->tmC), p.C - kPad, rows + kPadRows, p.pitch, TMB, TB) ||
        !p.A32 || !p.C32)
        return -1;
    if (!p.flags || cudaMemsetAsync(p.flags, 0, leaf_flag_bytes(p.L, p.S), st) != cudaSuccess) return -1;
    ctx->phase_id = 0;
    ctx->mid_ev = nullptr;
    ctx->mid_cap = ctx->mid_n = 0;
    return 0;
}

// Middle + dependent phase of the tiles I in [tile_lo, tile_hi) of tile
// diagonal delta; `phase` counts the leaf launches that used the flags of
// these tile rows (the look-back epochs).  Returns the number of kernels launched.
int tiled_delta_ep(const Problem &p, TiledCtx *ctx, int delta, int tile_lo, int tile_hi, cudaStream_t st, int &phase) {
    using namespace tiled;
    if (tile_hi <= tile_lo) return 0;
    int launches = 0;
    if (delta >= 2) {
        const int sms = ctx->sms;
        static int coarse = -1;  // ROTOR_COARSE=0|1 (A/B)
        if (coarse < 0) {
            const char *e = getenv("ROTOR_COARSE");
            coarse = e ? atoi(e) : 1;
        }
        static int variant = -1;  // ROTOR_MIDDLE=exact|wide (A/B runs; default wide)
        if (variant < 0) {
            const char *e = getenv("ROTOR_MIDDLE");
            variant = (e && !strcmp(e, "exact")) ? 0 : 2;
        }
        const int nt = tile_hi - tile_lo;
        const bool timed = ctx->mid_ev && ctx->mid_n < ctx->mid_cap;
        if (timed) cudaEventRecord(ctx->mid_ev[2 * ctx->mid_n], st);
        if (variant == 2) {
            const int items_w = nt * ((p.S + 1 + TMW - 1) / TMW);
            // ring geometry (same-box A/B, ms of middle per config-4 solve, r01 TMA
            // boxes): KC = 4 x 6 stages 79.1, x 5 77.3, x 4 76.8, x 3 76.6; KC = 8 x 3
            // 83.5 — the shallower ring leaves more of the SM's shared-memory/L1
            // carve-out to L1 (spill reloads, exact-pass operands)
            const size_t wx_b = n_wx_smem(p.n) ? (size_t)p.n * 4 : 0;
            const int gw = items_w < sms ? items_w : sms;
            // ROTOR_WRING=44|28|42 (KC x stages, A/B runs; default 8 x 2: half the
            // release / refill rounds per split of 4 x 4 — 41.9 vs 46.8 ms of
            // middle per config-4 solve; 4 x 3 45.8)
            static int ring = -1;
            if (ring < 0) {
                const char *e = getenv("ROTOR_WRING");
                ring = e ? atoi(e) : 82;
            }
            if (ring == 28)
                launch_wide<2, 8>(p, delta, tile_lo, nt, coarse, gw, wx_b, st);
            else if (ring == 44)
                launch_wide<4, 4>(p, delta, tile_lo, nt, coarse, gw, wx_b, st);
            else if (ring == 42)
                launch_wide<4, 2>(p, delta, tile_lo, nt, coarse, gw, wx_b, st);
            else
                launch_wide<WKC, WSTAGES>(p, delta, tile_lo, nt, coarse, gw, wx_b, st);
        } else {
            const int n_items = nt * ((p.S + 1 + TM - 1) / TM);
            const int grid = n_items < sms ? n_items : sms;  // persistent: one CTA per SM
            const size_t smem = SMEM_BYTES + (p.n <= WX_SMEM_MAX ? (size_t)p.n * 4 : 0);
            const CUtensorMap &tmA = *reinterpret_cast<const CUtensorMap *>(ctx->tmA);
            const CUtensorMap &tmC = *reinterpret_cast<const CUtensorMap *>(ctx->tmC);
            k_tile_middle<KC, STAGES><<<grid, THREADS, smem, st>>>(tmA, tmC, p, delta, tile_lo, nt);
        }
        if (timed) cudaEventRecord(ctx->mid_ev[2 * ctx->mid_n++ + 1], st);
        launches++;
    }
    return launches + launch_dependent(p, delta, tile_lo, tile_hi, st, p.flags, phase);
}

int tiled_delta(const Problem &p, TiledCtx *ctx, int delta, int tile_lo, int tile_hi, cudaStream_t st) {
    return tiled_delta_ep(p, ctx, delta, tile_lo, tile_hi, st, ctx->phase_id);
}

inline int env_int(const char *name, int dflt) {
    const char *e = getenv(name);
    return e ? atoi(e) : dflt;
}

namespace {
// Per-thread, per-device streams and events of the tile-DAG schedule.
struct DagRes {
    std::vector<cudaStream_t> st;
    std::vector<cudaEvent_t> ev;
    cudaEvent_t start = nullptr;
};
constexpr int DAG_MAX_STREAMS = 64;  // rows share streams beyond this (long chains: nb > 64)
DagRes *dag_res(int nb) {
    static thread_local std::map<int, DagRes> res;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    DagRes &r = res[dev];
    if (!r.start && cudaEventCreateWithFlags(&r.start, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    static const int prio = env_int("ROTOR_DAG_PRIO", 1);  // rows with lower I first (127.4 vs 129.1 ms per solve; 0: all equal)
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    const int ns = min(nb, DAG_MAX_STREAMS);
    while ((int)r.st.size() < ns) {
        cudaStream_t s;
        const int i = (int)r.st.size();
        // priority levels spread over the rows: row 0 the highest
        const int pr = prio ? greatest + (least - greatest) * i / max(1, ns - 1) : least;
        if (cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, pr) != cudaSuccess) return nullptr;
        r.st.push_back(s);
    }
    while ((int)r.ev.size() < nb) {  // one event per tile row
        cudaEvent_t e;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
        r.ev.push_back(e);
    }
    return &r;
}
}  // namespace

// The whole fill.  schedule 1: diagonal by diagonal on `st` (every launch
// covers all tiles of a tile diagonal; the middle launches can be timed).
// schedule 0 (default): the tile DAG.  Tile (I, J) depends only on tiles of
// its row I and column J with smaller J - I (Theorem 1 reads strictly shorter
// intervals); its row's tiles run in order on stream I, and its
// column's through tile (I+1, J), whose own dependencies cover the rest, so
// each tile task waits on ONE event: (I+1, J) done.  Tiles of different rows
// then overlap — a tile's latency-bound dependent phase with other tiles'
// middles — instead of every diagonal ending in a device-wide barrier.
// Returns the number of kernels launched, or -1 on a launch/setup error.
int launch_fill_tiled(const Problem &p, cudaStream_t st, int schedule, cudaEvent_t *mid_ev, int mid_cap, int *mid_n) {
    // (A CUDA-graph replay of the whole DAG — one capture per problem, one
    // cudaGraphLaunch per solve — measured no faster: 118.7 vs 118.9 ms per
    // config-4 solve; the per-launch host and GPU gaps are not what bounds it.)
    TiledCtx ctx;
    if (tiled_prepare(p, &ctx, st)) return -1;
    ctx.mid_ev = mid_ev;
    ctx.mid_cap = mid_cap;
    const int nb = tiled_nb(p.n);
    int launches = 0;
    DagRes *r = schedule == 0 ? dag_res(nb) : nullptr;
    if (!r) {
        for (int delta = 0; delta < nb; delta++) {
            char nm[40];
            snprintf(nm, sizeof nm, "rotor.fill.delta=%d", delta);
            nvtxRangePushA(nm);
            launches += tiled_delta(p, &ctx, delta, 0, nb - delta, st);
            nvtxRangePop();
        }
    } else {
        std::vector<int> phase(nb, 0);  // (middle launches are timed on their own streams; they overlap)
        // ROTOR_TRACE=<file>: per tile task, the host enqueue time and the GPU
        // time its middle starts / its dependent phase ends (timing events,
        // relative to the fill's start) — a timeline of the DAG (diagnostic)
        static const char *trace = getenv("ROTOR_TRACE");
        std::vector<cudaEvent_t> tev;
        std::vector<double> thost;
        auto t_host0 = std::chrono::steady_clock::now();
        cudaEvent_t tstart = nullptr;
        if (trace) {
            cudaEventCreate(&tstart);
            cudaEventRecord(tstart, st);
        }
        // row I on stream I mod ns: rows sharing a stream only add order between
        // tasks that are enqueued in dependency order anyway (diagonal-major)
        const int ns = (int)r->st.size();
        auto row_st = [&](int I) { return r->st[I % ns]; };
        cudaEventRecord(r->start, st);
        for (int k = 0; k < ns; k++) cudaStreamWaitEvent(r->st[k], r->start, 0);
        for (int delta = 0; delta < nb; delta++) {
            char nm[40];
            snprintf(nm, sizeof nm, "rotor.fill.delta=%d", delta);
            nvtxRangePushA(nm);  // host enqueue of the tile diagonal's tasks
            for (int I = 0; I + delta < nb; I++) {
                // (I+1, I+delta) is the latest record of ev[I+1]: row I+1 is enqueued after row I
                if (delta >= 1) cudaStreamWaitEvent(row_st(I), r->ev[I + 1], 0);
                if (trace) {
                    cudaEvent_t a, z;
                    cudaEventCreate(&a);
                    cudaEventCreate(&z);
                    thost.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_host0).count());
                    cudaEventRecord(a, row_st(I));
                    launches += tiled_delta_ep(p, &ctx, delta, I, I + 1, row_st(I), phase[I]);
                    cudaEventRecord(z, row_st(I));
                    tev.push_back(a);
                    tev.push_back(z);
                } else {
                    launches += tiled_delta_ep(p, &ctx, delta, I, I + 1, row_st(I), phase[I]);
                }
                cudaEventRecord(r->ev[I], row_st(I));
            }
            nvtxRangePop();
        }
        for (int I = 0; I < nb; I++) cudaStreamWaitEvent(st, r->ev[I], 0);  // (I < ns covers every stream)
        if (trace) {
            const double host_total =
                std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_host0).count();
            cudaStreamSynchronize(st);
            FILE *f = fopen(trace, "w");
            if (f) {
                fprintf(f, "I,J,host_us,start_us,end_us\n");
                size_t k = 0;
                for (int delta = 0; delta < nb; delta++)
                    for (int I = 0; I + delta < nb; I++, k++) {
                        float a = 0, z = 0;
                        cudaEventElapsedTime(&a, tstart, tev[2 * k]);
                        cudaEventElapsedTime(&z, tstart, tev[2 * k + 1]);
                        fprintf(f, "%d,%d,%.1f,%.1f,%.1f\n", I, I + delta, thost[k], a * 1e3, z * 1e3);
                    }
                fprintf(f, "# host enqueue total %.1f us\n", host_total);
                fclose(f);
            }
            for (auto e : tev) cudaEventDestroy(e);
            cudaEventDestroy(tstart);
        }
    }
    if (mid_n) *mid_n = ctx.mid_n;
    return launches;
}

// ---------------------------------------------------------------------------
// Sharded fill support: pack / unpack the C and A rows of a range of tiles of
// one tile diagonal into a contiguous buffer [tile][C|A][TB s][TB t][S+1].
// Cells that do not exist (s > t, t > n; A at t = n) are skipped both ways.
// ---------------------------------------------------------------------------
// One finished tile travels as its C rows only (TB x TB x (S+1) fp64): the
// receiver rebuilds A(s,t,m) = fl(fl(P[t] - P[s-1]) + C(s,t,m)) with the same
// association as the producing kernels (Q12), so its A rows are bit-identical
// and the exchange volume is half of sending both tables.
size_t tiled_tile_bytes(int S) { return (size_t)tiled::TB * tiled::TB * (S + 1) * sizeof(double); }

// mode 0: pack this table's tiles into buf; 1: unpack buf into this table;
// 2: pull the tiles straight from another table of the same layout (`src`,
// another device's C through peer memory: the fused P2P halo) into this one.
__global__ void k_tile_pack(Problem p, int delta, int tile_lo, double *buf, const double *src, int mode) {
    using namespace tiled;
    const int n = p.n, W = p.S + 1;
    const int tile = blockIdx.z, a = blockIdx.y / TB, c = blockIdx.y % TB;
    const int I = tile_lo + tile, J = I + delta;
    const int s = I * TB + 1 + a, t = J * TB + 1 + c;
    if (s > n || t > n || s > t) return;
    const int64_t row = cell_index(n, s, t);
    double *crow = p.C + row * p.pitch;
    const double *in = mode == 2 ? src + row * p.pitch : buf + (((int64_t)tile * TB + a) * TB + c) * W;
    double *packed = buf + (((int64_t)tile * TB + a) * TB + c) * W;
    const bool has_a = t < n;  // A(s, n) is never an operand
    const double u = has_a ? __dadd_rn(p.P[t], -p.P[s - 1]) : 0.0;
    const int w = p.wx[s - 1];
    for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < W; m += gridDim.x * blockDim.x) {
        if (mode) {
            const double v = mode == 2 ? __ldcv(in + m) : in[m];  // .cv: the owner wrote it this diagonal
            store_final_c(p, s, t, m, w, v);
            if (has_a) store_final_a(p, s, t, m, __dadd_rn(u, v));
        } else {
            packed[m] = crow[m];
        }
    }
}

int tiled_pack(const Problem &p, int delta, int tile_lo, int tile_hi, double *buf, int unpack, cudaStream_t st) {
    if (tile_hi <= tile_lo) return 0;
    dim3 grid(4, tiled::TB * tiled::TB, tile_hi - tile_lo);
    k_tile_pack<<<grid, 256, 0, st>>>(p, delta, tile_lo, buf, nullptr, unpack ? 1 : 0);
    if (!unpack) return 1;
    tiled::launch_quads(p, delta, tile_lo, tile_hi - tile_lo, st);
    return 2;
}

int tiled_pull(const Problem &p, const double *src_C, int delta, int tile_lo, int tile_hi, cudaStream_t st) {
    if (tile_hi <= tile_lo) return 0;
    dim3 grid(4, tiled::TB * tiled::TB, tile_hi - tile_lo);
    k_tile_pack<<<grid, 256, 0, st>>>(p, delta, tile_lo, nullptr, src_C, 2);
    tiled::launch_quads(p, delta, tile_lo, tile_hi - tile_lo, st);
    return 2;
}

}  // namespace rotor
