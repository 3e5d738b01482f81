// Tiled fill of the Theorem-1 table — the fast path.
//
// The split candidates of a cell (s,t) are
//     cand(s') = fl( A(s, s'-1, m) + C(s', t, m - wx[s'-1]) ),  s' = s+1..t,
// with A(s,c,m) = fl( fl(P[c] - P[s-1]) + C(s,c,m) ) stored next to C when a
// cell is finalised (Q12 association: fl(fl(U + pre) + suf)).  For a fixed m
// this is a min-plus product over s' (the m-shift depends on s' only), so the
// triangle is cut into TB x TB tiles of (s,t), processed by tile diagonal
// Delta = J - I.  For a tile (I,J), Delta >= 2:
//   * middle: s' in blocks I+1..J-1 — every operand is final (shorter tile
//     diagonals): a dense min-plus product with TB-fold operand reuse, operands
//     streamed by TMA into shared memory (k_tile_middle);
//   * dependent: s' in [s+1, i1-1] (B operand in this tile) and [j0, t]
//     (A operand in this tile): finished in 2*TB-1 local anti-diagonal steps
//     with a grid-wide barrier between steps (k_tile_dep, cooperative), which
//     also applies the gates, the F_all candidate, and writes C and A.
// Delta = 1 has no middle; Delta = 0 (diagonal tiles) is a local triangle.
// The min is exact and every candidate has the fixed association above, so the
// table is bit-identical to the wavefront / oracle fill (order-independent).
#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>

#include "rotor_common.cuh"
#include "rotor_kernels.cuh"

namespace cg = cooperative_groups;

namespace rotor {
namespace tiled {

constexpr int TB = 32;      // tile edge in stages
constexpr int KC = 8;       // splits per pipeline stage
constexpr int TM = 16;      // m values per CTA (middle kernel)
constexpr int STAGES = 3;   // TMA pipeline depth
constexpr int THREADS = 256;
constexpr int RS = 8, RT = 8;                 // register tile (s x t) per thread
// A TMA box must start on a 16-byte boundary of the row (an odd fp64 start
// column faults with "illegal instruction", scripts/tma_probe.cu): the shifted
// C boxes start at the even column below the wanted one and are TMB = TM + 2
// wide; the consumer adds the per-row offset (0 or 1).
constexpr int TMB = TM + 2;
constexpr int A_STAGE = TB * KC * TM;         // doubles [TB][KC][TM]
constexpr int B_STAGE = KC * TB * TMB;        // doubles [KC][TB][TMB]
constexpr size_t SMEM_BYTES = (size_t)STAGES * (A_STAGE + B_STAGE) * 8 + STAGES * 8 + STAGES * KC * 4 + 64;

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

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }

// ---------------------------------------------------------------------------
// Middle phase of tile diagonal delta >= 2: partial(s,t,m) = min over s' in
// blocks I+1..J-1 of A(s,s'-1,m) + C(s',t,m-wx[s'-1]); written into C.
// grid = (ceil((S+1)/TM), tiles), block = 256; thread = one m, an 8x8 (s,t) tile.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(THREADS, 1)
    k_tile_middle(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmC, Problem p,
                  int delta) {
    extern __shared__ __align__(1024) double smem[];  // no static smem: the dynamic base is aligned
    double *As = smem;                       // [STAGES][TB][KC][TM]
    double *Bs = smem + STAGES * A_STAGE;    // [STAGES][KC][TB][TMB]
    uint64_t *bars = reinterpret_cast<uint64_t *>(Bs + STAGES * B_STAGE);
    int *soff = reinterpret_cast<int *>(bars + STAGES);  // [STAGES][KC] column offset of each C box

    const int I = blockIdx.y, J = I + delta;
    const int i0 = I * TB + 1, j0 = J * TB + 1, i1 = i0 + TB;
    const int m0 = blockIdx.x * TM;
    const int n = p.n;
    const int iters = (delta - 1) * TB / KC;
    const int tid = threadIdx.x;

    auto issue = [&](int it) {
        const int st = it % STAGES;
        const int sp0 = i1 + it * KC;
        uint64_t *bar = &bars[st];
        // column offsets first: the expect_tx arrive (release) orders them
        // before the consumers' barrier wait (acquire)
        for (int k = 0; k < KC; k++) soff[st * KC + k] = (max(m0 - p.wx[sp0 + k - 1], -kPad) + kPad) & 1;
        mbar_expect_tx(bar, (uint32_t)((A_STAGE + B_STAGE) * 8));
        double *a_dst = As + st * A_STAGE;
        for (int a = 0; a < TB; a++) {
            const int s = i0 + a;  // cells (s, sp0-1 .. sp0+KC-2)
            tma_load_2d(a_dst + a * KC * TM, &tmA, m0 + kPad, (int)cell_index(n, s, sp0 - 1), bar);
        }
        double *b_dst = Bs + st * B_STAGE;
        for (int k = 0; k < KC; k++) {
            const int sp = sp0 + k;  // cells (sp, j0 .. j0+TB-1) at m - wx[sp-1]
            // A chunk whose shifted window starts below -kPad lies wholly under
            // m = wx[sp-1] <= m_null(s,t): every cell it feeds is gated, so the
            // (clamped) values loaded for it are never used (DESIGN Q6).
            const int c0 = max(m0 - p.wx[sp - 1], -kPad) + kPad;
            tma_load_2d(b_dst + k * TB * TMB, &tmC, c0 & ~1, (int)cell_index(n, sp, j0), bar);
        }
    };

    if (tid == 0) {
        for (int s = 0; s < STAGES; s++) mbar_init(&bars[s], 1);
        // make the initialised barriers visible to the async (TMA) proxy; the
        // .cluster-scoped fence.mbarrier_init faults in a non-cluster launch
        // (scripts/tma_probe.cu, variant 1)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
        for (int it = 0; it < STAGES && it < iters; it++) issue(it);
    }

    const int mi = tid & 15;
    const int g = tid >> 4;
    const int sg = g >> 2, tg = g & 3;
    double acc[RS][RT];
#pragma unroll
    for (int i = 0; i < RS; i++)
#pragma unroll
        for (int j = 0; j < RT; j++) acc[i][j] = INFINITY;

    for (int it = 0; it < iters; it++) {
        const int st = it % STAGES;
        mbar_wait(&bars[st], (uint32_t)((it / STAGES) & 1));
        const double *a_s = As + st * A_STAGE + (sg * RS) * KC * TM + mi;
        const double *b_s = Bs + st * B_STAGE + (tg * RT) * TMB + mi;
#pragma unroll
        for (int k = 0; k < KC; k++) {
            double a[RS], b[RT];
            const double *bk = b_s + k * TB * TMB + soff[st * KC + k];
#pragma unroll
            for (int i = 0; i < RS; i++) a[i] = a_s[i * KC * TM + k * TM];
#pragma unroll
            for (int j = 0; j < RT; j++) b[j] = bk[j * TMB];
#pragma unroll
            for (int i = 0; i < RS; i++)
#pragma unroll
                for (int j = 0; j < RT; j++) acc[i][j] = dmin(acc[i][j], __dadd_rn(a[i], b[j]));
        }
        __syncthreads();  // every thread is done reading stage st
        if (tid == 0 && it + STAGES < iters) issue(it + STAGES);
    }

    const int m = m0 + mi;
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
}

// ---------------------------------------------------------------------------
// Dependent phase of tile diagonal delta (cooperative; grid-wide barrier
// between the local anti-diagonal steps).  One warp = one cell x 32 m values.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void finish_cell(const Problem &p, const double *A, double *Aw, int s, int t, int m,
                                            int lo1, int hi1, int lo2, int hi2, bool partial) {
    const int n = p.n;
    const int64_t pitch = p.pitch;
    const int64_t cst = cell_index(n, s, t);
    // Values written by other CTAs in earlier steps of this launch are read with
    // ld.global.cg (L2, never a stale L1 line).
    double c1 = INFINITY;
    if (m >= m_null(p, s, t)) {
        double best = partial ? __ldcg(&p.C[cst * pitch + m]) : INFINITY;
        const int64_t rs = cell_index(n, s, s);  // A(s, c) at row rs + (c - s)
        for (int sp = lo1; sp <= hi1; sp++) {
            const int mm = m - p.wx[sp - 1];  // >= 0 under the m_null gate (DESIGN Q6)
            const double v = __dadd_rn(__ldcg(&A[(rs + (sp - 1 - s)) * pitch + m]),
                                       __ldcg(&p.C[cell_index(n, sp, t) * pitch + mm]));
            best = dmin(best, v);
        }
        for (int sp = lo2; sp <= hi2; sp++) {
            const int mm = m - p.wx[sp - 1];
            const double v = __dadd_rn(__ldcg(&A[(rs + (sp - 1 - s)) * pitch + m]),
                                       __ldcg(&p.C[cell_index(n, sp, t) * pitch + mm]));
            best = dmin(best, v);
        }
        c1 = best;
    }
    double c = c1;
    if (!p.restricted && m >= m_all(p, s, t)) {  // m - wbx[s] >= 0 under the m_all gate
        const double v = __dadd_rn(p.w[s], __ldcg(&p.C[cell_index(n, s + 1, t) * pitch + (m - p.wbx[s])]));
        c = dmin(c, v);
    }
    p.C[cst * pitch + m] = c;
    if (t < n) Aw[cst * pitch + m] = __dadd_rn(__dadd_rn(p.P[t], -p.P[s - 1]), c);
}

__global__ void __launch_bounds__(256) k_tile_dep(Problem p, double *A, int delta, int partial) {
    cg::grid_group grid = cg::this_grid();
    const int n = p.n, S = p.S;
    const int nb = (n + TB - 1) / TB;
    const int ntiles = nb - delta;
    const int n_mg = (S + 1 + 31) / 32;
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int e_lo = delta == 0 ? 1 : 0;
    const int e_hi = delta == 0 ? TB - 1 : 2 * TB - 2;
    for (int e = e_lo; e <= e_hi; e++) {
        // cells of local step e in one tile
        const int a_lo = delta == 0 ? 0 : max(0, (TB - 1) - e);
        const int a_hi = delta == 0 ? TB - 1 - e : min(TB - 1, 2 * TB - 2 - e);
        const int cnt = a_hi - a_lo + 1;
        const long long items = (long long)ntiles * cnt * n_mg;
        for (long long item = warp; item < items; item += nwarps) {
            const int mg = (int)(item % n_mg);
            const long long rest = item / n_mg;
            const int q = (int)(rest % cnt);
            const int I = (int)(rest / cnt);
            const int J = I + delta;
            const int a = a_lo + q;
            const int i0 = I * TB + 1, j0 = J * TB + 1;
            const int s = i0 + a;
            const int t = delta == 0 ? s + e : j0 + (a + e - (TB - 1));
            const int m = mg * 32 + lane;
            if (s > n || t > n || m > S) continue;
            if (delta == 0) {
                finish_cell(p, A, A, s, t, m, s + 1, t, 1, 0, false);
            } else {
                const int i1 = i0 + TB;
                finish_cell(p, A, A, s, t, m, s + 1, min(t, i1 - 1), j0, t, partial != 0);
            }
        }
        grid.sync();
    }
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

int dep_grid_blocks() {
    static int blocks = 0;
    if (!blocks) {
        int dev = 0, sms = 0, per = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_tile_dep, 256, 0);
        blocks = sms * (per > 0 ? per : 1);
    }
    return blocks;
}

}  // namespace tiled

size_t tiled_extra_bytes(int, int) { return 0; }  // the A table is part of the Layout (rotor_abi.cu)

// Returns the number of kernels launched, or -1 on a launch/setup error.
int launch_fill_tiled(const Problem &p, cudaStream_t st) {
    using namespace tiled;
    static bool attr = false;
    if (!attr) {
        if (cudaFuncSetAttribute(k_tile_middle, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES) !=
            cudaSuccess)
            return -1;
        attr = true;
    }
    const int n = p.n;
    const int nb = (n + TB - 1) / TB;
    const int64_t rows = (int64_t)n * (n + 1) / 2;
    CUtensorMap tmA, tmC;  // over the whole allocations: left pad columns and spare rows included
    if (!make_map(&tmA, p.A - kPad, rows + kPadRows, p.pitch, TM, KC) ||
        !make_map(&tmC, p.C - kPad, rows + kPadRows, p.pitch, TMB, TB))
        return -1;
    const int dep_blocks = dep_grid_blocks();
    int launches = 0;
    for (int delta = 0; delta < nb; delta++) {
        if (delta >= 2) {
            dim3 grid((p.S + 1 + TM - 1) / TM, nb - delta);
            k_tile_middle<<<grid, THREADS, SMEM_BYTES, st>>>(tmA, tmC, p, delta);
            launches++;
        }
        Problem pp = p;
        double *A = p.A;
        int d = delta, part = delta >= 2 ? 1 : 0;
        void *args[] = {&pp, &A, &d, &part};
        if (cudaLaunchCooperativeKernel((void *)k_tile_dep, dim3(dep_blocks), dim3(256), args, 0, st) != cudaSuccess)
            return -1;
        launches++;
    }
    return launches;
}

}  // namespace rotor
