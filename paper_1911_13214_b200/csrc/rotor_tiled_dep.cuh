// Dependent phase of the tiled fill — two-level (included by rotor_tiled.cu
// inside namespace rotor::tiled).
//
// Inside a TB x TB tile (I,J) the splits that need values of the tile itself
// are s' in [s+1, i1-1] (left: C of rows below) and [j0, t] (right: A of the
// same row).  Cut the tile into NSB x NSB sub-tiles of SB x SB cells, (alpha,
// gamma) = (row sub-block of I, column sub-block of J).  Sub-tile (alpha,gamma)
// depends on sub-tiles (alpha' > alpha, gamma) and (alpha, gamma' < gamma), so
// sub-tiles are processed by sub-anti-diagonal eps = gamma - alpha + NSB-1;
// for each sub-tile
//   * product: the left splits in sub-blocks alpha+1.. of I and the right
//     splits in sub-blocks ..gamma-1 of J, whose operands are final: an SB x SB
//     min-plus product per m (8x8 register tile per lane), min-ed into the
//     partial value held in C (k_sub_product);
//   * leaf: the splits inside its own row sub-block / column sub-block, the
//     gates, F_all, and the writes of C and A, one local row per launch from
//     the bottom (k_sub_leaf): a row needs the rows below (complete, at
//     shifted m) and its own earlier columns at the same m (registers).
// Diagonal tiles (Delta = 0) use the same scheme with sub-diagonals
// delta' = gamma - alpha = 0..NSB-1 (products for delta' >= 2).
// Only cells x SB x (S+1) transitions remain in the leaves (vs cells x TB);
// the rest runs as products with SB-fold register reuse.

constexpr int SB = 8;
constexpr int NSB = TB / SB;
constexpr int DEP_THREADS = 128;

// number of sub-tiles of phase e, and the q-th one
__host__ __device__ inline int sub_count(int delta, int e) {
    return delta == 0 ? NSB - e : NSB - (e >= NSB - 1 ? e - (NSB - 1) : (NSB - 1) - e);
}
__host__ __device__ inline void sub_at(int delta, int e, int q, int &alpha, int &gamma) {
    if (delta == 0) {
        alpha = q;
        gamma = q + e;
    } else {
        const int dd = e - (NSB - 1);  // gamma - alpha
        alpha = (dd >= 0 ? 0 : -dd) + q;
        gamma = alpha + dd;
    }
}

// C / A loads: `fresh` = written earlier in this launch sequence of the same
// tile diagonal (another CTA, earlier kernel of this Delta) -> L2 (.cg);
// otherwise written by an earlier tile diagonal -> plain (L1-cacheable).
__device__ __forceinline__ double ld(const double *p, bool fresh) { return fresh ? __ldcg(p) : *p; }
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

constexpr int PH = SB / 2;  // columns per product lane

// The same product with the operands staged through a per-warp shared-memory
// ring by cp.async (PNS splits in flight per warp, no operand registers held
// across the load latency): lane (mi, half) copies rows / columns half*4..+3
// of the split's A column and shifted C row at m = m0 + mi; after the stage
// lands every lane reads all SB A values and its own PH C values.
constexpr int PNS = 5;  // splits in flight per warp (5: 121.2 vs 121.9 ms per solve with 4; 40 KB static smem)
constexpr int PW = DEP_THREADS / 32;

__device__ __forceinline__ void cp_async8(double *dst, const double *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// src_bytes = 0: nothing is read, the 8 bytes are zero-filled
__device__ __forceinline__ void cp_async8_zfill(double *dst, const double *src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int MINB>
__global__ void __launch_bounds__(DEP_THREADS, MINB) k_sub_product_async(Problem p, int delta, int e, int tile_lo,
                                                                         int ntiles) {
    // per warp and split: the element offsets of its operand rows A(s0, s'-1)
    // and C(s', t0) (shifted by -w) and its shift w, computed once by the
    // warp's lanes in parallel (each lane's own rows / m are a constant offset)
    constexpr int NSPMAX = 2 * (TB - SB) + MLIST_CAP + 1;
    __shared__ long long soff[PW][NSPMAX][2];
    __shared__ int sw[PW][NSPMAX];
    __shared__ double ring[PW][PNS][2][SB][16];  // [warp][stage][A | C][row | column][m]
    const int n = p.n, S = p.S;
    const int cnt = sub_count(delta, e);
    const int n_mg = (S + 1 + 15) / 16;
    const int wid = threadIdx.x >> 5;
    const int item = (blockIdx.x * DEP_THREADS + threadIdx.x) >> 5;
    if (item >= ntiles * cnt * n_mg) return;
    const int lane = threadIdx.x & 31;
    const int mi = lane & 15, half = lane >> 4;
    const int m = (item % n_mg) * 16 + mi;
    const int jh = half * PH;
    const int rest = item / n_mg;
    int alpha, gamma;
    sub_at(delta, e, rest % cnt, alpha, gamma);
    const int I = tile_lo + rest / cnt, J = I + delta;
    const int i0 = I * TB + 1, j0 = J * TB + 1;
    const int s0 = i0 + SB * alpha, t0 = j0 + SB * gamma;
    int lo1, hi1, lo2 = 1, hi2 = 0;
    bool partial;
    if (delta == 0) {
        lo1 = i0 + SB * (alpha + 1);
        hi1 = t0 - 1;
        partial = false;
    } else {
        lo1 = s0 + SB;
        hi1 = i0 + TB - 1;
        lo2 = j0;
        hi2 = t0 - 1;
        partial = delta >= 2;
    }
    // the middle's fired splits for this sub-tile and 32-m chunk (delta >= 2)
    const uint16_t *lst = nullptr;
    int n3 = 0;
    bool mid_partial = false;  // the middle overflowed its list and wrote the exact partial itself
    if (partial) {
        lst = p.mlist + mlist_index(n_mc32(S), I, (item % n_mg) * 16 / 32, alpha * NSB + gamma);
        const int h = lst[0];
        mid_partial = h == MLIST_OVERFLOW;
        n3 = mid_partial ? 0 : h;
    }
    const int n1 = max(0, hi1 - lo1 + 1), n2 = max(0, hi2 - lo2 + 1), nsp = n1 + n2 + n3;
    if (s0 > n || t0 > n) return;      // no cells (uniform over the warp)
    if (nsp == 0 && (!partial || mid_partial)) return;  // nothing to add; the partial (if any) is final
    const int64_t pitch = p.pitch;
    const bool mlive = m <= S;
    const int sp_mid = i0 + TB;  // s' of middle split index 0
    // split idx: 0..n1-1 -> s' = lo1 + idx (left), n1..n1+n2-1 -> s' = lo2 + idx - n1
    // (right), then the middle's recorded splits s' = sp_mid + lst[1 + ...]
    for (int idx = lane; idx < nsp; idx += 32) {
        const int sp = idx < n1 ? lo1 + idx : (idx < n1 + n2 ? lo2 + idx - n1 : sp_mid + lst[1 + idx - n1 - n2]);
        const int w = p.wx[sp - 1];
        soff[wid][idx][0] = a_index(s0, sp - 1) * pitch;
        soff[wid][idx][1] = cell_index(n, sp, t0) * pitch - w;
        sw[wid][idx] = w;
    }
    __syncwarp();
    // rows s0+jh.. of an A column and cells (s', t0+jh..) are consecutive table rows
    const int64_t pitch4[PH] = {0, pitch, 2 * pitch, 3 * pitch};
    const int64_t lane_off = (int64_t)jh * pitch + m;
    unsigned rows_a = 0, rows_c = 0;  // which of the lane's rows / columns exist
#pragma unroll
    for (int i = 0; i < PH; i++) {
        rows_a |= (s0 + jh + i <= n) << i;
        rows_c |= (t0 + jh + i <= n) << i;
    }
    int nx = 0;
    auto issue_next = [&]() {
        double(*st)[SB][16] = ring[wid][nx % PNS];
        const int w = sw[wid][nx];
        // A skipped operand is zero-filled: m < w means every cell the split
        // feeds is gated (m < w <= m_null, DESIGN Q6), so its partial is never
        // read; a row / column past the last stage feeds only cells that do not
        // exist.  Branch-free copies (src-size 0 reads nothing).
        const bool use = mlive && m >= w;
        const double *la = p.A + soff[wid][nx][0] + lane_off;
        const double *lc = p.C + soff[wid][nx][1] + lane_off + (use ? 0 : w);
#pragma unroll
        for (int i = 0; i < PH; i++) {
            cp_async8_zfill(&st[0][jh + i][mi], la + pitch4[i], use && ((rows_a >> i) & 1));
            cp_async8_zfill(&st[1][jh + i][mi], lc + pitch4[i], use && ((rows_c >> i) & 1));
        }
        ++nx;
    };
    // the lane's cells (s0+i, t0+jh+j): row i starts cell_index(n, s0+i, t0+jh),
    // rows s -> s+1 are n-s cells apart (s-major), columns consecutive
    double acc[SB][PH];
    {
        const double *cr = p.C + cell_index(n, s0, t0 + jh) * pitch + m;
#pragma unroll
        for (int i = 0; i < SB; i++) {
#pragma unroll
            for (int j = 0; j < PH; j++)
                acc[i][j] = (mid_partial && mlive && s0 + i <= n && ((rows_c >> j) & 1)) ? __ldcg(cr + pitch4[j])
                                                                                           : INFINITY;
            cr += (int64_t)(n - (s0 + i)) * pitch;
        }
    }
#pragma unroll
    for (int k = 0; k < PNS - 1; k++) {
        if (k < nsp) issue_next();
        cp_async_commit();
    }
    for (int idx = 0; idx < nsp; idx++) {
        if (idx + PNS - 1 < nsp) issue_next();
        cp_async_commit();
        cp_async_wait<PNS - 1>();  // split idx landed (this lane's copies)
        __syncwarp();              // ... and every lane's
        const double(*st)[SB][16] = ring[wid][idx % PNS];
        double a[SB], c[PH];
#pragma unroll
        for (int i = 0; i < SB; i++) a[i] = st[0][i][mi];
#pragma unroll
        for (int j = 0; j < PH; j++) c[j] = st[1][jh + j][mi];
#pragma unroll
        for (int i = 0; i < SB; i++)
#pragma unroll
            for (int j = 0; j < PH; j++) acc[i][j] = dmin(acc[i][j], __dadd_rn(a[i], c[j]));
        __syncwarp();  // stage idx % PNS is refilled by the next iteration's issue
    }
    if (!mlive) return;
    double *cw = p.C + cell_index(n, s0, t0 + jh) * pitch + m;
#pragma unroll
    for (int i = 0; i < SB; i++) {
        if (s0 + i > n) break;
#pragma unroll
        for (int j = 0; j < PH; j++)
            if ((rows_c >> j) & 1) cw[pitch4[j]] = acc[i][j];
        cw += (int64_t)(n - (s0 + i)) * pitch;
    }
}

// Finish cell (s,t) at m from its running minimum c1 (already gated): F_all
// candidate, store C and A; returns A(s,t,m).
__device__ __forceinline__ double finish(const Problem &p, int s, int t, int m, double c1) {
    const int n = p.n;
    const int64_t pitch = p.pitch;
    double c = c1;
    if (!p.restricted && m >= m_all(p, s, t)) {  // m - wbx[s] >= 0 under the gate; row s+1 is final
        const double v = __dadd_rn(p.w[s], __ldcg(&p.C[cell_index(n, s + 1, t) * pitch + (m - p.wbx[s])]));
        c = dmin(c, v);
    }
    store_final_c(p, s, t, m, p.wx[s - 1], c);
    const double a = __dadd_rn(__dadd_rn(p.P[t], -p.P[s - 1]), c);
    if (t < n) store_final_a(p, s, t, m, a);
    return a;
}

// One local row r of the diagonal sub-tile (alpha, alpha) of diagonal tile I
// (delta = 0, phase 0), at one m: cells (s, s+1..ea), splits s' in (s, t].  The
// lane walks the row's cells left to right; right-range A operands stay in
// registers.  (Off-diagonal sub-tiles: leaf_row_tab.)
__device__ __forceinline__ void leaf_row_diag(const Problem &p, int alpha, int I, int r, int m) {
    const int n = p.n;
    const int i0 = I * TB + 1;
    const int s0 = i0 + SB * alpha, t0 = s0;
    const int s = s0 + r;
    if (s > n || m > p.S) return;  // sub-tiles past the last stage have no cells
    const int64_t pitch = p.pitch;
    double AR[SB + 1];  // AR[c] = A(s, t0 + c - 1)
    if (s == n) return;  // the last stage's row has no cell right of its leaf
    const double leaf = p.A[a_index(s, s) * pitch + m];  // the leaf (k_leaf, an earlier launch)
#pragma unroll
    for (int c = 0; c < SB; c++)  // AR[r + 1] = leaf, with compile-time register indices
        if (c == r) AR[c + 1] = leaf;
#pragma unroll
    for (int c = 0; c < SB; c++) {
        if (c <= r) continue;
        const int t = t0 + c;
        if (t > n) break;
        double c1 = INFINITY;
        if (m >= m_null(p, s, t)) {  // every shifted index is >= 0 under this gate (DESIGN Q6)
            double best = INFINITY;
#pragma unroll
            for (int cq = 0; cq < SB; cq++) {  // s' = t0 + cq + 1 in (s, t]
                if (cq < r || cq >= c) continue;
                const int sp = t0 + cq + 1;
                const double cv = __ldcg(&p.C[cell_index(n, sp, t) * pitch + (m - p.wx[sp - 1])]);
                best = dmin(best, __dadd_rn(AR[cq + 1], cv));
            }
            c1 = best;
        }
        AR[c + 1] = finish(p, s, t, m, c1);
    }
}

// Leaf phase e: CTA = one sub-tile x LEAF_M consecutive m (thread = one m),
// all SB local rows bottom-up in ONE launch.  Row r at m reads rows > r at
// m - shift, which may belong to lower m-chunks (other CTAs): after each row a
// CTA publishes `flags[sub][chunk] = (phase_id << 4) | rows_done` (release) and
// before each row waits (acquire) until every lower chunk of the same sub-tile
// has done the rows below (decoupled look-back).  A CTA's (sub-tile, chunk) is
// not its blockIdx but a ticket drawn on arrival (leaf_ticket): every lower
// ticket belongs to a CTA that is already resident, and lower chunks never wait
// on higher ones, so the chain progresses whatever order the hardware
// dispatches CTAs in.
constexpr int LEAF_M = 128;

// The launch's logical block index, in arrival order.  atomicInc wraps the
// counter back to 0 on the launch's last ticket, so consecutive launches on
// one counter (stream-ordered: each tile row / schedule has its own) need no
// reset; the fill zeroes the counters once with the flags.
__device__ __forceinline__ int leaf_ticket(unsigned *ticket) {
    __shared__ int s_ticket;
    if (threadIdx.x == 0) s_ticket = (int)atomicInc(ticket, gridDim.x - 1);
    __syncthreads();
    return s_ticket;
}
// right-range (column c, split cq < c) pairs of a sub-tile row staged in shared
// memory; the pair cq = c is the leaf cell C(t, t, m - wx[t-1]) of Eq. (1),
// computed in closed form instead (8 KB less per CTA)
constexpr int NPAIR = SB * (SB - 1) / 2;
constexpr int LEAF_MIN_BLOCKS = 8;  // 32 warps/SM for the latency-bound leaf (<= 64 registers)
#ifndef LEAF_RS_BLOCKS
#define LEAF_RS_BLOCKS 5  // k_sub_leaf_row<true>: 36 KB of staged operands per CTA, <= 96 registers
#endif

// (k_sub_leaf_diag: the diagonal sub-tiles of the diagonal tiles, delta = 0,
// phase 0; k_sub_leaf_row: every other sub-tile.)
__global__ void __launch_bounds__(LEAF_M, LEAF_MIN_BLOCKS)
    k_sub_leaf_diag(Problem p, int delta, int e, int *flags, int phase_id, int tile_lo, unsigned *ticket) {
    const int n = p.n;
    const int n_chunks = (p.S + 1 + LEAF_M - 1) / LEAF_M;
    const int cnt = sub_count(delta, e);
    const int bid = leaf_ticket(ticket);
    const int q = bid % n_chunks;
    const int sub = bid / n_chunks;  // tile I * cnt + sub-tile index
    int alpha, gamma;
    sub_at(delta, e, sub % cnt, alpha, gamma);
    const int I = tile_lo + sub / cnt;
    const int m = q * LEAF_M + threadIdx.x;
    // flags of this sub-tile: indexed by the ABSOLUTE tile row I (tiles of
    // different launches may be in flight at once, each with its own epochs)
    int *my_flags = flags + ((int64_t)I * NSB + sub % cnt) * n_chunks;
    for (int r = SB - 1; r >= 0; r--) {
        if (r < SB - 1) {
            const int need = (phase_id << 4) | (SB - 1 - r);  // rows SB-1 .. r+1 done
            for (int qq = threadIdx.x; qq < q; qq += LEAF_M) {
                int v;
                do {
                    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(my_flags + qq) : "memory");
                } while (v < need);
            }
            __syncthreads();
        }
        leaf_row_diag(p, alpha, I, r, m);
        __syncthreads();  // every thread of this chunk finished row r
        if (threadIdx.x == 0) {  // release (cumulative over the barrier): the chunk's row r is visible
            const int done = (phase_id << 4) | (SB - r);
            asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(my_flags + q), "r"(done) : "memory");
        }
    }
    // The last column c = i0 + TB - 1 of a diagonal tile is the A operand of a
    // middle's first split (s' = i0 + TB): its two bottom row groups lie in the
    // last diagonal sub-tile (A(s, c), s < c, written above by this thread;
    // A(c, c) by k_leaf), the others in off-diagonal sub-tiles (k_sub_leaf_row).
    if (alpha == NSB - 1 && m <= p.S) {
        const int s0 = I * TB + 1 + SB * alpha, c = s0 + SB - 1;
        if (c < n) {
#pragma unroll
            for (int h = 0; h < 2; h++) {
                float v = INFINITY;
#pragma unroll
                for (int k = 0; k < 4; k++) v = fminf(v, p.A32[shadow_index(p.sarows, srow_a(n, s0 + 4 * h + k, c), m)]);
                p.A32[shadow_index(p.sarows, sa_col(n, I, c) + kQuad + 2 * alpha + h, m)] = v;
            }
        }
    }
}

// Per-sub-tile scalars of an off-diagonal leaf, staged once in shared memory
// so the row path has no dependent global round trip.
struct LeafTab {
    int mnull[SB][SB], mall[SB][SB];  // m_null / m_all of cell (s0+r, t0+c); INT_MAX: no cell / gate shut
    int wxl[SB];                      // wxl[j] = wx[s0+j-1]: shift of the left split s' = s0+j
    int wxr[SB];                      // wxr[c] = wx[t0+c-1]: shift of the right split s' = t0+c
    int wself[SB];                    // wx[s0+r-1]: the C32 pre-shift of row r's cells
    int wbx[SB];                      // wbx[s0+r]: F_all shift of row r
    int mdiag[SB];                    // m_all(t0+c, t0+c) of the leaf cell C(t0+c, t0+c) (INT_MAX past the last stage)
    double wd[SB];                    // w[t0+c]: its value (Eq. 1)
    double w[SB], Ps[SB], Pt[SB];     // w[s0+r], P[s0+r-1], P[t0+c]
    int64_t crow[SB + 1];             // element offset of C cell (s0+j, t0) (columns t0+c follow, pitch apart)
    int64_t cleft[SB];                // 8 (crow[j] - wxl[j]): byte offset of the left split s' = s0+j's operand row, shifted
    int64_t cfall[SB];                // 8 (crow[r+1] - wbx[r]): byte offset of row r's F_all operand row, shifted
    int64_t arow[SB];                 // element offset of A(s0+r, t0-1)
    int64_t aleft[SB][SB - 1];        // element offset of A(s0+r, s0+r+k) (left split s' = s0+r+k+1)
    int q_lo;                         // lowest m-chunk a shifted read of a row below can reach
};

__device__ __forceinline__ void leaf_tab_fill(const Problem &p, int s0, int t0, int m0, int chunk_m, LeafTab &T) {
    const int n = p.n;
    if (threadIdx.x < SB * SB) {
        const int rr = threadIdx.x / SB, cc = threadIdx.x % SB, ss = s0 + rr, tt = t0 + cc;
        const bool ok = ss <= n && tt <= n;  // ss < tt in an off-diagonal sub-tile
        T.mnull[rr][cc] = ok ? m_null(p, ss, tt) : INT_MAX;
        T.mall[rr][cc] = ok && !p.restricted ? m_all(p, ss, tt) : INT_MAX;
        if (cc == 0) {
            const bool row = ss < n;  // rows s < t <= n
            T.wxl[rr] = rr > 0 && ss <= n ? p.wx[ss - 1] : 0;
            T.wself[rr] = ss <= n ? p.wx[ss - 1] : 0;
            T.wxr[rr] = t0 + rr <= n ? p.wx[t0 + rr - 1] : 0;
            T.mdiag[rr] = t0 + rr <= n ? m_all(p, t0 + rr, t0 + rr) : INT_MAX;
            T.wd[rr] = t0 + rr <= n ? p.w[t0 + rr] : 0.0;
            T.wbx[rr] = row ? p.wbx[ss] : 0;
            T.w[rr] = row ? p.w[ss] : 0.0;
            T.Ps[rr] = ss <= n ? p.P[ss - 1] : 0.0;
            T.Pt[rr] = p.P[min(t0 + rr, n)];
            T.arow[rr] = ss <= n ? a_index(ss, t0 - 1) * p.pitch : 0;
        }
        if (cc < SB - 1) T.aleft[rr][cc] = ss + cc < n ? a_index(ss, ss + cc) * p.pitch : 0;
        if (threadIdx.x <= SB) T.crow[threadIdx.x] = s0 + (int)threadIdx.x <= n
                                                          ? cell_index(n, s0 + threadIdx.x, t0) * p.pitch : 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int wmax = 0;
        for (int k = 0; k < SB; k++) wmax = max(wmax, max(T.wxl[k], T.wbx[k]));
        T.q_lo = m0 - wmax <= 0 ? 0 : (m0 - wmax) / chunk_m;
    } else if (threadIdx.x <= SB) {  // one 64-bit offset per operand row instead of two loads + an add per candidate
        const int k = threadIdx.x - 1;
        T.cleft[k] = (T.crow[k] - T.wxl[k]) * 8;
        T.cfall[k] = (T.crow[k + 1] - T.wbx[k]) * 8;
    }
    __syncthreads();
}

// Off-diagonal leaf row r at one m (thread = m), scalars from the table; the
// same arithmetic as the wavefront's Eq. (2) for the in-sub-tile splits.
// r: the row index as a compile-time constant (every loop trimmed and fully
// unrolled: 8 row bodies, ~26 KB of SASS each; one runtime-row body, 3.6x less
// code, measured slower in the tile-DAG schedule too: 143.2 vs 131.1 ms per solve)
// qa: the running quad minima of the sub-tile's columns over the rows of the
// current 4-row group (k_sub_leaf_row writes them after rows 4 and 0).
template <int r, bool RS, class Wait, class Lap>
__device__ __forceinline__ void leaf_row_tab(const Problem &p, const LeafTab &T, bool fresh, bool partial, int s0,
                                             int t0, int m, bool live, const double *Rs, float (&qa)[SB], Wait wait,
                                             Lap after_pass1) {
    const int n = p.n;
    const int64_t pitch = p.pitch;
    const int s = s0 + r;
    // operands written by earlier launches first — their loads are in flight
    // during the look-back wait: A(s, ·) of the left splits, A(s, t0-1), and
    // the partial minimum of the row's cells
    // addresses from the staged row offsets: cells (s, t0+c) are consecutive rows
    double *Cm = p.C + m;
    double AL[SB - 1];  // AL[k] = A(s, s + k): left split s' = s + k + 1 <= ea
#pragma unroll
    for (int k = 0; k < SB - 1; k++)
        AL[k] = (live && k < SB - 1 - r) ? ld(p.A + T.aleft[r][k] + m, fresh) : INFINITY;
    double AR[SB + 1];  // AR[c] = A(s, t0 + c - 1)
    AR[0] = live ? __ldcg(p.A + T.arow[r] + m) : INFINITY;
    double B[SB], F[SB];
    bool gate[SB];
    const int64_t crow = T.crow[r];
    {
        const double *pb = Cm + crow;
#pragma unroll
        for (int c = 0; c < SB; c++) {
            gate[c] = live && m >= T.mnull[r][c];  // INT_MAX past the last stage
            B[c] = (gate[c] && partial) ? __ldcg(pb) : INFINITY;
            pb += pitch;
        }
    }
    wait();  // the rows below are complete at every m this row reads (flags + barrier)
    if (!live) return;
    // byte addressing with a running column pointer: per candidate one
    // shared-memory offset, one 64-bit add and the load (the element-index form
    // recomputed pitch * c and scaled for every load)
    const char *colb = reinterpret_cast<const char *>(Cm);
    const int64_t pitch_b = pitch * 8;
#pragma unroll
    for (int c = 0; c < SB; c++) {
        double best = B[c];
        if (gate[c]) {
#pragma unroll
            for (int k = 0; k < SB - 1; k++) {  // left: C of the rows below in this sub-tile
                if (k >= SB - 1 - r) break;
                const int j = r + k + 1;  // s' = s0 + j
                const double cv = __ldcg(reinterpret_cast<const double *>(colb + T.cleft[j]));
                best = dmin(best, __dadd_rn(AL[k], cv));
            }
        }
        B[c] = best;
        F[c] = m >= T.mall[r][c] ? __dadd_rn(T.w[r], __ldcg(reinterpret_cast<const double *>(colb + T.cfall[r])))
                                 : INFINITY;
        colb += pitch_b;
    }
    after_pass1();               // (timing only)
    if (RS) cp_async_wait<0>();  // this thread's right-range operands are in shared memory
    // the row's outputs, addressed incrementally: cells (s, t0+c) are consecutive
    // C rows, and consecutive C32 shadow rows (pre-shifted by wx[s-1]) followed
    // by the row's quad minima; A(s, t) -> A(s, t+1) is t rows further on
    // (a_index), kSR shadow rows (srow_a)
    const int w = T.wself[r];
    const int J = (t0 - 1) / TB;
    const int64_t c_row32 = sc_row(J, s) + (t0 - 1 - TB * J);
    const int64_t q_row32 = sc_row(J, s) + kQuad + (t0 - 1 - TB * J) / 4;  // the row's two column groups
    float *c32_hi = (m + w <= p.S) ? p.C32 + shadow_index(p.scrows, c_row32, m + w) : nullptr;
    float *c32_lo = (m < w) ? p.C32 + shadow_index(p.scrows, c_row32, m) : nullptr;
    float *q32_hi = (m + w <= p.S) ? p.C32 + shadow_index(p.scrows, q_row32, m + w) : nullptr;
    float *q32_lo = (m < w) ? p.C32 + shadow_index(p.scrows, q_row32, m) : nullptr;
    float qc[2] = {INFINITY, INFINITY};
    // running output pointers: C(s, t) -> C(s, t+1) one row, A(s, t) -> A(s, t+1)
    // t rows (a_index), A32 kSR shadow rows = kSR * kSW floats
    double *pc = Cm + crow;
    double *pa = p.A + a_index(s, t0) * pitch + m;
    int64_t a_step = (int64_t)t0 * pitch;
    float *pa32 = p.A32 + shadow_index(p.sarows, srow_a(n, s, t0), m);
#pragma unroll
    for (int c = 0; c < SB; c++) {
        const int t = t0 + c;
        if (t > n) break;
        double c1 = INFINITY;
        if (gate[c]) {
            double best = B[c];
#pragma unroll
            for (int cq = 0; cq < SB; cq++) {  // right: s' = t0 + cq <= t
                if (cq > c) break;
                double cv;
                if (cq == c)  // the leaf cell C(t, t, m - wx[t-1]), Eq. (1)
                    cv = m - T.wxr[c] >= T.mdiag[c] ? T.wd[c] : INFINITY;
                else
                    cv = RS ? Rs[(c * (c - 1) / 2 + cq) * LEAF_M + threadIdx.x]
                            : ld(&p.C[cell_index(n, t0 + cq, t) * pitch + (m - T.wxr[cq])], fresh);
                best = dmin(best, __dadd_rn(AR[cq], cv));
            }
            c1 = best;
        }
        const double cc = dmin(c1, F[c]);
        *pc = cc;  // store_final_c, unrolled
        pc += pitch;
        const float c32 = __double2float_rd(cc);
        if (c32_hi) c32_hi[c * kSW] = c32;
        if (c32_lo) c32_lo[c * kSW] = INFINITY;
        qc[c / 4] = fminf(qc[c / 4], c32);
        const double a = __dadd_rn(__dadd_rn(T.Pt[c], -T.Ps[r]), cc);
        if (t < n) {  // store_final_a
            const float a32 = __double2float_rd(a);
            *pa = a;
            *pa32 = a32;
            qa[c] = fminf(qa[c], a32);
        }
        pa += a_step;
        a_step += pitch;
        pa32 += kSR * kSW;
        AR[c + 1] = a;
    }
    // the row's two column-group minima (a group with no cell: +inf)
    if (q32_hi) {
        q32_hi[0] = qc[0];
        q32_hi[kSW] = qc[1];
    }
    if (q32_lo) {
        q32_lo[0] = INFINITY;
        q32_lo[kSW] = INFINITY;
    }
}

// (CTA width measured: 64 m 247.1, 128 m 238.9, 256 m 239.7 ms per solve; one
// runtime-row body instead of 8 unrolled row copies (17 K instructions, ncu
// shows instruction-fetch stalls) measured slower: 238.1 vs 228.8.)
// RS: the right-range operands R[c][cq] = C(t0+cq, t0+c, m - wx[t0+cq-1]),
// the same for every row, are loaded once into shared memory (thread-private
// columns, NPAIR x LEAF_M doubles) instead of once per row.
template <bool RS, bool TIMED = false>
__global__ void __launch_bounds__(LEAF_M, RS ? LEAF_RS_BLOCKS : LEAF_MIN_BLOCKS) k_sub_leaf_row(Problem p, int delta, int e, int *flags,
                                                                        int phase_id, int tile_lo, unsigned *ticket) {
    __shared__ LeafTab T;
    extern __shared__ double Rsm[];  // [NPAIR][LEAF_M] when RS
    const int n = p.n;
    const int n_chunks = (p.S + 1 + LEAF_M - 1) / LEAF_M;
    const int cnt = sub_count(delta, e);
    // time split (options.counters; thread 0, global timer): setup / look-back
    // wait / row work / barrier + release, summed into counters 24..28
    constexpr bool timed = TIMED;  // (the counters solve only: the timing state costs registers)
    unsigned long long tm0 = 0, t_wait = 0, t_work = 0, t_sync = 0, t_pass1 = 0;
    if (timed && threadIdx.x == 0) tm0 = gtimer();
    const int bid = leaf_ticket(ticket);  // before any early exit: every CTA draws one
    const int q = bid % n_chunks;
    const int sub = bid / n_chunks;
    int alpha, gamma;
    sub_at(delta, e, sub % cnt, alpha, gamma);
    const int I = tile_lo + sub / cnt, J = I + delta;
    const int s0 = I * TB + 1 + SB * alpha, t0 = J * TB + 1 + SB * gamma;
    if (s0 > n || t0 > n) return;  // no cells (uniform over the sub-tile)
    const int m = q * LEAF_M + threadIdx.x;
    const bool fresh = (delta == 0);
    const bool partial = delta == 0 ? (e >= 2) : (delta >= 2 || alpha < NSB - 1 || gamma > 0);
    int *my_flags = flags + ((int64_t)I * NSB + sub % cnt) * n_chunks;  // by absolute tile row (see k_sub_leaf_diag)
    leaf_tab_fill(p, s0, t0, q * LEAF_M, LEAF_M, T);
    const int q_lo = T.q_lo;
    if (RS) {
        const int64_t pitch = p.pitch;
#pragma unroll
        for (int c = 0; c < SB; c++)
#pragma unroll
            for (int cq = 0; cq < c; cq++) {
                const int t = t0 + c, w = T.wxr[cq];
                double *dst = &Rsm[(c * (c - 1) / 2 + cq) * LEAF_M + threadIdx.x];
                if (m <= p.S && t <= n && m >= w)  // lands while the first row's pass 1 runs
                    cp_async8(dst, &p.C[cell_index(n, t0 + cq, t) * pitch + (m - w)]);
                else
                    *dst = INFINITY;
            }
        cp_async_commit();
    }
    float qa[SB];  // quad minima of the columns over the current 4-row group
#pragma unroll
    for (int c = 0; c < SB; c++) qa[c] = INFINITY;
    unsigned long long tm = (timed && threadIdx.x == 0) ? gtimer() : 0;
    const unsigned long long t_setup = tm - tm0;
    auto lap = [&](unsigned long long &acc) {
        if (timed && threadIdx.x == 0) {
            const unsigned long long x = gtimer();
            acc += x - tm;
            tm = x;
        }
    };
#pragma unroll
    for (int r = SB - 1; r >= 0; r--) {
        auto wait = [&]() {  // uniform over the CTA (every thread calls it once per row)
            lap(t_work);
            if (r == SB - 1) return;
            const int need = (phase_id << 4) | (SB - 1 - r);  // rows SB-1 .. r+1 done
            for (int qq = q_lo + (int)threadIdx.x; qq < q; qq += LEAF_M) {
                int v;
                do {
                    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(my_flags + qq) : "memory");
                } while (v < need);
            }
            __syncthreads();
            lap(t_wait);
        };
        auto pass1 = [&]() { lap(t_pass1); };
        const bool live = m <= p.S;
        if (s0 + r > n) {  // no such row (uniform)
            wait();
        } else {
            switch (r) {  // compile-time row index: the row's loops fully unrolled
                case 0: leaf_row_tab<0, RS>(p, T, fresh, partial, s0, t0, m, live, Rsm, qa, wait, pass1); break;
                case 1: leaf_row_tab<1, RS>(p, T, fresh, partial, s0, t0, m, live, Rsm, qa, wait, pass1); break;
                case 2: leaf_row_tab<2, RS>(p, T, fresh, partial, s0, t0, m, live, Rsm, qa, wait, pass1); break;
                case 3: leaf_row_tab<3, RS>(p, T, fresh, partial, s0, t0, m, live, Rsm, qa, wait, pass1); break;
                case 4: leaf_row_tab<4, RS>(p, T, fresh, partial, s0, t0, m, live, Rsm, qa, wait, pass1); break;
                case 5: leaf_row_tab<5, RS>(p, T, fresh, partial, s0, t0, m, live, Rsm, qa, wait, pass1); break;
                case 6: leaf_row_tab<6, RS>(p, T, fresh, partial, s0, t0, m, live, Rsm, qa, wait, pass1); break;
                default: leaf_row_tab<7, RS>(p, T, fresh, partial, s0, t0, m, live, Rsm, qa, wait, pass1); break;
            }
        }
        if ((r & 3) == 0 && live) {  // rows r..r+3 done: the columns' quad minima (A(s, t) exists for t < n)
            const int64_t q0 = sa_col(n, I, t0) + kQuad + (s0 - 1 - TB * I + r) / 4;
#pragma unroll
            for (int c = 0; c < SB; c++) {
                if (t0 + c < n) p.A32[shadow_index(p.sarows, q0 + (int64_t)c * kSR, m)] = qa[c];
                qa[c] = INFINITY;
            }
        }
        lap(t_work);
        __syncthreads();
        if (threadIdx.x == 0)
            asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(my_flags + q), "r"((phase_id << 4) | (SB - r))
                         : "memory");
        lap(t_sync);
    }
    if (timed && threadIdx.x == 0) {
        atomicAdd(p.counters + 24, 1ull);
        atomicAdd(p.counters + 25, t_setup);
        atomicAdd(p.counters + 26, t_wait);
        atomicAdd(p.counters + 27, t_work);
        atomicAdd(p.counters + 28, t_sync);
        atomicAdd(p.counters + 29, t_pass1);
    }
}

// (Rejected variants, measured and removed: a column-parallel leaf — thread =
// (m, column), the row chain by warp shuffles, 327 vs 291 ms — and a leaf with
// both the right-range operands and its own results in shared memory, 147 vs
// 119 ms at the time; profiles/r01_tiled_v4.md, r01_tiled_v5.md.)

// Flags of the leaf look-back: one int per (tile row I, sub-tile of a phase,
// m-chunk), then one ticket counter per tile row (indexed by the launch's
// tile_lo: the DAG's row, the diagonal schedule's / a shard's first row).
inline size_t leaf_flag_words(int L, int S) {
    const int nb = (L + 1 + TB - 1) / TB;
    const int chunks = (S + 1 + LEAF_M - 1) / LEAF_M;
    return (size_t)nb * NSB * chunks;
}
inline size_t leaf_flag_bytes(int L, int S) {
    const int nb = (L + 1 + TB - 1) / TB;
    return (leaf_flag_words(L, S) + nb) * sizeof(int);
}

// Off-diagonal leaf kernel: k_sub_leaf_row<true> (the right-range operands
// staged in shared memory; the default, the fastest measured) or
// k_sub_leaf_row<false> (ROTOR_LEAF=tab, for A/B measurements).  (A third
// variant with the scalars read from global memory was removed in round 2.)
inline bool leaf_staged() {
    static const bool v = [] {
        const char *e = getenv("ROTOR_LEAF");
        return !(e && !strcmp(e, "tab"));
    }();
    return v;
}

// Product kernel: ROTOR_PROD=2 k_sub_product_async at 3 CTAs/SM (default:
// 222.4 ms per config-4 solve), 1 the same at 4 CTAs/SM (223.2); a variant
// with the operands through registers (231.4) was removed.
constexpr int PRODUCT_MINB_DEFAULT = 2;
inline int product_minb() {
    static const int v = [] {
        const char *e = getenv("ROTOR_PROD");
        return e ? atoi(e) : PRODUCT_MINB_DEFAULT;
    }();
    return v;
}

// Launch the dependent phase of tile diagonal delta; returns the launch count.
// phase_id: running counter of leaf launches in this solve (flags zeroed at
// the start of the fill, so phase ids >= 1 never match stale values).
// Tiles I in [tile_lo, tile_hi) of the diagonal (all of them in a single-GPU solve;
// a rank's share in a sharded one).
inline int launch_dependent(const Problem &p, int delta, int tile_lo, int tile_hi, cudaStream_t st, int *flags,
                            int &phase_id) {
    const int ntiles = tile_hi - tile_lo;
    if (ntiles <= 0) return 0;
    const int n_mg = (p.S + 1 + 15) / 16;  // product: a warp per (sub-tile, 16 m)
    const int n_chunks = (p.S + 1 + LEAF_M - 1) / LEAF_M;
    const int phases = delta == 0 ? NSB : 2 * NSB - 1;
    int launches = 0;
    for (int e = 0; e < phases; e++) {
        const int cnt = sub_count(delta, e);
        const int warps = ntiles * cnt * n_mg;
        const int blocks = (warps * 32 + DEP_THREADS - 1) / DEP_THREADS;
        bool has_product;
        if (delta == 0) {
            has_product = e >= 2;
        } else if (delta >= 2) {
            has_product = true;  // every sub-tile: at least the middle's recorded splits (mlist)
        } else {
            int a, g;
            sub_at(delta, e, 0, a, g);
            has_product = !(cnt == 1 && a == NSB - 1 && g == 0);
        }
        if (has_product) {
            if (product_minb() == 1)
                k_sub_product_async<4><<<blocks, DEP_THREADS, 0, st>>>(p, delta, e, tile_lo, ntiles);
            else
                k_sub_product_async<3><<<blocks, DEP_THREADS, 0, st>>>(p, delta, e, tile_lo, ntiles);
            launches++;
        }
        const int lb = ntiles * cnt * n_chunks;
        unsigned *ticket = reinterpret_cast<unsigned *>(flags + leaf_flag_words(p.L, p.S)) + tile_lo;
        if (delta == 0 && e == 0)
            k_sub_leaf_diag<<<lb, LEAF_M, 0, st>>>(p, delta, e, flags, ++phase_id, tile_lo, ticket);
        else if (leaf_staged() && p.counters)
            k_sub_leaf_row<true, true><<<lb, LEAF_M, NPAIR * LEAF_M * 8, st>>>(p, delta, e, flags, ++phase_id, tile_lo,
                                                                                ticket);
        else if (leaf_staged())
            k_sub_leaf_row<true><<<lb, LEAF_M, NPAIR * LEAF_M * 8, st>>>(p, delta, e, flags, ++phase_id, tile_lo, ticket);
        else
            k_sub_leaf_row<false><<<lb, LEAF_M, 0, st>>>(p, delta, e, flags, ++phase_id, tile_lo, ticket);
        launches++;
    }
    return launches;
}
