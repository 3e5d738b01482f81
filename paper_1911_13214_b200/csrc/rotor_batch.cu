// Fused batched solver: many independent (chain, limit)
// tables — the paper's multi-limit sweep, "Algorithm 1 for 10 different memory
// limits" — in ONE launch.  A persistent CTA takes problems from an
// atomic queue (handed out longest chain first, so the tail is short) and runs
// the whole path for each inside its own workspace slot:
// precompute (discretisation with that limit's slot size M/S),
// leaf, every diagonal d (barrier between diagonals), Algorithm-2 walk.  The
// per-cell arithmetic is the wavefront kernel's (rotor_device.cuh) with
// candidates skipped by an exact monotone-in-m bound (batch_cell_group): the
// minimum is the same set's, so every table is bit-identical to a single solve.
#include "rotor_device.cuh"
#include "rotor_kernels.cuh"

namespace rotor {

// Slot layout for chains of at most L_max stages (all offsets 256 B aligned).
struct SlotLayout {
    int64_t pitch, rows;
    size_t off_i32[5], off_P, off_w, off_mnull, off_stack, off_C, bytes;
    int stack_cap;
};

__host__ __device__ inline size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

__host__ __device__ inline SlotLayout slot_layout(int L_max, int S) {
    SlotLayout y;
    const int64_t n = (int64_t)L_max + 1;
    y.pitch = ((int64_t)kPad + S + 1 + 31) / 32 * 32;
    y.rows = n * (n + 1) / 2;
    y.stack_cap = (int)(4 * n + 64);
    size_t off = 0;
    for (int i = 0; i < 5; i++) {
        y.off_i32[i] = off;
        off += al256((size_t)(n + 2) * 4);
    }
    y.off_P = off;
    off += al256((size_t)(n + 2) * 8);
    y.off_w = off;
    off += al256((size_t)(n + 2) * 8);
    y.off_mnull = off;
    off += al256((size_t)(n * n) * 4);
    y.off_stack = off;
    off += al256((size_t)y.stack_cap * 16);
    y.off_C = off;
    off += al256((size_t)(y.rows + kPadRows) * y.pitch * 8);
    y.bytes = off;
    return y;
}

// One warp computes the cells (s, t, mlo .. mlo+31) (lanes past mend idle) —
// the same value as wavefront_cell for each, with candidates skipped by an
// exact bound.  C(s', t', m) is nonincreasing in m (Eq. 1-2: every operand
// index m or m - w grows with m, the feasibility thresholds m_null/m_all and
// the leaf threshold only admit more options, the min of nonincreasing terms
// is nonincreasing, and fl(a + b) is monotone in a and b), so for the NS
// groups of 32/NS lanes (consecutive m), with mtop a group's largest m,
//   lb_k = fl(fl(U_k + C[s,s+k-1,mtop]) + C[s+k,t,mtop-wx[s+k-1]])
// is <= candidate k's value at every m of the group.  Candidate k cannot
// lower any of the group's minima when lb_k >= the group's largest current
// best; the group then skips its loads of k (two 8-byte bounds instead of two
// 8*32/NS-byte row pieces).  Lane (q, c) bounds candidate k0 + c for group q,
// CB = 32/NS candidates per pass; the candidate with the least bound and C_2
// (F_all) are evaluated first so that the others meet a good best.  The batch
// keeps no D table, so only the minimum value matters and any evaluation
// order gives the same bits.
template <int NS>
__device__ __forceinline__ void batch_cell_group(const Problem &p, int s, int t, int mlo, int mend, int lane) {
    constexpr int CB = 32 / NS;
    const int n = p.n;
    const int64_t pitch = p.pitch;
    const int m = mlo + lane;
    const bool live = m < mend;
    const int mhi = min(mlo + 31, mend - 1);
    const int mn = m_null(p, s, t);
    const bool act = live && m >= mn;
    // C_2 (F_all): its load is issued here and consumed after the first bounds
    const bool fa = !p.restricted && live && m >= m_all(p, s, t);
    const int mma = m - p.wbx[s];
    double sub = INFINITY;
    if (fa && mma >= 0) sub = p.C[cell_index(n, s + 1, t) * pitch + mma];
    double best = INFINITY;
    if (mhi < mn) {
        if (fa) best = __dadd_rn(p.w[s], sub);
    } else {  // warp-uniform: lane mhi - mlo is active
        const int q = lane / CB, c = lane % CB;
        const int mtop = min(mlo + (q + 1) * CB - 1, mend - 1);
        const bool gact = mtop >= max(mlo + q * CB, mn);  // group q has an active lane
        const double Ps = p.P[s - 1];
        const int d = t - s;
        const int rs = (int)cell_index(n, s, s);
        for (int k0 = 1; k0 <= d; k0 += CB) {
            const int k = k0 + c;
            double U = 0.0, lb = INFINITY;
            int prow = 0, srow = 0, wxs = 0;
            if (k <= d) {
                const int sp = s + k;
                U = __dadd_rn(p.P[sp - 1], -Ps);
                wxs = p.wx[sp - 1];
                prow = rs + k - 1;
                srow = (int)cell_index(n, sp, t);
                const int mmh = mtop - wxs;
                if (gact && mmh >= 0)
                    lb = __dadd_rn(__dadd_rn(U, p.C[(int64_t)prow * pitch + mtop]), p.C[(int64_t)srow * pitch + mmh]);
            }
            unsigned skip = 0;
            if (k0 == 1) {  // seed: the least bound over all groups (lowest lane on ties)
                if (fa) best = __dadd_rn(p.w[s], sub);
                double v = lb;
                int j = lane;
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
                    const int j2 = __shfl_xor_sync(0xffffffffu, j, o);
                    if (v2 < v || (v2 == v && j2 < j)) {
                        v = v2;
                        j = j2;
                    }
                }
                j %= CB;
                if (v < INFINITY) {
                    const double Uj = __shfl_sync(0xffffffffu, U, j);
                    const int pj = __shfl_sync(0xffffffffu, prow, j);
                    const int sj = __shfl_sync(0xffffffffu, srow, j);
                    const int wj = __shfl_sync(0xffffffffu, wxs, j);
                    if (act) {
                        const int mm = m - wj;
                        const double suf = (mm >= 0) ? p.C[(int64_t)sj * pitch + mm] : INFINITY;
                        best = fmin(best, __dadd_rn(__dadd_rn(Uj, p.C[(int64_t)pj * pitch + m]), suf));
                    }
                }
                skip = 1u << j;
            }
            double B = act ? best : -INFINITY;  // group max of the current minima
#pragma unroll
            for (int o = CB / 2; o; o >>= 1) B = fmax(B, __shfl_xor_sync(0xffffffffu, B, o));
            const unsigned ball = __ballot_sync(0xffffffffu, k <= d && lb < B);
            const unsigned cm = CB == 32 ? 0xffffffffu : (1u << CB) - 1;
            unsigned need = 0;
#pragma unroll
            for (int g = 0; g < NS; g++) need |= (ball >> (g * CB)) & cm;
            need &= ~skip;
            const unsigned mine = (ball >> (q * CB)) & cm;
            while (need) {  // two candidates per pass: twice the loads in flight per warp
                const int j = __ffs(need) - 1;
                need &= need - 1;
                const int j2 = need ? __ffs(need) - 1 : j;  // odd count: j again (min is idempotent)
                need &= need - 1;
                const double Uj = __shfl_sync(0xffffffffu, U, j), Uj2 = __shfl_sync(0xffffffffu, U, j2);
                const int pj = __shfl_sync(0xffffffffu, prow, j), pj2 = __shfl_sync(0xffffffffu, prow, j2);
                const int sj = __shfl_sync(0xffffffffu, srow, j), sj2 = __shfl_sync(0xffffffffu, srow, j2);
                const int wj = __shfl_sync(0xffffffffu, wxs, j), wj2 = __shfl_sync(0xffffffffu, wxs, j2);
                const bool e1 = act && ((mine >> j) & 1u), e2 = act && ((mine >> j2) & 1u);
                const int mm = m - wj, mm2 = m - wj2;
                double pr = INFINITY, sf = INFINITY, pr2 = INFINITY, sf2 = INFINITY;
                if (e1) pr = p.C[(int64_t)pj * pitch + m];
                if (e1 && mm >= 0) sf = p.C[(int64_t)sj * pitch + mm];
                if (e2) pr2 = p.C[(int64_t)pj2 * pitch + m];
                if (e2 && mm2 >= 0) sf2 = p.C[(int64_t)sj2 * pitch + mm2];
                if (e1) best = fmin(best, __dadd_rn(__dadd_rn(Uj, pr), sf));
                if (e2) best = fmin(best, __dadd_rn(__dadd_rn(Uj2, pr2), sf2));
            }
        }
    }
    if (live) p.C[cell_index(n, s, t) * pitch + m] = best;
}

template <int NS>
__device__ __forceinline__ void batch_fill_chunk(const Problem &p, int L, int m0, int wm) {
    const int n = L + 1, G = (wm + 31) >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int d = 1; d <= L; d++) {
        for (int it = wid; it < (n - d) * G; it += blockDim.x >> 5) {
            const int s = 1 + it / G;
            batch_cell_group<NS>(p, s, s + d, m0 + 32 * (it % G), m0 + wm, lane);
        }
        __syncthreads();
    }
}

#ifndef BATCH_MINB
#define BATCH_MINB 3  // config 5 (pruned, 64-m chunks), ms per sweep: 2 per SM 19.1, 3 18.3, 4 19.2 (spills at 32 registers)
#endif
int batch_ctas_per_sm() { return BATCH_MINB; }

__global__ void __launch_bounds__(512, BATCH_MINB) k_batch(BatchArgs b) {  // BATCH_MINB resident per SM (rotor_abi.cu)
    __shared__ int prob;
    const SlotLayout y = slot_layout(b.L_max, b.S);
    char *slot = b.pool + (size_t)blockIdx.x * y.bytes;
    while (true) {
        if (threadIdx.x == 0) {
            const int k = atomicAdd(b.counter, 1);
            prob = k < b.n_problems ? b.order[k] : b.n_problems;
        }
        __syncthreads();
        const int pi = prob;
        __syncthreads();
        if (pi >= b.n_problems) break;
        const int ci = b.prob_chain[pi];
        const int L = b.chain_L[ci];
        const int64_t co = (int64_t)ci * b.chain_stride;
        rotor_chain ch;
        ch.uf = b.uf + co;
        ch.ub = b.ub + co;
        ch.wx = b.wx + co;
        ch.wbx = b.wbx + co;
        ch.wy = b.wy + co;
        ch.of = b.of + co;
        ch.ob = b.ob + co;
        Problem p{};
        p.L = L;
        p.n = L + 1;
        p.S = b.S;
        p.restricted = b.restricted;
        p.pitch = y.pitch;
        p.wx = (int32_t *)(slot + y.off_i32[0]);
        p.wbx = (int32_t *)(slot + y.off_i32[1]);
        p.wy = (int32_t *)(slot + y.off_i32[2]);
        p.of = (int32_t *)(slot + y.off_i32[3]);
        p.ob = (int32_t *)(slot + y.off_i32[4]);
        p.P = (double *)(slot + y.off_P);
        p.w = (double *)(slot + y.off_w);
        p.mnullT = (int32_t *)(slot + y.off_mnull);
        p.stack = (int4 *)(slot + y.off_stack);
        p.stack_cap = y.stack_cap;
        p.C = (double *)(slot + y.off_C) + kPad;
        p.D = nullptr;
        p.A = nullptr;
        p.res_cost = b.cost + pi;
        p.res_nops = b.nops + pi;
        p.res_status = b.status + pi;
        p.ops = b.ops ? b.ops + b.ops_off[pi] : nullptr;
        p.ops_cap = b.ops ? b.ops_cap[pi] : 0;

        precompute_cta(ch, b.limits[pi], p);
        const int n = p.n, W = b.S + 1;
        for (int idx = threadIdx.x; idx < n * W; idx += blockDim.x) leaf_cell(p, 1 + idx / W, idx % W);
        __syncthreads();
        // m-chunk-major order (b.mc m at a time, every diagonal of the chunk
        // before the next chunk): valid because every operand lies at the same m
        // (prefix C(s, s'-1, m), a shorter diagonal) or at a lower m (suffix and
        // F_all at m - shift); the chunk's slice of the table stays in L2 while
        // its diagonals run, instead of the whole table streaming per diagonal
        const int mc = b.mc > 0 ? b.mc : W;
        for (int m0 = 0; m0 < W; m0 += mc) {
            const int wm = min(mc, W - m0);
            if (b.prune == 1) {
                batch_fill_chunk<1>(p, L, m0, wm);
            } else if (b.prune == 2) {
                batch_fill_chunk<2>(p, L, m0, wm);
            } else if (b.prune == 4) {
                batch_fill_chunk<4>(p, L, m0, wm);
            } else {
                for (int d = 1; d <= L; d++) {
                    for (int idx = threadIdx.x; idx < (n - d) * wm; idx += blockDim.x) {
                        const int s = 1 + idx / wm;
                        wavefront_cell(p, s, s + d, m0 + idx % wm);
                    }
                    __syncthreads();
                }
            }
        }
        reconstruct_cta(p);
    }
}

size_t batch_slot_bytes(int L_max, int S) { return slot_layout(L_max, S).bytes; }

// Gather every problem's ops (src + src_off[k], cnt[k] of them) into one
// contiguous array (dst + dst_off[k]) for a single device-to-host copy.
__global__ void k_compact_ops(const rotor_op *src, const int64_t *src_off, const int64_t *cnt, const int64_t *dst_off,
                              rotor_op *dst, int P) {
    for (int k = blockIdx.x; k < P; k += gridDim.x) {
        const rotor_op *a = src + src_off[k];
        rotor_op *b = dst + dst_off[k];
        for (int64_t i = threadIdx.x; i < cnt[k]; i += blockDim.x) b[i] = a[i];
    }
}

void launch_compact_ops(const rotor_op *src, const int64_t *src_off, const int64_t *cnt, const int64_t *dst_off,
                        rotor_op *dst, int P, cudaStream_t st) {
    k_compact_ops<<<P < 1024 ? P : 1024, 128, 0, st>>>(src, src_off, cnt, dst_off, dst, P);
}

void launch_batch(const BatchArgs &b, int n_slots, cudaStream_t st) { k_batch<<<n_slots, 512, 0, st>>>(b); }

}  // namespace rotor
