// Device building blocks of the solver, shared by the per-table kernels
// (rotor_kernels.cu) and the fused batched kernel (rotor_batch.cu).
//
// PAPER.md: discretisation §5.2; limits P:702-715; Theorem 1
// P:717-739; Algorithm 1; Algorithm 2 P:829-847.  Readings (fill
// order Q3, F_null range Q4, top budget Q5, m domain Q6, rounding Q7, tie rule
// Q11, fp64 association Q12, infinity Q13) in DESIGN.md §3.
#pragma once
#include <math.h>

#include "rotor_common.cuh"

namespace rotor {

// ceil(x * S / M) exactly (128-bit), clamped to S+1: any size above S slots
// behaves identically (every gate containing it fails, every shift by it lands
// below m = 0).  §5.2, Q7.
__device__ __forceinline__ int32_t slots_of(uint64_t x, uint64_t M, int S) {
    unsigned __int128 num = (unsigned __int128)x * (unsigned)S + (M - 1);
    unsigned __int128 q = num / M;
    return q > (unsigned __int128)(S + 1) ? (S + 1) : (int32_t)q;
}

// Discretise sizes, prefix sums P, w, m_null table.  Called by every thread of
// one CTA; ends with the status written to *p.res_status.
__device__ __forceinline__ void precompute_cta(const rotor_chain &ch, uint64_t M, const Problem &p) {
    const int n = p.n, L = p.L, S = p.S;
    __shared__ int bad;
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    for (int l = threadIdx.x; l <= n; l += blockDim.x) {
        if (l <= L) p.wx[l] = slots_of(ch.wx[l], M, S);
        p.wy[l] = slots_of(ch.wy[l], M, S);
        if (l >= 1) {
            p.wbx[l] = slots_of(ch.wbx[l - 1], M, S);
            p.of[l] = slots_of(ch.of[l - 1], M, S);
            p.ob[l] = slots_of(ch.ob[l - 1], M, S);
            double a = ch.uf[l - 1], b = ch.ub[l - 1];
            if (!(a >= 0.0 && a < INFINITY) || !(b >= 0.0 && b < INFINITY)) bad = 1;
            p.w[l] = __dadd_rn(a, b);  // w_s = fl(uf + ub)  (Q12)
        }
    }
    if (threadIdx.x == 0) {  // P[k] = fl(P[k-1] + uf[k]), sequential (Q12)
        double acc = 0.0;
        p.P[0] = 0.0;
        for (int k = 1; k <= n; k++) {
            acc = __dadd_rn(acc, ch.uf[k - 1]);
            p.P[k] = acc;
        }
    }
    __syncthreads();
    // m_null(s,t) = wy[t] + max(wx[s] + of[s], max_{s<j<t} (wx[j-1] + wx[j] + of[j]))
    for (int s = 1 + threadIdx.x; s <= n; s += blockDim.x) {
        const int base = p.wx[s <= L ? s : L] + p.of[s];
        int run = -1;
        for (int t = s + 1; t <= n; t++) {
            int v = base > run ? base : run;
            p.mnullT[(int64_t)(t - 1) * n + (s - 1)] = p.wy[t] + v;
            int g = p.wx[t - 1] + (t <= L ? p.wx[t] : 0) + p.of[t];
            run = g > run ? g : run;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) *p.res_status = bad ? ROTOR_EINPUT : ROTOR_OK;
}

// Eq. (1): C[s,s,m] = uf[s]+ub[s] if m >= m_all(s,s) else +inf.
__device__ __forceinline__ void leaf_cell(const Problem &p, int s, int m) {
    const int ma = m_all(p, s, s);
    const int64_t off = cell_index(p.n, s, s) * p.pitch + m;
    const double c = (m >= ma) ? p.w[s] : INFINITY;
    if (p.D) p.D[off] = (m >= ma) ? 0 : kNone;
    if (p.A) {
        store_final_c(p, s, s, m, p.wx[s - 1], c);
        if (s < p.n) store_final_a(p, s, s, m, __dadd_rn(__dadd_rn(p.P[s], -p.P[s - 1]), c));
    } else {
        p.C[off] = c;
    }
}

// Eq. (2) for one cell (s, t = s+d, m), candidates in Algorithm 2's order:
//   C_1 = min_{k=1..d} fl(fl(U(s,s+k) + C[s,s+k-1,m]) + C[s+k,t,m-wx[s+k-1]])  if m >= m_null(s,t)
//   C_2 = fl(w[s] + C[s+1,t,m-wbx[s]])                                         if m >= m_all(s,t)
//   C = min(C_1, C_2); D: smallest k under strict <, F_all only if strictly smaller (Q11).
__device__ __forceinline__ void wavefront_cell(const Problem &p, int s, int t, int m) {
    const int n = p.n;
    const int64_t pitch = p.pitch;
    double best = INFINITY;
    int arg = kNone;
    if (m >= m_null(p, s, t)) {
        const double Ps = p.P[s - 1];
        // s-major rows: (s, s+k-1) = rs + k - 1; (s+k, t) = R(s+k) + (t-s-k), and
        // R(s+k+1) + (t-s-k-1) - (R(s+k) + (t-s-k)) = n - s - k.
        const double *pre = p.C + cell_index(n, s, s) * pitch + m;
        int64_t suf_row = cell_index(n, s + 1, t);
        for (int k = 1; k <= t - s; k++) {
            const int sp = s + k;
            const double U = __dadd_rn(p.P[sp - 1], -Ps);
            const int mm = m - p.wx[sp - 1];
            const double suf = (mm >= 0) ? p.C[suf_row * pitch + mm] : INFINITY;
            const double v = __dadd_rn(__dadd_rn(U, *pre), suf);
            if (v < best) {
                best = v;
                arg = k;
            }
            pre += pitch;
            suf_row += n - s - k;
        }
    }
    if (!p.restricted && m >= m_all(p, s, t)) {
        const int mm = m - p.wbx[s];
        const double sub = (mm >= 0) ? p.C[cell_index(n, s + 1, t) * pitch + mm] : INFINITY;
        const double v = __dadd_rn(p.w[s], sub);
        if (v < best) {
            best = v;
            arg = 0;
        }
    }
    const int64_t off = cell_index(n, s, t) * pitch + m;
    p.C[off] = best;
    if (p.D) p.D[off] = isinf(best) ? kNone : (uint16_t)arg;
}

// Algorithm 2's decision at a finished cell: smallest k = s'-s with
// C[s,t,m] == C_ck(s,s',t,m) (C_1 exists only where m >= m_null),
// 0 for F_all / leaf, kNone if C = +inf.
__device__ __forceinline__ uint16_t decision_cell(const Problem &p, int s, int t, int m) {
    const int n = p.n;
    const int64_t pitch = p.pitch;
    const double c = p.C[cell_index(n, s, t) * pitch + m];
    if (isinf(c)) return kNone;
    if (s == t || m < m_null(p, s, t)) return 0;
    const double Ps = p.P[s - 1];
    for (int k = 1; k <= t - s; k++) {
        const int sp = s + k;
        const double U = __dadd_rn(p.P[sp - 1], -Ps);
        const double pre = p.C[cell_index(n, s, sp - 1) * pitch + m];
        const int mm = m - p.wx[sp - 1];
        const double suf = (mm >= 0) ? p.C[cell_index(n, sp, t) * pitch + mm] : INFINITY;
        if (__dadd_rn(__dadd_rn(U, pre), suf) == c) return (uint16_t)k;
    }
    return 0;
}

// Algorithm 2 (OptRec) as an explicit-stack DFS run by one CTA.
// At node (s,t,m): leaf -> (F_all^s, B^s); else the smallest s' with
// C[s,t,m] = C_ck(s,s',t,m) gives (F_ck^s, F_null^{s+1..s'-1} (Q4),
// OptRec(s',t,m-wx[s'-1]), OptRec(s,s'-1,m)); otherwise (F_all^s,
// OptRec(s+1,t,m-wbx[s]), B^s).  The candidate scan over s' is spread over the
// CTA (min-index reduction); a D table recorded during the fill is used
// instead when present (same decision by construction).  Results go to
// p.res_cost / p.res_nops / p.res_status / p.ops.
enum : int { kTaskNode = 0, kTaskEmitB = 1 };

__device__ __forceinline__ void reconstruct_cta(const Problem &p) {
    __shared__ int4 cur;
    __shared__ int top;
    __shared__ int kbest;
    __shared__ long long cnt;
    __shared__ int err;
    const int n = p.n;
    const int64_t pitch = p.pitch;
    __syncthreads();
    if (threadIdx.x == 0) {
        cnt = 0;
        err = 0;
        top = 0;
        int st = *p.res_status;
        const int m_top = p.S - p.wx[0];  // Alg. 1 return OptRec(C, 1, L+1, M - wx[0]) (Q5)
        double c = (m_top >= 0) ? p.C[cell_index(n, 1, n) * pitch + m_top] : INFINITY;
        *p.res_cost = c;
        if (st != ROTOR_OK) {
            err = st;
        } else if (isinf(c)) {
            err = ROTOR_INFEASIBLE;
        } else {
            p.stack[top++] = make_int4(kTaskNode, 1, n, m_top);
        }
    }
    __syncthreads();
    while (true) {
        if (threadIdx.x == 0) {
            if (top > 0 && err == 0) {
                cur = p.stack[--top];
            } else {
                cur = make_int4(-1, 0, 0, 0);
            }
            kbest = 0x7fffffff;
        }
        __syncthreads();
        const int4 task = cur;
        if (task.x < 0) break;
        const int s = task.y, t = task.z, m = task.w;
        if (task.x == kTaskEmitB) {
            if (threadIdx.x == 0) {
                if (cnt < p.ops_cap) p.ops[cnt] = rotor_op{ROTOR_BWD, s};
                cnt++;
            }
            __syncthreads();
            continue;
        }
        const double c = p.C[cell_index(n, s, t) * pitch + m];
        if (s == t) {
            if (threadIdx.x == 0) {
                if (isinf(c)) err = ROTOR_EINVALID;
                if (cnt < p.ops_cap) p.ops[cnt] = rotor_op{ROTOR_FALL, s};
                if (cnt + 1 < p.ops_cap) p.ops[cnt + 1] = rotor_op{ROTOR_BWD, s};
                cnt += 2;
            }
            __syncthreads();
            continue;
        }
        const int d = t - s;
        if (p.D) {
            if (threadIdx.x == 0) {
                uint16_t code = p.D[cell_index(n, s, t) * pitch + m];
                kbest = (code == kNone) ? -1 : (code == 0 ? 0x7fffffff : code);
            }
        } else if (m >= m_null(p, s, t)) {
            const double Ps = p.P[s - 1];
            for (int k = 1 + threadIdx.x; k <= d; k += blockDim.x) {
                const int sp = s + k;
                const double U = __dadd_rn(p.P[sp - 1], -Ps);
                const double pre = p.C[cell_index(n, s, sp - 1) * pitch + m];
                const int mm = m - p.wx[sp - 1];
                const double suf = (mm >= 0) ? p.C[cell_index(n, sp, t) * pitch + mm] : INFINITY;
                const double v = __dadd_rn(__dadd_rn(U, pre), suf);
                if (v == c) atomicMin(&kbest, k);
            }
        }
        __syncthreads();
        const int k = kbest;
        if (k < 0 || isinf(c)) {
            if (threadIdx.x == 0) err = ROTOR_EINVALID;
            __syncthreads();
            break;
        }
        if (k != 0x7fffffff) {
            // F_ck^s, F_null^{s+1..s'-1}, then OptRec(s', t, m - wx[s'-1]), OptRec(s, s'-1, m)
            const int sp = s + k;
            for (int i = threadIdx.x; i < k; i += blockDim.x) {
                long long pos = cnt + i;
                if (pos < p.ops_cap) p.ops[pos] = rotor_op{i == 0 ? ROTOR_FCK : ROTOR_FNULL, s + i};
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                cnt += k;
                if (top + 2 > p.stack_cap) {
                    err = ROTOR_EINVALID;
                } else {
                    p.stack[top++] = make_int4(kTaskNode, s, sp - 1, m);
                    p.stack[top++] = make_int4(kTaskNode, sp, t, m - p.wx[sp - 1]);
                }
            }
        } else {
            if (threadIdx.x == 0) {
                if (p.restricted) {
                    err = ROTOR_EINVALID;
                } else if (top + 2 > p.stack_cap) {
                    err = ROTOR_EINVALID;
                } else {
                    if (cnt < p.ops_cap) p.ops[cnt] = rotor_op{ROTOR_FALL, s};
                    cnt++;
                    p.stack[top++] = make_int4(kTaskEmitB, s, 0, 0);
                    p.stack[top++] = make_int4(kTaskNode, s + 1, t, m - p.wbx[s]);
                }
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (err == 0) {
            *p.res_nops = cnt;
            *p.res_status = cnt > p.ops_cap ? ROTOR_ETRUNC : ROTOR_OK;
        } else {
            *p.res_nops = -1;
            *p.res_status = err;
            if (err == ROTOR_INFEASIBLE) *p.res_cost = INFINITY;
        }
    }
    __syncthreads();
}

}  // namespace rotor
