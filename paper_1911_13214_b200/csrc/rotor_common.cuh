// Shared device-side definitions of the B200 solver (product path only; the
// oracle in oracle/ never includes this file).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "rotor.h"

namespace rotor {

constexpr uint16_t kNone = 0xFFFF;  // D code of an infeasible cell
// Table rows carry kPad columns left of m = 0 and the tables kPadRows spare
// rows at the end, so every TMA box of the tiled fill (m0 - shift >= -kPad,
// row + box height <= rows + kPadRows) lies inside the allocation.  The pads
// only ever feed candidates of cells the m_null gate discards (DESIGN Q6).
constexpr int kPad = 16;
constexpr int kPadRows = 32;
constexpr int kStatusOk = ROTOR_OK;

// Device view of one DP problem inside a workspace.
//
// Indices follow the paper (1-based stages, n = L+1):
//   wx[l] l=0..L, wy[l] l=0..n, wbx/of/ob[l] l=1..n   (int32 slots, clamped to S+1)
//   P[k] = uf[1] + ... + uf[k] (sequential fp64), k = 0..n
//   w[s] = uf[s] + ub[s]
//   mnullT[(t-1)*n + (s-1)] = m_null(s,t), s < t
// Table C: cell(s,t) = (s-1)*n - (s-1)*(s-2)/2 + (t-s) (s-major, the canonical
// layout of include/rotor.h); row of a cell = pitch doubles, m = 0..S.
struct Problem {
    int L, n, S;
    int restricted;
    int64_t pitch;  // doubles per cell row
    int32_t *wx, *wbx, *wy, *of, *ob;
    double *P, *w;
    int32_t *mnullT;
    double *C;
    uint16_t *D;  // nullable
    double *A;    // nullable: A(s,c,m) = fl(fl(P[c]-P[s-1]) + C(s,c,m)), row a_index(s,c) (tiled fill)
    int *flags;   // nullable: tiled fill's leaf look-back flags (tiled_extra_bytes)
    uint16_t *mlist;  // nullable: the pruned middle's fired-split lists (tiled_extra_bytes)
    // nullable (tiled fill): fp32 round-down shadows of C and A, read by the
    // pruned middle kernel's lower-bound filter, in the block-major layout of
    // srow_a / srow_c (m-chunked by shadow_index over sarows / scrows rows),
    // each (tile block, table column / row) followed by its 8 quad minima.
    // C32 is stored PRE-SHIFTED by the shift of the cell's first stage:
    // C32(s,t,m) = rd(C(s, t, m - wx[s-1])), +inf for m < wx[s-1] (the split
    // operand C(s', t, m - wx[s'-1]) depends on s' only).
    float *C32, *A32;
    int64_t sarows, scrows;
    // nullable: profile counters of the pruned middle (rotor_counters order)
    unsigned long long *counters;
    // reconstruction / results
    int4 *stack;
    int32_t stack_cap;
    double *res_cost;
    int64_t *res_nops;
    int32_t *res_status;
    rotor_op *ops;
    int64_t ops_cap;
};

__host__ __device__ inline int64_t cell_index(int n, int s, int t) {
    int64_t r = s - 1;  // s-major: cells (s, s..n) are contiguous rows
    return r * n - r * (r - 1) / 2 + (t - s);
}

// Row of A(s,c) in the A table: column-major over the upper triangle
// (c(c-1)/2 + s-1), so the cells (i0..i0+31, c) of one c — one TMA box of the
// tiled middle kernel — are consecutive rows.
__host__ __device__ inline int64_t a_index(int s, int c) { return (int64_t)c * (c - 1) / 2 + (s - 1); }

__device__ __forceinline__ int m_all(const Problem &p, int s, int t) {
    // m_all(s,t) = max(wy[t] + wbx[s] + of[s], wy[s] + wbx[s] + ob[s])
    int a = p.wy[t] + p.wbx[s] + p.of[s];
    int b = p.wy[s] + p.wbx[s] + p.ob[s];
    return a > b ? a : b;
}

__device__ __forceinline__ int m_null(const Problem &p, int s, int t) {
    return p.mnullT[(int64_t)(t - 1) * p.n + (s - 1)];
}

// fp32 shadow layout: the row is cut into chunks of kSW = 32 m; chunk q of all
// rows is contiguous, so the 32 m of consecutive rows are one contiguous block
// (one bulk copy, full DRAM bursts) instead of separate 128-byte row pieces.
constexpr int kSW = 32;
__host__ __device__ __forceinline__ int64_t shadow_index(int64_t srows, int64_t row, int m) {
    return ((int64_t)(m >> 5) * srows + row) * kSW + (m & (kSW - 1));
}

// Block-major shadow rows.  kTB = the tiled fill's tile edge; every (block,
// column) of A32 and (block, row) of C32 owns kSR = 40 consecutive rows: its 32
// cells, then 8 QUAD MINIMA — the min over 4 consecutive cells of the group
// (rows s of A32(., c); columns t of C32(s, .), one row s so one pre-shift),
// over existing cells only (+inf if none).  One split s' of a middle tile
// (I, J) reads A32 rows (I, c = s' - 1) and C32 rows (J, s'): the splits of
// one ring stage are consecutive columns / rows, so each operand set of a
// stage — KC x (32 cells + 8 minima) rows — is ONE contiguous block.
constexpr int kTB = 32;
constexpr int kSR = 40;
constexpr int kQuad = 32;  // row of group 0's minimum inside a (block, column / row)
// A32: [block I of s][column c = i0(I)..n][kSR]; A(s, c) exists for s <= c
__host__ __device__ __forceinline__ int64_t sa_col(int n, int I, int c) {
    return (int64_t)kSR * ((int64_t)I * n - (int64_t)kTB * I * (I - 1) / 2 + (c - (kTB * I + 1)));
}
__host__ __device__ __forceinline__ int64_t srow_a(int n, int s, int c) {
    const int I = (s - 1) / kTB;
    return sa_col(n, I, c) + (s - 1 - kTB * I);
}
// C32: [block J of t][row s = 1..min(n, 32 (J + 1))][kSR]
__host__ __device__ __forceinline__ int64_t sc_row(int J, int s) {
    return (int64_t)kSR * ((int64_t)kTB * J * (J + 1) / 2 + (s - 1));
}
__host__ __device__ __forceinline__ int64_t srow_c(int s, int t) {
    const int J = (t - 1) / kTB;
    return sc_row(J, s) + (t - 1 - kTB * J);
}
inline int64_t shadow_rows_a(int n) {
    const int64_t nb = (n + kTB - 1) / kTB;
    return (int64_t)kSR * (nb * n - (int64_t)kTB * nb * (nb - 1) / 2);
}
inline int64_t shadow_rows_c(int n) {
    const int nb = (n + kTB - 1) / kTB;
    return sc_row(nb - 1, n + 1);
}

// Store a finished cell's C and A with their fp32 round-down shadows
// (cvt.rm: a lower bound of the fp64 value, +inf stays +inf).  w = wx[s-1]
// of its first stage s (the pre-shift of C32): the thread of m writes shadow
// column m + w, and column m with +inf when m < w, so columns 0..S are all
// written once.  (The quad minima are written by the tiled fill's leaves.)
__device__ __forceinline__ void store_final_c(const Problem &p, int s, int t, int m, int w, double c) {
    p.C[cell_index(p.n, s, t) * p.pitch + m] = c;
    if (p.C32) {
        const int64_t r = srow_c(s, t);
        if (m + w <= p.S) p.C32[shadow_index(p.scrows, r, m + w)] = __double2float_rd(c);
        if (m < w) p.C32[shadow_index(p.scrows, r, m)] = INFINITY;
    }
}
__device__ __forceinline__ void store_final_a(const Problem &p, int s, int t, int m, double a) {
    p.A[a_index(s, t) * p.pitch + m] = a;
    if (p.A32) p.A32[shadow_index(p.sarows, srow_a(p.n, s, t), m)] = __double2float_rd(a);
}

}  // namespace rotor
