// Fused batched solver: many independent (chain, limit)
// tables — the paper's multi-limit sweep, "Algorithm 1 for 10 different memory
// limits" — in ONE launch.  A persistent CTA takes problems from an
// atomic queue (handed out longest chain first, so the tail is short) and runs
// the whole path for each inside its own workspace slot:
// precompute (discretisation with that limit's slot size M/S),
// leaf, every diagonal d (barrier between diagonals), Algorithm-2 walk.  The
// per-cell arithmetic is the wavefront kernel's (rotor_device.cuh), so every
// table is bit-identical to a single solve.
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

__global__ void __launch_bounds__(512, 4) k_batch(BatchArgs b) {  // 4 resident per SM (rotor_abi.cu)
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
            for (int d = 1; d <= L; d++) {
                for (int idx = threadIdx.x; idx < (n - d) * wm; idx += blockDim.x) {
                    const int s = 1 + idx / wm;
                    wavefront_cell(p, s, s + d, m0 + idx % wm);
                }
                __syncthreads();
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
