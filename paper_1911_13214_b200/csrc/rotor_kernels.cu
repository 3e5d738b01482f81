// Per-table kernels: precompute (K0), leaf diagonal (K1), wavefront diagonal
// (K2, the reference fill kernel), Algorithm-2 walker (K3) and the argmin
// export.  The arithmetic lives in rotor_device.cuh (shared with the batched
// kernel) — see its header for the paper passages and readings.
#include "rotor_device.cuh"
#include "rotor_kernels.cuh"

namespace rotor {

__global__ void k_precompute(rotor_chain ch, uint64_t M, Problem p) { precompute_cta(ch, M, p); }

__global__ void k_leaf(Problem p) {
    const int s = blockIdx.y + 1;
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m <= p.S) leaf_cell(p, s, m);
}

// One launch per diagonal d >= 1, one thread per (s, m) cell; loads of
// C[·,·,m] are coalesced along m (consecutive threads).
__global__ void k_diag_wavefront(Problem p, int d) {
    const int s = blockIdx.y + 1;
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m <= p.S) wavefront_cell(p, s, s + d, m);
}

__global__ void k_reconstruct(Problem p) { reconstruct_cta(p); }

__global__ void k_derive_argmin(Problem p, int d, uint16_t *Dout, int64_t dpitch) {
    const int s = blockIdx.y + 1;
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m <= p.S) Dout[cell_index(p.n, s, s + d) * dpitch + m] = decision_cell(p, s, s + d, m);
}

// ---------------------------------------------------------------------------
// host-side launchers
// ---------------------------------------------------------------------------
void launch_precompute(const rotor_chain &dch, uint64_t M, const Problem &p, cudaStream_t st) {
    k_precompute<<<1, 1024, 0, st>>>(dch, M, p);
}

void launch_leaf(const Problem &p, cudaStream_t st) {
    dim3 block(256);
    dim3 grid((p.S + 1 + block.x - 1) / block.x, p.n);
    k_leaf<<<grid, block, 0, st>>>(p);
}

void launch_diag_wavefront(const Problem &p, int d, cudaStream_t st) {
    dim3 block(128);
    dim3 grid((p.S + 1 + block.x - 1) / block.x, p.n - d);
    k_diag_wavefront<<<grid, block, 0, st>>>(p, d);
}

void launch_reconstruct(const Problem &p, cudaStream_t st) { k_reconstruct<<<1, 1024, 0, st>>>(p); }

void launch_derive_argmin(const Problem &p, int d, uint16_t *Dout, int64_t dpitch, cudaStream_t st) {
    dim3 block(128);
    dim3 grid((p.S + 1 + block.x - 1) / block.x, p.n - d);
    k_derive_argmin<<<grid, block, 0, st>>>(p, d, Dout, dpitch);
}

}  // namespace rotor
