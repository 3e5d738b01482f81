#pragma once
#include "rotor_common.cuh"

namespace rotor {

void launch_precompute(const rotor_chain &dch, uint64_t M, const Problem &p, cudaStream_t st);
void launch_leaf(const Problem &p, cudaStream_t st);
void launch_diag_wavefront(const Problem &p, int d, cudaStream_t st);
void launch_reconstruct(const Problem &p, cudaStream_t st);
void launch_derive_argmin(const Problem &p, int d, uint16_t *Dout, int64_t dpitch, cudaStream_t st);

// Tiled fill (rotor_tiled.cu). Returns the number of kernels launched.
int launch_fill_tiled(const Problem &p, cudaStream_t st);
size_t tiled_extra_bytes(int L, int S);

}  // namespace rotor
