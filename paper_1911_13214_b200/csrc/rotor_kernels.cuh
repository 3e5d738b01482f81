#pragma once
#include "rotor_common.cuh"

namespace rotor {

void launch_precompute(const rotor_chain &dch, uint64_t M, const Problem &p, cudaStream_t st);
void launch_leaf(const Problem &p, cudaStream_t st);
void launch_diag_wavefront(const Problem &p, int d, cudaStream_t st);
void launch_reconstruct(const Problem &p, cudaStream_t st);
void launch_derive_argmin(const Problem &p, int d, uint16_t *Dout, int64_t dpitch, cudaStream_t st);

// Fused batched solver (rotor_batch.cu).
struct BatchArgs {
    int n_problems, S, restricted, L_max;
    const int32_t *prob_chain;  // [n_problems] chain index of each problem
    const uint64_t *limits;     // [n_problems] memory limit M (bytes)
    const int32_t *chain_L;     // [n_chains]
    int64_t chain_stride;       // entries between consecutive chains in the arrays below (>= L_max + 2)
    const double *uf, *ub;
    const uint64_t *wx, *wbx, *wy, *of, *ob;
    char *pool;                 // gridDim.x slots of batch_slot_bytes(L_max, S)
    double *cost;
    int64_t *nops;
    int32_t *status;
    rotor_op *ops;              // nullable
    const int64_t *ops_off, *ops_cap;
    int *counter;               // work queue head, zeroed before the launch
};
size_t batch_slot_bytes(int L_max, int S);
void launch_batch(const BatchArgs &b, int n_slots, cudaStream_t st);

// Tiled fill (rotor_tiled.cu). Returns the number of kernels launched.
int launch_fill_tiled(const Problem &p, cudaStream_t st);
size_t tiled_extra_bytes(int L, int S);

}  // namespace rotor
