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
    const int32_t *order;       // [n_problems] hand-out order of the queue (longest chains first)
    int mc;                     // m-chunk of the fill order (0: whole rows, diagonal by diagonal)
    int prune;                  // 1/2/4: warp-group cells with the monotone-in-m candidate bound per 32/prune m (batch_cell_group); 0: wavefront_cell
};
size_t batch_slot_bytes(int L_max, int S);
int batch_ctas_per_sm();  // k_batch's __launch_bounds__ residency: persistent CTAs per SM
void launch_batch(const BatchArgs &b, int n_slots, cudaStream_t st);
void launch_compact_ops(const rotor_op *src, const int64_t *src_off, const int64_t *cnt, const int64_t *dst_off,
                        rotor_op *dst, int P, cudaStream_t st);

// Tiled fill (rotor_fill_tiled.cu). Returns the number of kernels launched (-1: setup error).
// mid_ev (optional, 2 * mid_cap events): recorded around each middle-kernel launch
// schedule: 0 = the tile DAG over several streams (default), 1 = diagonal by diagonal on st
int launch_fill_tiled(const Problem &p, cudaStream_t st, int schedule, cudaEvent_t *mid_ev = nullptr, int mid_cap = 0,
                      int *mid_n = nullptr);
size_t tiled_extra_bytes(int L, int S);
size_t tiled_list_offset(int L, int S);  // of the middle's fired-split lists within the extra bytes

// Pieces of the tiled fill for a sharded (multi-rank) solve.
struct TiledCtx {
    alignas(64) unsigned char tmA[128];  // CUtensorMap of the A table
    alignas(64) unsigned char tmC[128];  // CUtensorMap of the C table
    int phase_id;                        // leaf launches so far (look-back flag epochs)
    cudaEvent_t *mid_ev;                 // optional (profiling): event pairs around the middle launches
    int mid_cap, mid_n;                  // pairs available / recorded
    int sms;                             // SM count of the device (set by tiled_prepare)
};
int tiled_nb(int n);  // number of TB-stage blocks
// candidates of the middle ranges per m (cells s in block I, t in block J,
// splits s' in blocks I+1..J-1, J - I >= 2; existing cells only)
int64_t tiled_middle_candidates(int n);
int tiled_prepare(const Problem &p, TiledCtx *ctx, cudaStream_t st);
int tiled_delta(const Problem &p, TiledCtx *ctx, int delta, int tile_lo, int tile_hi, cudaStream_t st);
size_t tiled_tile_bytes(int S);
int tiled_pack(const Problem &p, int delta, int tile_lo, int tile_hi, double *buf, int unpack, cudaStream_t st);
// copy the tiles' C rows from another table of the same layout (e.g. a peer
// device's, through peer memory) and rebuild A and the shadows (the P2P halo)
int tiled_pull(const Problem &p, const double *src_C, int delta, int tile_lo, int tile_hi, cudaStream_t st);

}  // namespace rotor
