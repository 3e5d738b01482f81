// Tiled fill — placeholder until the blocked kernel lands: runs the wavefront.
#include "rotor_common.cuh"
#include "rotor_kernels.cuh"

namespace rotor {

size_t tiled_extra_bytes(int, int) { return 0; }

int launch_fill_tiled(const Problem &p, cudaStream_t st) {
    for (int d = 1; d <= p.L; d++) launch_diag_wavefront(p, d, st);
    return p.L;
}

}  // namespace rotor
