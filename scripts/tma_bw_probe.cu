// Probe: DRAM throughput of TMA box loads with the middle kernel's access shape
// (32 rows x 16 fp64, rows `pitch` bytes apart) vs contiguous boxes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tbw scripts/tma_bw_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int STAGES = 8, BOX_COLS = 16, BOX_ROWS = 32;

__global__ void __launch_bounds__(32) kern(const __grid_constant__ CUtensorMap tm, long long rows, int cols,
                                           int iters, unsigned long long seed, double *sink) {
    extern __shared__ __align__(1024) double buf[];  // [STAGES][BOX_ROWS][BOX_COLS]
    __shared__ __align__(8) uint64_t bar[STAGES];
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; s++)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(1));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    unsigned long long x = seed + blockIdx.x * 0x9E3779B97F4A7C15ull;
    double acc = 0;
    auto issue = [&](int it) {
        const int s = it % STAGES;
        x = x * 6364136223846793005ull + 1442695040888963407ull;
        const long long r = (long long)((x >> 20) % (unsigned long long)(rows - BOX_ROWS));
        const int c = (int)((x >> 8) % (unsigned long long)(cols / BOX_COLS)) * BOX_COLS;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])),
                     "r"(BOX_ROWS * BOX_COLS * 8)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
            "%3}], [%4];" ::"r"(smem_u32(buf + s * BOX_ROWS * BOX_COLS)),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(c), "r"((int)r), "r"(smem_u32(&bar[s]))
            : "memory");
    };
    if (threadIdx.x == 0)
        for (int it = 0; it < STAGES; it++) issue(it);
    for (int it = 0; it < iters; it++) {
        const int s = it % STAGES;
        asm volatile(
            "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                smem_u32(&bar[s])),
            "r"((it / STAGES) & 1)
            : "memory");
        acc += buf[s * BOX_ROWS * BOX_COLS + threadIdx.x];
        __syncwarp();
        if (threadIdx.x == 0 && it + STAGES < iters) issue(it + STAGES);
    }
    if (acc == 12345.0) sink[0] = acc;
}

int main() {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    const size_t bytes = 16ull << 30;
    double *g, *sink;
    cudaMalloc(&g, bytes);
    cudaMalloc(&sink, 64);
    cudaMemset(g, 0, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t smem = STAGES * BOX_ROWS * BOX_COLS * 8;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    struct V { const char *name; long long pitch_doubles; } vs[] = {
        {"rows 32 KB apart (middle kernel)", 4032}, {"rows 4 KB apart", 512}, {"contiguous (pitch = box)", 16}};
    for (auto v : vs) {
        CUtensorMap tm;
        const long long rows = bytes / 8 / v.pitch_doubles;
        cuuint64_t dims[2] = {(cuuint64_t)v.pitch_doubles, (cuuint64_t)rows};
        cuuint64_t strides[1] = {(cuuint64_t)v.pitch_doubles * 8};
        cuuint32_t box[2] = {BOX_COLS, BOX_ROWS}, es[2] = {1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        for (int cps : {1, 4, 8}) {
            const int grid = sms * cps, iters = 4000;
            kern<<<grid, 32, smem>>>(tm, rows, (int)v.pitch_doubles, 100, 1, sink);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            kern<<<grid, 32, smem>>>(tm, rows, (int)v.pitch_doubles, iters, 7, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double gb = (double)grid * iters * BOX_ROWS * BOX_COLS * 8 / 1e9;
            printf("%-36s CTAs/SM=%d  %.0f GB/s  (%s)\n", v.name, cps, gb / (ms * 1e-3),
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
