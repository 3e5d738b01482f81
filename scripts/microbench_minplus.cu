// Microbenchmark: sustained min-plus transition rate of the B200 SM for the
// inner loop shape of the tiled fill (register tile RS x RT, operands from
// shared memory, m along lanes).  Three min variants:
//   0: v < acc ? v : acc on doubles       (DADD + DSETP + 2 FSEL)
//   1: 64-bit integer min on the bit patterns of non-negative doubles
//   2: DADD only (upper bound of the fp64 pipe)
//   5: the pruned middle kernel's filter on fp32 operands in shared memory
//      (FADD.RM + FSETP.LT.OR per candidate, 8 x 8 register tile, one m per
//      lane, per-split fire mask OR-reduced over the warp) — its issue ceiling
//   4: fp32 lower-bound filter (cvt.rm.f32.f64 of the operands, FADD.RM, FMNMX;
//      per 8 splits one exact compare of the chunk minimum against the fp64
//      accumulator) — the pruned middle kernel's steady state with no exact pass
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb microbench_minplus.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE, int RS, int RT>
__global__ void __launch_bounds__(256) kern(double *out, int iters) {
    __shared__ double As[8][RS][32];
    __shared__ double Bs[8][RT][32];
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 8 * RS * 32; i += blockDim.x) (&As[0][0][0])[i] = 1.0 + (i % 7) * 0.125;
    for (int i = threadIdx.x; i < 8 * RT * 32; i += blockDim.x) (&Bs[0][0][0])[i] = 2.0 + (i % 5) * 0.25;
    __syncthreads();
    double acc[RS][RT];
#pragma unroll
    for (int i = 0; i < RS; i++)
#pragma unroll
        for (int j = 0; j < RT; j++) acc[i][j] = 1e300;
    if (MODE == 4) {
        for (int it = 0; it < iters; it++) {
            float mn[RS][RT];
#pragma unroll
            for (int k = 0; k < 8; k++) {
                float a[RS], b[RT];
#pragma unroll
                for (int i = 0; i < RS; i++) a[i] = __double2float_rd(As[(k + it) & 7][i][lane]);
#pragma unroll
                for (int j = 0; j < RT; j++) b[j] = __double2float_rd(Bs[(k + it) & 7][j][lane]);
#pragma unroll
                for (int i = 0; i < RS; i++)
#pragma unroll
                    for (int j = 0; j < RT; j++) {
                        const float v = __fadd_rd(a[i], b[j]);
                        mn[i][j] = k == 0 ? v : fminf(mn[i][j], v);
                    }
            }
            bool need = false;
#pragma unroll
            for (int i = 0; i < RS; i++)
#pragma unroll
                for (int j = 0; j < RT; j++) need |= (double)mn[i][j] < acc[i][j];
            if (__any_sync(0xffffffffu, need)) acc[it & 7 & (RS - 1)][0] = (double)mn[0][0];
        }
    } else
    for (int it = 0; it < iters; it++) {
#pragma unroll 4
        for (int k = 0; k < 8; k++) {
            double a[RS], b[RT];
#pragma unroll
            for (int i = 0; i < RS; i++) a[i] = As[k][i][lane];
#pragma unroll
            for (int j = 0; j < RT; j++) b[j] = Bs[k][j][lane];
#pragma unroll
            for (int i = 0; i < RS; i++)
#pragma unroll
                for (int j = 0; j < RT; j++) {
                    double v = __dadd_rn(a[i], b[j]);
                    if (MODE == 0 || (MODE == 3 && j < RT - 2)) {
                        acc[i][j] = v < acc[i][j] ? v : acc[i][j];
                    } else if (MODE == 1 || MODE == 3) {
                        long long x = __double_as_longlong(v), y = __double_as_longlong(acc[i][j]);
                        acc[i][j] = __longlong_as_double(x < y ? x : y);
                    } else {
                        acc[i][j] = __dadd_rn(acc[i][j], v) ;
                    }
                }
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < RS; i++)
#pragma unroll
        for (int j = 0; j < RT; j++) s += acc[i][j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// MODE 5 kernel: operands fp32 [8 splits][8 rows][32 m] in shared memory
__global__ void __launch_bounds__(512, 1) kern_filter(float *out, int iters) {
    __shared__ float As[8][8][32];
    __shared__ float Bs[8][8][32];
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 8 * 8 * 32; i += blockDim.x) {
        (&As[0][0][0])[i] = 1.0f + (i % 7) * 0.125f;
        (&Bs[0][0][0])[i] = 2.0f + (i % 5) * 0.25f;
    }
    __syncthreads();
    float bestf[8][8];
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 8; j++) bestf[i][j] = 0.5f + 0.01f * (i * 8 + j) + 0.001f * lane;
    unsigned acc = 0;
    for (int it = 0; it < iters; it++) {
        unsigned needk = 0;
#pragma unroll 1
        for (int k = 0; k < 8; k++) {
            const int kk = (k + it) & 7;
            float a[8], b[8];
#pragma unroll
            for (int i = 0; i < 8; i++) a[i] = As[kk][i][lane];
#pragma unroll
            for (int j = 0; j < 8; j++) b[j] = Bs[kk][j][lane];
            bool nk = false;
#pragma unroll
            for (int i = 0; i < 8; i++)
#pragma unroll
                for (int j = 0; j < 8; j++) nk |= __fadd_rd(a[i], b[j]) < bestf[i][j];
            needk |= (unsigned)nk << k;
        }
        acc += __reduce_or_sync(0xffffffffu, needk);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
}

void run_filter() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms, threads = 512, iters = 2000;
    float *out;
    cudaMalloc(&out, blocks * threads * sizeof(float));
    kern_filter<<<blocks, threads>>>(out, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern_filter<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double tr = (double)blocks * threads * iters * 8 * 64;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%-28s 8x8 tile  %.3e candidates/s  (%.1f cand/clk/SM at %d MHz)  err=%s\n", "middle filter (fp32 smem)",
           tr / (ms * 1e-3), tr / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000, cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

template <int MODE, int RS, int RT>
void run(const char *name) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 2, threads = 256, iters = 3200;
    double *out;
    cudaMalloc(&out, blocks * threads * sizeof(double));
    kern<MODE, RS, RT><<<blocks, threads>>>(out, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<MODE, RS, RT><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double tr = (double)blocks * threads * iters * 8 * RS * RT;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%-28s RS=%d RT=%d  %.3e transitions/s  (%.1f tr/clk/SM at %d MHz)  err=%s\n", name, RS, RT, tr / (ms * 1e-3),
           tr / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000, cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main() {
    run_filter();
    run<0, 4, 4>("dsetp-min");
    run<0, 4, 8>("dsetp-min");
    run<0, 8, 8>("dsetp-min");
    run<3, 8, 8>("mixed (2 of 8 cols int64)");
    run<3, 4, 8>("mixed (2 of 8 cols int64)");
    run<1, 4, 8>("int64-min");
    run<1, 8, 8>("int64-min");
    run<2, 4, 8>("dadd-only");
    run<2, 8, 8>("dadd-only");
    run<4, 8, 4>("fp32 filter");
    run<4, 4, 8>("fp32 filter");
    return 0;
}
