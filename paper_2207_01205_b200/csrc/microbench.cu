// microbench.cu — measured roofline denominators for the FOFSE kernels.
//
// MEASURED_PEAKS.json (driver-written) carries HBM copy bandwidth and the bf16
// GEMM rate only; K2 is bound by shared-memory bandwidth and the FP32/FP64
// pipes, so bench.py measures those peaks on the same box:
//   kind 0: shared-memory load bandwidth, LDS.64, conflict-free   [GB/s]
//   kind 1: shared-memory load bandwidth, LDS.32, conflict-free   [GB/s]
//   kind 2: FP32 FFMA throughput (register operands)              [TFLOP/s]
//   kind 3: FP64 DFMA throughput                                   [TFLOP/s]
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "../../include/fofse.h"

namespace {

constexpr int MB_THREADS = 512;
constexpr int MB_ITERS = 4096;

template <class V>
__global__ void __launch_bounds__(MB_THREADS) smem_bw(float* out, int iters) {
    __shared__ V buf[MB_THREADS * 4];
    for (int i = threadIdx.x; i < MB_THREADS * 4; i += blockDim.x) {
        if constexpr (sizeof(V) == 8)
            buf[i] = V{(float)i, (float)(i + 1)};
        else
            buf[i] = (float)i;
    }
    __syncthreads();
    float acc = 0.f;
    const int t = threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const V v = buf[(t + k * MB_THREADS + it) & (MB_THREADS * 4 - 1)];
            if constexpr (sizeof(V) == 8)
                acc += v.x + v.y;
            else
                acc += v;
        }
    }
    if (acc == -1.f) out[0] = acc;
}

__global__ void __launch_bounds__(MB_THREADS) ffma_rate(float* out, int iters) {
    float a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-7f + k;
    const float b = 0.9999f, c = 1e-6f;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], b, c);
    float s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == -1.f) out[0] = s;
}

__global__ void __launch_bounds__(MB_THREADS) dfma_rate(float* out, int iters) {
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-7 + k;
    const double b = 0.9999, c = 1e-6;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == -1.0) out[0] = (float)s;
}

}  // namespace

extern "C" int fofse_microbench(int32_t device, int32_t kind, double* value) {
    if (!value) return FOFSE_EINVAL;
    if (cudaSetDevice(device) != cudaSuccess) return FOFSE_ECUDA;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    float* out = nullptr;
    if (cudaMalloc(&out, 16) != cudaSuccess) return FOFSE_ECUDA;
    const int grid = sms * 4;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto launch = [&](int iters) {
        switch (kind) {
            case 0: smem_bw<float2><<<grid, MB_THREADS>>>(out, iters); break;
            case 1: smem_bw<float><<<grid, MB_THREADS>>>(out, iters); break;
            case 2: ffma_rate<<<grid, MB_THREADS>>>(out, iters); break;
            default: dfma_rate<<<grid, MB_THREADS>>>(out, iters); break;
        }
    };
    const int iters = kind >= 2 ? (kind == 3 ? MB_ITERS / 8 : MB_ITERS) : MB_ITERS;
    launch(iters / 8);  // warm-up
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        launch(iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (err != cudaSuccess) return FOFSE_ECUDA;
    const double threads = static_cast<double>(grid) * MB_THREADS;
    double work;
    switch (kind) {
        case 0: work = threads * iters * 4 * 8.0; break;   // bytes
        case 1: work = threads * iters * 4 * 4.0; break;   // bytes
        default: work = threads * iters * 64 * 2.0; break; // flops
    }
    *value = kind < 2 ? work / (best * 1e-3) / 1e9 : work / (best * 1e-3) / 1e12;
    return FOFSE_OK;
}
