// pd_peaks.cu -- roofline denominators measured on the box itself ("FP32 and L2 peaks are
// not in MEASURED_PEAKS.json; measure both on the box in the same job: an FFMA-chain kernel and an
// L2-resident read kernel").  Not on the hot path: bench.py calls them once, next to the timed steps.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pd.h"

namespace pd {
namespace {

constexpr int kChains = 8;     // independent FFMA chains per thread (covers the 4-cycle FMA latency x 2)
constexpr int kIters = 4096;   // unrolled by 16 below

// Every thread runs kChains independent a = a * b + c chains; one FFMA = one FP32 lane-op (the unit of
// SURVEY.md §8(d)'s W_min and of the 148 SM x 128 lane x f_clk nominal peak).
__global__ void __launch_bounds__(256) k_ffma(float* out, float b, float c) {
    float a[kChains];
#pragma unroll
    for (int k = 0; k < kChains; ++k) a[k] = threadIdx.x * 1e-3f + k;
#pragma unroll 16
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int k = 0; k < kChains; ++k) a[k] = fmaf(a[k], b, c);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < kChains; ++k) s += a[k];
    if (s == 12345.678f) out[0] = s;  // keeps the chains live; never true for the inputs used
}

// L2-resident read: `passes` sweeps over a buffer well inside the 126 MB L2, 16-byte loads that bypass L1
// (ld.global.cg), so every byte is an L2 hit after the first sweep.
__global__ void __launch_bounds__(512) k_l2read(const float4* __restrict__ buf, int64_t n4, int passes, float* out) {
    float acc = 0.f;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int p = 0; p < passes; ++p)
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
            const float4 v = __ldcg(&buf[i]);
            acc += v.x + v.y + v.z + v.w;
        }
    if (acc == 12345.678f) out[0] = acc;
}

}  // namespace
}  // namespace pd

extern "C" {

// Measured FP32 FFMA throughput of `device` in lane-ops/s (best of `reps` launches, CUDA events), and
// the SM clock it ran at is up to the caller (nvidia-smi).  Errors: PD_EINVAL, PD_ECUDA.
pd_status pd_measure_fp32_peak(int device, int reps, double* lane_ops_per_s) {
    if (!lane_ops_per_s || reps < 1) return PD_EINVAL;
    if (cudaSetDevice(device) != cudaSuccess) return PD_ECUDA;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    float* out = nullptr;
    if (cudaMalloc(&out, 16) != cudaSuccess) return PD_ECUDA;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 8;  // 8 x 256 threads = 64 warps per SM (full occupancy)
    double best = 0.0;
    for (int r = 0; r < reps + 1; ++r) {
        cudaEventRecord(e0);
        pd::k_ffma<<<blocks, 256>>>(out, 0.999999f, 1e-7f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = (double)blocks * 256 * pd::kIters * pd::kChains;
        if (r > 0 && ms > 0.f) best = ops / (ms * 1e-3) > best ? ops / (ms * 1e-3) : best;
    }
    cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (err != cudaSuccess) return PD_ECUDA;
    *lane_ops_per_s = best;
    return PD_OK;
}

// Measured L2 read bandwidth of `device` in bytes/s: a `bytes`-sized buffer (<= 64 MB recommended: the
// L2 is 126 MB in two partitions) swept 32 times per launch after a warming launch; best of `reps`.
pd_status pd_measure_l2_peak(int device, int64_t bytes, int reps, double* bytes_per_s) {
    if (!bytes_per_s || reps < 1 || bytes < (1 << 20)) return PD_EINVAL;
    if (cudaSetDevice(device) != cudaSuccess) return PD_ECUDA;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int64_t n4 = bytes / 16;
    float4* buf = nullptr;
    float* out = nullptr;
    if (cudaMalloc(&buf, n4 * 16) != cudaSuccess) return PD_ECUDA;
    if (cudaMalloc(&out, 16) != cudaSuccess) {
        cudaFree(buf);
        return PD_ECUDA;
    }
    cudaMemset(buf, 0, n4 * 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int passes = 32, blocks = sms * 4;
    double best = 0.0;
    for (int r = 0; r < reps + 1; ++r) {
        cudaEventRecord(e0);
        pd::k_l2read<<<blocks, 512>>>(buf, n4, passes, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double b = (double)n4 * 16 * passes;
        if (r > 0 && ms > 0.f) best = b / (ms * 1e-3) > best ? b / (ms * 1e-3) : best;
    }
    cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(buf);
    cudaFree(out);
    if (err != cudaSuccess) return PD_ECUDA;
    *bytes_per_s = best;
    return PD_OK;
}

}  // extern "C"
