// k_selftest.cu -- on-device peak probes used as roofline denominators for
// the FP32/SFU-bound kernels (MEASURED_PEAKS.json only carries HBM and bf16
// tensor peaks). Each thread runs 8 independent FFMA (or MUFU.EX2) chains so
// the pipe, not latency, is the limit; grid = 8 CTAs x 256 threads per SM.
#include "nrm_common.cuh"
#include "nrm_internal.h"

namespace nrm {
namespace {

__global__ void __launch_bounds__(256) k_fp32_peak(float* out, int iters, float a, float b) {
    float x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3f + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = fmaf(x[k], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.678f) out[0] = s;  // keep the chains alive
}

__global__ void __launch_bounds__(256) k_mufu_peak(float* out, int iters) {
    float x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = -1e-3f * (threadIdx.x + k);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = ex2_approx(x[k]) - 1.0f;
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.678f) out[0] = s;
}

}  // namespace

cudaError_t run_peak_probe(int which, int num_sms, int iters, float* scratch, cudaStream_t st,
                           float* ms, int64_t* launches) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const dim3 grid(num_sms * 8), block(256);
    // warm-up
    if (which == 0) k_fp32_peak<<<grid, block, 0, st>>>(scratch, iters / 8 + 1, 0.999f, 1e-3f);
    else k_mufu_peak<<<grid, block, 0, st>>>(scratch, iters / 8 + 1);
    cudaEventRecord(e0, st);
    if (which == 0) k_fp32_peak<<<grid, block, 0, st>>>(scratch, iters, 0.999f, 1e-3f);
    else k_mufu_peak<<<grid, block, 0, st>>>(scratch, iters);
    cudaEventRecord(e1, st);
    *launches += 2;
    cudaError_t e = cudaEventSynchronize(e1);
    if (e == cudaSuccess) e = cudaEventElapsedTime(ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (e == cudaSuccess) e = cudaGetLastError();
    return e;
}

}  // namespace nrm
