// Development probe: legacy mma.sync throughput on this GPU (TF32 m16n8k8,
// BF16 m16n8k16) -- decides whether a 3xTF32 accumulation can pay for K1.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_tf32(float* out, int iters) {
    unsigned a[4] = {threadIdx.x, 1u, 2u, 3u}, b[2] = {5u, 7u};
    float d[8][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
                         : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    float s = 0;
    for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
    if (s == 1.2345f) out[0] = s;
}
__global__ void k_bf16(float* out, int iters) {
    unsigned a[4] = {threadIdx.x, 1u, 2u, 3u}, b[2] = {5u, 7u};
    float d[8][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
                         : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    float s = 0;
    for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
    if (s == 1.2345f) out[0] = s;
}
int main() {
    float* o;
    cudaMalloc(&o, 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int which = 0; which < 2; ++which) {
        for (int warps = 4; warps <= 16; warps *= 2) {
            const int iters = 4096;
            auto run = [&] {
                if (which == 0) k_tf32<<<sms * 4, 32 * warps>>>(o, iters);
                else k_bf16<<<sms * 4, 32 * warps>>>(o, iters);
            };
            run();
            cudaEventRecord(e0);
            run();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double mmas = (double)sms * 4 * warps * iters * 8;
            const double flop = mmas * 2.0 * 16 * 8 * (which == 0 ? 8 : 16);
            printf("%s warps/CTA %2d: %.1f TFLOP/s (%.3f ms)\n", which == 0 ? "tf32 m16n8k8 " : "bf16 m16n8k16", warps,
                   flop / ms / 1e9, ms);
        }
    }
    return 0;
}
