// tcgen05 (5th-generation tensor core) TF32 probe for the node-field
// contraction shape: D[64 cols][192] = sum_k A[col][k] B[n][k],
// A = ex (M = 64 tile columns), B = ey * q_j (N = 6 components x 32 rows),
// 3xTF32 split products (Al Bh + Ah Bl + Ah Bh), FP32 accumulation in TMEM.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tcgen05_probe tcgen05_probe.cu
//   ./tcgen05_probe            # correctness (vs FP64 host) + fragment map + throughput
//
// Operands live in shared memory in the canonical K-major, no-swizzle
// ("interleave") UMMA layout: 8-row x 16-byte core matrices, rows 16 B apart,
// the two 16-byte K halves of one MMA (K = 8 TF32) LBO apart, 8-row groups
// SBO = 128 B apart, consecutive K steps 2 * rows * 16 B apart.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                    \
    do {                                                                                         \
        cudaError_t e_ = (x);                                                                    \
        if (e_ != cudaSuccess) {                                                                 \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);      \
            exit(1);                                                                             \
        }                                                                                        \
    } while (0)

constexpr int M = 64, N = 192, K = 32, THREADS = 128;

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// byte offset of element (r, k) of an R-row K-major operand
__host__ __device__ constexpr int kmaj_off(int r, int k, int R) {
    return (k / 8) * (2 * R * 16) + ((k % 8) / 4) * (R * 16) + (r / 8) * 128 + (r % 8) * 16 + (k % 4) * 4;
}

__device__ __forceinline__ uint64_t umma_desc(unsigned saddr, unsigned lbo, unsigned sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version (sm_100)
    return d;                // base offset 0, layout type 0 (no swizzle)
}

constexpr uint32_t kIdesc = (1u << 4)               // D: F32
                            | (2u << 7) | (2u << 10)  // A, B: TF32
                            | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);

__device__ __forceinline__ void mma_tf32_ss(unsigned tmem_d, uint64_t da, uint64_t db, unsigned accum) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(kIdesc), "r"(accum));
}

__device__ __forceinline__ float tf32_hi(float x) {
    unsigned r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

__global__ void __launch_bounds__(THREADS) k_probe(const float* __restrict__ A, const float* __restrict__ B,
                                                   float* __restrict__ D, unsigned* __restrict__ raw, int reps,
                                                   long long* cycles) {
    extern __shared__ __align__(1024) unsigned char sm[];  // 2 M K + 2 N K floats
    __shared__ __align__(8) unsigned long long bar;
    __shared__ unsigned tmem_base;
    float* ah = reinterpret_cast<float*>(sm);
    float* al = ah + M * K;
    float* bh = al + M * K;
    float* bl = bh + N * K;
    const int t = threadIdx.x, w = t >> 5, lane = t & 31;
    if (w == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(sa(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    for (int e = t; e < M * K; e += THREADS) {
        const int r = e / K, k = e % K;
        const float v = A[e], h = tf32_hi(v);
        *reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(ah) + kmaj_off(r, k, M)) = h;
        *reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(al) + kmaj_off(r, k, M)) = v - h;
    }
    for (int e = t; e < N * K; e += THREADS) {
        const int r = e / K, k = e % K;
        const float v = B[e], h = tf32_hi(v);
        *reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(bh) + kmaj_off(r, k, N)) = h;
        *reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(bl) + kmaj_off(r, k, N)) = v - h;
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic smem writes -> tensor core
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const unsigned tmem = tmem_base;
    long long c0 = clock64();
    unsigned phase = 0;
    for (int rep = 0; rep < reps; ++rep) {
        if (t == 0) {
#pragma unroll
            for (int ks = 0; ks < K / 8; ++ks) {
                const uint64_t dah = umma_desc(sa(ah) + ks * 2 * M * 16, M * 16, 128);
                const uint64_t dal = umma_desc(sa(al) + ks * 2 * M * 16, M * 16, 128);
                const uint64_t dbh = umma_desc(sa(bh) + ks * 2 * N * 16, N * 16, 128);
                const uint64_t dbl = umma_desc(sa(bl) + ks * 2 * N * 16, N * 16, 128);
                mma_tf32_ss(tmem, dal, dbh, ks > 0 ? 1u : 0u);
                mma_tf32_ss(tmem, dah, dbl, 1u);
                mma_tf32_ss(tmem, dah, dbh, 1u);
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                             sa(&bar))
                         : "memory");
        }
        // wait for the MMAs (phase flips each rep)
        unsigned done = 0;
        while (!done)
            asm volatile(
                "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                : "=r"(done)
                : "r"(sa(&bar)), "r"(phase)
                : "memory");
        phase ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;\n");
    }
    long long c1 = clock64();
    if (t == 0) *cycles = c1 - c0;
    // TMEM -> registers: warp w reads its lane quadrant (lanes 32w .. 32w + 15
    // hold rows 16w .. 16w + 15 for M = 64) with the 16x256b shape, 8 columns
    // per x1; raw dump: raw[((w * 24 + cb) * 32 + lane) * 4 + i]
    for (int cb = 0; cb < N / 8; ++cb) {
        unsigned r0, r1, r2, r3;
        const unsigned ta = tmem + ((unsigned)(32 * w) << 16) + (unsigned)(8 * cb);
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0, %1, %2, %3}, [%4];\n"
                     : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                     : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        unsigned* o = raw + ((size_t)(w * (N / 8) + cb) * 32 + lane) * 4;
        o[0] = r0;
        o[1] = r1;
        o[2] = r2;
        o[3] = r3;
        // hypothesis: the mma.sync accumulator fragment (g = lane / 4, c = lane % 4):
        // r0 (row g, col 2c), r1 (row g, col 2c+1), r2 (row g+8, col 2c), r3 (row g+8, col 2c+1)
        const int g = lane >> 2, c = lane & 3, row = 16 * w + g, col = 8 * cb + 2 * c;
        D[row * N + col] = __uint_as_float(r0);
        D[row * N + col + 1] = __uint_as_float(r1);
        D[(row + 8) * N + col] = __uint_as_float(r2);
        D[(row + 8) * N + col + 1] = __uint_as_float(r3);
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tmem));
}

int main() {
    std::vector<float> A(M * K), B(N * K), D(M * N, NAN);
    srand(7);
    for (auto& v : A) v = (float)rand() / RAND_MAX;
    for (auto& v : B) v = 2.f * (float)rand() / RAND_MAX - 1.f;
    float *dA, *dB, *dD;
    unsigned* dR;
    long long* dC;
    CK(cudaMalloc(&dA, A.size() * 4));
    CK(cudaMalloc(&dB, B.size() * 4));
    CK(cudaMalloc(&dD, D.size() * 4));
    CK(cudaMalloc(&dR, 4 * 24 * 32 * 4 * 4));
    CK(cudaMalloc(&dC, 8));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(dD, 0xff, D.size() * 4));
    const int smem = 2 * M * K * 4 + 2 * N * K * 4;
    CK(cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_probe<<<1, THREADS, smem>>>(dA, dB, dD, dR, 1, dC);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    std::vector<unsigned> R(4 * 24 * 32 * 4);
    CK(cudaMemcpy(R.data(), dR, R.size() * 4, cudaMemcpyDeviceToHost));
    double maxrel = 0, maxabs = 0;
    int bad = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double ref = 0, mag = 0;
            for (int k = 0; k < K; ++k) {
                ref += (double)A[m * K + k] * B[n * K + k];
                mag += fabs((double)A[m * K + k] * B[n * K + k]);
            }
            const double err = fabs(D[m * N + n] - ref);
            maxabs = fmax(maxabs, err);
            maxrel = fmax(maxrel, err / mag);
            if (!(err <= 1e-5 * mag)) ++bad;
        }
    printf("fragment-map hypothesis: %d / %d elements off (max |err| %.3g, max err/sum|ab| %.3g)\n", bad, M * N, maxabs,
           maxrel);
    if (bad) {  // locate a few raw values
        for (int w = 0; w < 1; ++w)
            for (int lane = 0; lane < 8; ++lane)
                for (int i = 0; i < 4; ++i) {
                    const float v = __builtin_bit_cast(float, R[((size_t)(w * 24 + 0) * 32 + lane) * 4 + i]);
                    int fm = -1, fn = -1;
                    for (int m = 0; m < M && fm < 0; ++m)
                        for (int n = 0; n < N; ++n) {
                            double ref = 0;
                            for (int k = 0; k < K; ++k) ref += (double)A[m * K + k] * B[n * K + k];
                            if (fabs(ref - v) < 1e-4 * (1 + fabs(ref))) {
                                fm = m;
                                fn = n;
                                break;
                            }
                        }
                    printf("warp %d lane %d reg %d -> (m %d, n %d)\n", w, lane, i, fm, fn);
                }
    }
    // throughput: reps of (K/8 k-steps x 3 MMAs) of 64 x 192 x 8
    const int reps = 20000;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int ctas = 148 * 2;
    CK(cudaEventRecord(e0));
    k_probe<<<ctas, THREADS, smem>>>(dA, dB, dD, dR, reps, dC);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double flops = 2.0 * M * N * 8 * (K / 8) * 3 * (double)reps * ctas;
    printf("throughput: %d CTAs x %d reps: %.3f ms -> %.1f TFLOP/s TF32 (3 products per k-step; serial commit+wait per rep)\n",
           ctas, reps, ms, flops / ms / 1e9);
    return bad ? 2 : 0;
}
