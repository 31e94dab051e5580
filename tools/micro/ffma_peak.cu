// FP32 FMA-pipe ceiling on this part: register-only outer-product blocks with
// the conv kernel's operand pattern (8 scalar a x 4 packed b pairs -> 32
// FFMA2 per k step), plus scalar FFMA for comparison.  Reports TFLOP/s and the
// SM clock it ran at (nvidia-smi is sampled by the caller).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma_peak ffma_peak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t ffma2(float a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm volatile("{\n\t.reg .b64 aa;\n\tmov.b64 aa, {%1, %1};\n\t"
                 "fma.rn.f32x2 %0, aa, %2, %3;\n\t}" : "=l"(d) : "f"(a), "l"(b), "l"(c));
    return d;
}

template <int ITERS>
__global__ void __launch_bounds__(256, 2) k_ffma2(float* out, float seed) {
    float a[8];
    uint64_t b[4];
    uint64_t acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + i);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        float lo = seed + j, hi = seed - j;
        b[j] = ((uint64_t)__float_as_uint(hi) << 32) | __float_as_uint(lo);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = ffma2(a[i], b[j], acc[i][j]);
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = __uint_as_float(__float_as_uint(a[i]) ^ 1u);  // keep live
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) s += __uint_as_float((uint32_t)acc[i][j]) + __uint_as_float((uint32_t)(acc[i][j] >> 32));
    if (s == 1234.5f) out[threadIdx.x] = s;
}

template <int ITERS>
__global__ void __launch_bounds__(256, 2) k_ffma(float* out, float seed) {
    float a[8], b[8], acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = seed * (threadIdx.x + i); b[i] = seed + i; }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = __uint_as_float(__float_as_uint(a[i]) ^ 1u);
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) s += acc[i][j];
    if (s == 1234.5f) out[threadIdx.x] = s;
}


__device__ __forceinline__ uint64_t ffma2p(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}

template <int ITERS, int MI, int NJ, bool PAIR, bool JOUTER = false>
__global__ void __launch_bounds__(256, 1) k_shape(float* out, float seed) {
    float a[MI];
    uint64_t ap[MI];
    uint64_t b[NJ];
    uint64_t acc[MI][NJ];
#pragma unroll
    for (int i = 0; i < MI; ++i) {
        a[i] = seed * (threadIdx.x + i);
        ap[i] = ((uint64_t)__float_as_uint(a[i] + 1) << 32) | __float_as_uint(a[i]);
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        float lo = seed + j, hi = seed - j;
        b[j] = ((uint64_t)__float_as_uint(hi) << 32) | __float_as_uint(lo);
    }
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) acc[i][j] = 0;
    for (int it = 0; it < ITERS; ++it) {
        if (JOUTER) {
#pragma unroll
            for (int j = 0; j < NJ; ++j)
#pragma unroll
                for (int i = 0; i < MI; ++i) acc[i][j] = ffma2(a[i], b[j], acc[i][j]);
        } else {
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int j = 0; j < NJ; ++j)
                acc[i][j] = PAIR ? ffma2p(ap[i], b[j], acc[i][j]) : ffma2(a[i], b[j], acc[i][j]);
        }
#pragma unroll
        for (int i = 0; i < MI; ++i) {
            a[i] = __uint_as_float(__float_as_uint(a[i]) ^ 1u);
            ap[i] ^= 1ull;
        }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) s += __uint_as_float((uint32_t)acc[i][j]) + __uint_as_float((uint32_t)(acc[i][j] >> 32));
    if (s == 1234.5f) out[threadIdx.x] = s;
}

template <typename K>
void run(const char* name, K kern, int blocks_per_sm, double flops_per_thread) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    float* out;
    cudaMalloc(&out, 1024 * sizeof(float));
    const int blocks = sms * blocks_per_sm;
    kern<<<blocks, 256>>>(out, 1.0f);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int reps = 20;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) kern<<<blocks, 256>>>(out, 1.0f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = flops_per_thread * 256.0 * blocks * reps;
    printf("%-34s %2d CTA/SM  %8.2f TFLOP/s  (%.3f ms per launch)\n", name, blocks_per_sm,
           flops / (ms * 1e-3) / 1e12, ms / reps);
    cudaFree(out);
}

int main() {
    constexpr int IT = 4096;
    for (int b : {2, 4}) {
        run("FFMA2 8x4 pairs (conv pattern)", k_ffma2<IT>, b, 2.0 * 64 * IT);
        run("FFMA  8x8 scalar", k_ffma<IT>, b, 2.0 * 64 * IT);
        run("FFMA2 bcast 4x8", k_shape<IT, 4, 8, false>, b, 2.0 * 64 * IT);
        run("FFMA2 bcast 8x4 (shape kernel)", k_shape<IT, 8, 4, false>, b, 2.0 * 64 * IT);
        run("FFMA2 bcast 8x4 j-outer", k_shape<IT, 8, 4, false, true>, b, 2.0 * 64 * IT);
        run("FFMA2 bcast 4x8 j-outer", k_shape<IT, 4, 8, false, true>, b, 2.0 * 64 * IT);
        run("FFMA2 bcast 2x16", k_shape<IT, 2, 16, false>, b, 2.0 * 64 * IT);
        run("FFMA2 bcast 2x8", k_shape<IT, 2, 8, false>, b, 2.0 * 32 * IT);
        run("FFMA2 bcast 8x2", k_shape<IT, 8, 2, false>, b, 2.0 * 32 * IT);
        run("FFMA2 pair  8x4", k_shape<IT, 8, 4, true>, b, 2.0 * 64 * IT);
        run("FFMA2 pair  4x4", k_shape<IT, 4, 4, true>, b, 2.0 * 32 * IT);
    }
    return 0;
}
