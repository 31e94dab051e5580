// Minimal TMA tensor-store check: one CTA stages a 32 x 128 fp32 box in smem
// and stores it into a (pix, ch, img) tensor with cp.async.bulk.tensor.3d,
// including a negative start coordinate (clipped) — the pattern of the
// tcgen05 epilogue.  nvcc -gencode arch=compute_100a,code=sm_100a -o t tma_store_test.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

__global__ void k(const __grid_constant__ CUtensorMap tm, int c0, int c1, int c2, int mode) {
    extern __shared__ __align__(1024) float st[];
    for (int i = threadIdx.x; i < 32 * 128; i += blockDim.x) st[i] = (float)(i + 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t s = (uint32_t)__cvta_generic_to_shared(st);
        if (mode == 0)
            asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];"
                         ::"l"(reinterpret_cast<uint64_t>(&tm)), "r"(s), "r"(c0), "r"(c1), "r"(c2) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

int main() {
    const int ohw = 144, co = 256, n = 5;
    float* y;
    cudaMalloc(&y, (size_t)ohw * co * n * 4);
    cudaMemset(y, 0, (size_t)ohw * co * n * 4);
    CUtensorMap tm;
    cuuint64_t dims[3] = {(cuuint64_t)ohw, (cuuint64_t)co, (cuuint64_t)n};
    cuuint64_t strides[2] = {(cuuint64_t)ohw * 4, (cuuint64_t)ohw * co * 4};
    cuuint32_t box[3] = {128, 32, 1}, es[3] = {1, 1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, y, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 128 * 4);
    int cases[3][3] = {{100, 32, 1}, {100 - 144, 32, 2}, {0, 0, 0}};
    for (auto& c : cases) {
        k<<<1, 128, 32 * 128 * 4>>>(tm, c[0], c[1], c[2], 0);
        cudaError_t e = cudaDeviceSynchronize();
        printf("store at (%d,%d,%d): %s\n", c[0], c[1], c[2], cudaGetErrorString(e));
        if (e) return 1;
    }
    std::vector<float> h((size_t)ohw * co * n);
    cudaMemcpy(h.data(), y, h.size() * 4, cudaMemcpyDeviceToHost);
    // (100..143, ch 32..63, img 1) = box cols 0..43; (0..83, ch 32..63, img 2) = box cols 44..127
    auto at = [&](int p, int c, int i) { return h[((size_t)i * co + c) * ohw + p]; };
    printf("y(100,32,1)=%g expect 1; y(143,33,1)=%g expect %d; y(0,32,2)=%g expect 45; y(83,32,2)=%g expect 128; y(84,32,2)=%g expect 0\n",
           at(100, 32, 1), at(143, 33, 1), 128 + 44, at(0, 32, 2), at(83, 32, 2), at(84, 32, 2));
    return 0;
}
