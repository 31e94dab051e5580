// conv_tc.cu — separately labelled tensor-core variant: bf16-input, fp32-
// accumulate SMM-Conv on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// SMM-Conv writes the convolution as a sum over kernel taps (j, k) of shifted
// windows of the input times scalar weights (smm.py:84-114).  Batching the
// reference's per-(c, m) scalar updates over all input and output channels
// turns each tap into one GEMM: for tap (j, k),
//     Y[pixel, m] += X_shift(j,k)[pixel, c] * W[c, j, k, m]
// — the "shifted GEMM" form of SMM.  The shifted window is exactly a TMA box
// of the channels-last (NHWC) input at a shifted origin, and the zero packing
// of the reference's slice (smm.py:56-73) is TMA's out-of-bounds zero fill.
//
// Kernel structure (one 128-pixel x 128-channel output tile per CTA, 4 warps):
//   warp 0, one lane : TMA producer — per (tap, 64-channel block) loads the
//                      shifted A box (128 pixel rows x 128 B, SWIZZLE_128B) and
//                      the B box (128 out-channel rows x 128 B) into a
//                      3-stage ring, completion via mbarrier transaction bytes;
//   warp 1, one lane : tcgen05.mma issuer — 4 x (M=128, N=128, K=16) per stage,
//                      fp32 accumulator in TMEM (128 lanes x 128 columns),
//                      tcgen05.commit frees the stage / signals the epilogue;
//   all 4 warps      : epilogue — tcgen05.ld 32x32b (each thread one pixel
//                      row), fp32 NCHW stores (coalesced along pixels).
// Inputs: x in bf16 NHWC and weights in bf16 [tap][c_o][c_i] (K-major), made
// once by the pack kernels below (the weight pack plays the role of the
// reference's repack_weights, smm.py:164-167).  Stride 1 only.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <mutex>

#include "smmc_internal.cuh"
#include "tc_ptx.cuh"

namespace smmc {
namespace {

constexpr int TC_BM = 128;
constexpr int TC_BN = 128;
constexpr int TC_BK = 64;  // channels per stage: one 128-byte swizzle row
constexpr int TC_STAGES = 3;
constexpr int TC_THREADS = 128;
constexpr int TC_A_BYTES = TC_BM * TC_BK * 2;
constexpr int TC_B_BYTES = TC_BN * TC_BK * 2;
constexpr int TC_SMEM = TC_STAGES * (TC_A_BYTES + TC_B_BYTES) + 1024;

struct TcParams {
    float* y;
    int n, co, oh, ow, ohw;
    int kh, kw, ph, pw, taps, cblocks;
    int tw, th, nb;                 // pixel tile = box of tw x th x nb (w, h, images)
    int tiles_w, tiles_h;
    int flat;                       // 1x1/s1/p0: A is a 2-D [pixels][c] box of 128 rows
    uint32_t tx_bytes;              // A + B bytes per stage
};

__global__ void __launch_bounds__(TC_THREADS, 1)
conv_tc_bf16_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                    const TcParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + TC_STAGES * TC_A_BYTES;
    __shared__ __align__(8) uint64_t full_bar[TC_STAGES];
    __shared__ __align__(8) uint64_t empty_bar[TC_STAGES];
    __shared__ __align__(8) uint64_t done_bar;
    __shared__ uint32_t tmem_base_sh;

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    // ---- tile coordinates
    const int mt = blockIdx.x;
    const int co0 = blockIdx.y * TC_BN;
    int ow0 = 0, oh0 = 0, n0 = 0, px0 = 0;
    if (p.flat) {
        px0 = mt * TC_BM;
    } else {
        const int tw_i = mt % p.tiles_w;
        const int rest = mt / p.tiles_w;
        const int th_i = rest % p.tiles_h;
        ow0 = tw_i * p.tw;
        oh0 = th_i * p.th;
        n0 = (rest / p.tiles_h) * p.nb;
    }
    const int kblocks = p.taps * p.cblocks;

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tm_a);
        ptx::prefetch_tmap(&tm_b);
        for (int s = 0; s < TC_STAGES; ++s) {
            ptx::mbar_init(&full_bar[s], 1);
            ptx::mbar_init(&empty_bar[s], 1);
        }
        ptx::mbar_init(&done_bar, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc(&tmem_base_sh, TC_BN);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_base_sh;

    if (warp == 0) {
        if (lane == 0) {
            // ================= TMA producer
            for (int kb = 0; kb < kblocks; ++kb) {
                const int s = kb % TC_STAGES;
                const int use = kb / TC_STAGES;
                if (use > 0) ptx::mbar_wait(&empty_bar[s], (use - 1) & 1);
                const int tap = kb / p.cblocks;
                const int c0 = (kb - tap * p.cblocks) * TC_BK;
                const int j = tap / p.kh;  // kernel column (SMM tap order j*kh + k)
                const int kr = tap - j * p.kh;
                ptx::mbar_arrive_expect_tx(&full_bar[s], p.tx_bytes);
                if (p.flat)
                    ptx::tma_load_2d(sA + s * TC_A_BYTES, &tm_a, &full_bar[s], c0, px0);
                else
                    ptx::tma_load_4d(sA + s * TC_A_BYTES, &tm_a, &full_bar[s], c0, ow0 + j - p.pw,
                                     oh0 + kr - p.ph, n0);
                ptx::tma_load_3d(sB + s * TC_B_BYTES, &tm_b, &full_bar[s], c0, co0, tap);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            // ================= MMA issuer
            constexpr uint32_t idesc = ptx::idesc_bf16(TC_BM, TC_BN);
            for (int kb = 0; kb < kblocks; ++kb) {
                const int s = kb % TC_STAGES;
                ptx::mbar_wait(&full_bar[s], (kb / TC_STAGES) & 1);
                ptx::tc_fence_after();
                const uint64_t da = ptx::desc_k_sw128(sA + s * TC_A_BYTES);
                const uint64_t db = ptx::desc_k_sw128(sB + s * TC_B_BYTES);
#pragma unroll
                for (int k = 0; k < TC_BK / 16; ++k)  // K=16 per MMA = 32 B = 2 descriptor units
                    ptx::mma_bf16(tmem, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
                ptx::mma_commit(&empty_bar[s]);
            }
            ptx::mma_commit(&done_bar);
        }
        __syncwarp();
    }

    // ================= epilogue (all warps): TMEM -> registers -> NCHW fp32
    ptx::mbar_wait(&done_bar, 0);
    ptx::tc_fence_after();
    const int row = warp * 32 + lane;  // TMEM lane == tile row == output pixel
    bool valid;
    int64_t ybase;
    if (p.flat) {
        const int px = px0 + row;
        valid = px < p.n * p.ohw;
        const int n = valid ? px / p.ohw : 0;
        ybase = (int64_t)n * p.co * p.ohw + (px - n * p.ohw);
    } else {
        const int per_img = p.tw * p.th;
        const int nb = row / per_img;
        const int r2 = row - nb * per_img;
        const int hh = r2 / p.tw;
        const int ww = r2 - hh * p.tw;
        const int n = n0 + nb, oh = oh0 + hh, ow = ow0 + ww;
        valid = nb < p.nb && n < p.n && oh < p.oh && ow < p.ow;
        ybase = (int64_t)n * p.co * p.ohw + (int64_t)oh * p.ow + ow;
    }
#pragma unroll 1
    for (int cc = 0; cc < TC_BN / 32; ++cc) {
        uint32_t v[32];
        ptx::tmem_ld_32x32b_x32(tmem + ((uint32_t)(warp * 32) << 16) + cc * 32, v);
        if (valid) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const int co = co0 + cc * 32 + i;
                if (co < p.co) p.y[ybase + (int64_t)co * p.ohw] = __uint_as_float(v[i]);
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) ptx::tmem_dealloc(tmem, TC_BN);
}

// x fp32 NCHW -> bf16 NHWC (per image a [C][HW] -> [HW][C] transpose through smem)
__global__ void pack_input_nhwc_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ out,
                                       int c, int hw) {
    __shared__ float tile[32][33];
    const int n = blockIdx.z;
    const int p0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
    const float* xs = x + (int64_t)n * c * hw;
    __nv_bfloat16* os = out + (int64_t)n * c * hw;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int cc = c0 + i, pp = p0 + threadIdx.x;
        tile[i][threadIdx.x] = (cc < c && pp < hw) ? xs[(int64_t)cc * hw + pp] : 0.0f;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int pp = p0 + i, cc = c0 + threadIdx.x;
        if (pp < hw && cc < c) os[(int64_t)pp * c + cc] = __float2bfloat16_rn(tile[threadIdx.x][i]);
    }
}

// W_smm fp32 (c_i, k_w, k_h, c_o) -> bf16 [tap = j*k_h + k][c_o][c_i]
__global__ void pack_weights_kernel(const float* __restrict__ w, __nv_bfloat16* __restrict__ out,
                                    int c, int taps, int co) {
    const int64_t total = (int64_t)taps * co * c;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int ci = (int)(i % c);
        const int64_t r = i / c;
        const int m = (int)(r % co);
        const int t = (int)(r / co);
        out[i] = __float2bfloat16_rn(w[((int64_t)ci * taps + t) * co + m]);
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

}  // namespace

TcPlan plan_tc(const smmc_geom& g) {
    TcPlan pl{};
    const int oh = (g.h + 2 * g.p_h - g.k_h) / g.s_h + 1;
    const int ow = (g.w + 2 * g.p_w - g.k_w) / g.s_w + 1;
    pl.supported = g.s_h == 1 && g.s_w == 1 && (g.c_i % 8) == 0 && g.c_i >= 8 && g.n > 0;
    pl.flat = g.k_h == 1 && g.k_w == 1 && g.p_h == 0 && g.p_w == 0;
    if (pl.flat) {
        pl.tw = pl.th = pl.nb = 0;
        pl.tiles_m = ((int64_t)g.n * oh * ow + TC_BM - 1) / TC_BM;
    } else if (oh * ow <= TC_BM / 2) {
        // several small planes per tile
        pl.tw = ow;
        pl.th = oh;
        pl.nb = TC_BM / (oh * ow);
        pl.tiles_m = (g.n + pl.nb - 1) / pl.nb;
    } else {
        pl.tw = ow < TC_BM ? ow : TC_BM;
        pl.th = TC_BM / pl.tw;
        if (pl.th > oh) pl.th = oh;
        pl.nb = 1;
        pl.tiles_m = (int64_t)((ow + pl.tw - 1) / pl.tw) * ((oh + pl.th - 1) / pl.th) * g.n;
    }
    pl.tiles_n = (g.c_o + TC_BN - 1) / TC_BN;
    return pl;
}

cudaError_t launch_tc_bf16(const uint16_t* x_nhwc, const uint16_t* w_tc, float* y, const smmc_geom& g,
                           cudaStream_t s, const char** why) {
    const TcPlan pl = plan_tc(g);
    if (!pl.supported) {
        *why = "bf16 tensor-core variant needs stride 1 and c_i % 8 == 0";
        return cudaErrorNotSupported;
    }
    PFN_cuTensorMapEncodeTiled_v12000 enc = encode_fn();
    if (!enc) {
        *why = "cuTensorMapEncodeTiled unavailable from the driver";
        return cudaErrorNotSupported;
    }
    const int oh = (g.h + 2 * g.p_h - g.k_h) / g.s_h + 1;
    const int ow = (g.w + 2 * g.p_w - g.k_w) / g.s_w + 1;
    const int taps = g.k_h * g.k_w;
    CUtensorMap tm_a, tm_b;
    CUresult r;
    uint32_t a_rows;
    if (pl.flat) {
        const cuuint64_t dims[2] = {(cuuint64_t)g.c_i, (cuuint64_t)g.n * g.h * g.w};
        const cuuint64_t strides[1] = {(cuuint64_t)g.c_i * 2};
        const cuuint32_t box[2] = {TC_BK, TC_BM};
        const cuuint32_t es[2] = {1, 1};
        r = enc(&tm_a, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(x_nhwc), dims,
                strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        a_rows = TC_BM;
    } else {
        const cuuint64_t dims[4] = {(cuuint64_t)g.c_i, (cuuint64_t)g.w, (cuuint64_t)g.h,
                                    (cuuint64_t)g.n};
        const cuuint64_t strides[3] = {(cuuint64_t)g.c_i * 2, (cuuint64_t)g.w * g.c_i * 2,
                                       (cuuint64_t)g.h * g.w * g.c_i * 2};
        const cuuint32_t box[4] = {TC_BK, (cuuint32_t)pl.tw, (cuuint32_t)pl.th, (cuuint32_t)pl.nb};
        const cuuint32_t es[4] = {1, 1, 1, 1};
        r = enc(&tm_a, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint16_t*>(x_nhwc), dims,
                strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        a_rows = (uint32_t)(pl.tw * pl.th * pl.nb);
    }
    if (r != CUDA_SUCCESS) {
        *why = "cuTensorMapEncodeTiled(A) failed";
        return cudaErrorInvalidValue;
    }
    {
        const cuuint64_t dims[3] = {(cuuint64_t)g.c_i, (cuuint64_t)g.c_o, (cuuint64_t)taps};
        const cuuint64_t strides[2] = {(cuuint64_t)g.c_i * 2, (cuuint64_t)g.c_o * g.c_i * 2};
        const cuuint32_t box[3] = {TC_BK, TC_BN, 1};
        const cuuint32_t es[3] = {1, 1, 1};
        r = enc(&tm_b, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<uint16_t*>(w_tc), dims,
                strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) {
        *why = "cuTensorMapEncodeTiled(B) failed";
        return cudaErrorInvalidValue;
    }
    TcParams p{};
    p.y = y;
    p.n = g.n;
    p.co = g.c_o;
    p.oh = oh;
    p.ow = ow;
    p.ohw = oh * ow;
    p.kh = g.k_h;
    p.kw = g.k_w;
    p.ph = g.p_h;
    p.pw = g.p_w;
    p.taps = taps;
    p.cblocks = (g.c_i + TC_BK - 1) / TC_BK;
    p.tw = pl.tw;
    p.th = pl.th;
    p.nb = pl.nb;
    p.tiles_w = pl.flat ? 1 : (ow + pl.tw - 1) / pl.tw;
    p.tiles_h = pl.flat ? 1 : (oh + pl.th - 1) / pl.th;
    p.flat = pl.flat;
    p.tx_bytes = a_rows * TC_BK * 2 + TC_B_BYTES;

    static std::once_flag once;
    static cudaError_t attr = cudaSuccess;
    std::call_once(once, [] {
        attr = cudaFuncSetAttribute(conv_tc_bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    TC_SMEM);
    });
    if (attr != cudaSuccess) return attr;
    dim3 grid((unsigned)pl.tiles_m, (unsigned)pl.tiles_n);
    conv_tc_bf16_kernel<<<grid, TC_THREADS, TC_SMEM, s>>>(tm_a, tm_b, p);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_pack_input_nhwc(const float* x, uint16_t* out, const smmc_geom& g,
                                   cudaStream_t s) {
    const int hw = g.h * g.w;
    dim3 grid((hw + 31) / 32, (g.c_i + 31) / 32, g.n);
    pack_input_nhwc_kernel<<<grid, dim3(32, 8), 0, s>>>(x, reinterpret_cast<__nv_bfloat16*>(out),
                                                        g.c_i, hw);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_pack_weights_bf16(const float* w, uint16_t* out, const smmc_geom& g,
                                     cudaStream_t s) {
    const int64_t total = (int64_t)g.k_h * g.k_w * g.c_o * g.c_i;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    pack_weights_kernel<<<blocks, 256, 0, s>>>(w, reinterpret_cast<__nv_bfloat16*>(out), g.c_i,
                                               g.k_h * g.k_w, g.c_o);
    count_launches(1);
    return cudaGetLastError();
}

}  // namespace smmc
