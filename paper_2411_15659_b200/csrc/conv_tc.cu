// conv_tc.cu — separately labelled tensor-core variant: bf16-input, fp32-
// accumulate SMM-Conv on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// SMM-Conv writes the convolution as a sum over kernel taps (j, k) of shifted
// windows of the zero-padded input times scalar weights (smm.py:56-114).
// Batching the reference's per-(c, m) scalar updates over all input and output
// channels turns each tap into one GEMM:
//     Y[pixel, m] += X_pad_shift(j,k)[pixel, c] * W[c, j, k, m]
// — the "shifted GEMM" form of SMM.
//
// Zero packing.  The pack pass writes the input once as a zero-padded,
// channels-last bf16 tensor X_pad (n, h + 2p_h, w + 2p_w, c) — the reference's
// padded slice buffer (smm.py:56-73) materialised for all channels at once.
// In the flattened padded pixel index q = (n*Hp + r)*Wp + t, output pixel
// (oh, ow) of image n sits at q and tap (k, j) reads q + k*Wp + j: every tap's
// A operand is the SAME contiguous run of 128 rows shifted by a constant.
//
// conv_tc_halo_kernel (Wp small enough: (k_h-1)*Wp + k_w-1 + 128 <= 256 rows):
//   per 64-channel block ONE TMA box of R = 128 + (k_h-1)*Wp + (k_w-1) rows
//   (the "halo") is loaded; the k_h*k_w taps are UMMA smem descriptors whose
//   start address is offset by (k*Wp + j) rows inside it ("shifting" = pure
//   descriptor arithmetic, as shifted_view is pure view arithmetic in
//   smm.py:206-214).  A traffic drops by ~k_h*k_w versus one box per tap.
//   Rows whose q is not a valid output (padding columns/rows) are computed and
//   discarded.
// conv_tc_box_kernel (wide planes): per (tap, channel block) a 4-D box of
//   tw x th x nb output pixels at the shifted origin of X_pad.
//
// Both: one 128-pixel x 128-channel tile per CTA, 4 warps — warp 0 lane 0 TMA
// producer (mbarrier transaction bytes), warp 1 lane 0 tcgen05.mma issuer
// (M=128, N=128, K=16, fp32 accumulator in TMEM), all warps epilogue
// (tcgen05.ld 32x32b, each thread one pixel row, fp32 NCHW stores).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "smmc_internal.cuh"
#include "tc_ptx.cuh"

namespace smmc {
namespace {

constexpr int TC_BM = 128;
constexpr int TC_BN = 128;
constexpr int TC_BK = 64;  // channels per block: one 128-byte swizzle row
constexpr int TC_THREADS = 128;
constexpr int TC_B_BYTES = TC_BN * TC_BK * 2;

// box kernel ring
constexpr int BOX_STAGES = 3;
constexpr int BOX_A_BYTES = TC_BM * TC_BK * 2;
constexpr int BOX_SMEM = BOX_STAGES * (BOX_A_BYTES + TC_B_BYTES) + 1024;

// halo kernel rings: 2 A halos (<= 256 rows, stage size set at launch so that
// two CTAs fit one SM) and 3 per-tap B tiles
constexpr int HALO_A_STAGES = 2;
constexpr int HALO_B_STAGES = 3;
constexpr int HALO_SMEM_MAX = HALO_A_STAGES * 256 * 128 + HALO_B_STAGES * 2 * TC_B_BYTES + 1024;

struct TcParams {
    float* y;
    int n, co, oh, ow, ohw;
    int hp, wp;                     // padded input plane
    int kh, kw, taps, cblocks;
    // box kernel
    int tw, th, nb, tiles_w, tiles_h;
    // halo kernel
    int halo_rows;
    int halo_stage_bytes;           // A halo stage stride (1024-aligned)
    int b_stages;                   // persistent kernel: B ring depth
    int tiles_m, tiles_n;           // persistent kernel: tile space (tile = m * tiles_n + n)
    uint32_t tx_a, tx_b;            // TMA bytes per A box / B box
    // persistent kernel split-K over channel blocks (few-tile layers): work
    // item t = tile * splits + s covers channel blocks [s*cb_per_split, ...)
    // and writes fp32 partial planes ws[s] (n, co, oh, ow), summed in split
    // order by tc_split_reduce_kernel
    int splits, cb_per_split;
    float* ws;
    int64_t y_elems;
};

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
    return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// Descriptor of a K-major SW128 operand that starts `row` 128-byte rows into
// a 1024-byte-aligned TMA tile.  The 128-byte swizzle is a function of the
// absolute shared-memory address on both sides (TMA write, UMMA read), so a
// row-shifted start needs no base-offset correction (verified on B200: with
// the base-offset field set to row % 8 the parity tests fail, with 0 they pass).
__device__ __forceinline__ uint64_t desc_rows(const uint8_t* tile, int row) {
    return ptx::desc_k_sw128(tile + row * 128);
}

// Epilogue: TMEM (128 lanes x 128 fp32 columns) -> NCHW fp32.  `ybase` is the
// offset of (n, co=0, oh, ow) for this thread's pixel row.
template <int NCOL = TC_BN>
__device__ __forceinline__ void store_tile(const TcParams& p, uint32_t tmem, int warp, bool valid,
                                           int64_t ybase, int co0) {
#pragma unroll 1
    for (int cc = 0; cc < NCOL / 32; ++cc) {
        uint32_t v[32];
        ptx::tmem_ld_32x32b_x32(tmem + ((uint32_t)(warp * 32) << 16) + cc * 32, v);
        if (valid) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const int co = co0 + cc * 32 + i;
                if (co < p.co) {
                    SMMC_CHECK_RANGE(ybase + (int64_t)co * p.ohw, 1, p.y_elems);
                    p.y[ybase + (int64_t)co * p.ohw] = __uint_as_float(v[i]);
                }
            }
        }
    }
}

template <int HBN>
__global__ void __launch_bounds__(TC_THREADS, 1)
conv_tc_halo_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                    const TcParams p) {
    constexpr int HB_BYTES = HBN * TC_BK * 2;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    const int a_bytes = p.halo_stage_bytes;
    uint8_t* sA = smem;                                   // [HALO_A_STAGES][R rows x 128 B]
    uint8_t* sB = smem + HALO_A_STAGES * a_bytes;         // [HALO_B_STAGES][128 rows x 128 B]
    __shared__ __align__(8) uint64_t a_full[HALO_A_STAGES], a_empty[HALO_A_STAGES];
    __shared__ __align__(8) uint64_t b_full[HALO_B_STAGES], b_empty[HALO_B_STAGES];
    __shared__ __align__(8) uint64_t done_bar;
    __shared__ uint32_t tmem_base_sh;

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int q0 = blockIdx.x * TC_BM;  // first flattened padded pixel of the tile
    const int co0 = blockIdx.y * HBN;

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tm_a);
        ptx::prefetch_tmap(&tm_b);
        for (int s = 0; s < HALO_A_STAGES; ++s) {
            ptx::mbar_init(&a_full[s], 1);
            ptx::mbar_init(&a_empty[s], 1);
        }
        for (int s = 0; s < HALO_B_STAGES; ++s) {
            ptx::mbar_init(&b_full[s], 1);
            ptx::mbar_init(&b_empty[s], 1);
        }
        ptx::mbar_init(&done_bar, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 1) ptx::tmem_alloc(&tmem_base_sh, HBN);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_base_sh;

    if (warp == 0) {
        if (lane == 0) {
            // ================= TMA producer: one halo per channel block, B per tap
            int bi = 0;
            for (int cb = 0; cb < p.cblocks; ++cb) {
                const int sa = cb % HALO_A_STAGES;
                if (cb >= HALO_A_STAGES) ptx::mbar_wait(&a_empty[sa], ((cb / HALO_A_STAGES) - 1) & 1);
                ptx::mbar_arrive_expect_tx(&a_full[sa], p.tx_a);
                ptx::tma_load_2d(sA + sa * a_bytes, &tm_a, &a_full[sa], cb * TC_BK, q0);
                for (int tap = 0; tap < p.taps; ++tap, ++bi) {
                    const int sb = bi % HALO_B_STAGES;
                    if (bi >= HALO_B_STAGES) ptx::mbar_wait(&b_empty[sb], ((bi / HALO_B_STAGES) - 1) & 1);
                    ptx::mbar_arrive_expect_tx(&b_full[sb], p.tx_b);
                    ptx::tma_load_3d(sB + sb * HB_BYTES, &tm_b, &b_full[sb], cb * TC_BK, co0, tap);
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            // ================= MMA issuer
            constexpr uint32_t idesc = ptx::idesc_bf16(TC_BM, HBN);
            int bi = 0;
            for (int cb = 0; cb < p.cblocks; ++cb) {
                const int sa = cb % HALO_A_STAGES;
                ptx::mbar_wait(&a_full[sa], (cb / HALO_A_STAGES) & 1);
                for (int tap = 0; tap < p.taps; ++tap, ++bi) {
                    const int sb = bi % HALO_B_STAGES;
                    ptx::mbar_wait(&b_full[sb], (bi / HALO_B_STAGES) & 1);
                    ptx::tc_fence_after();
                    const int j = tap / p.kh;  // SMM tap order j*kh + k
                    const int kr = tap - j * p.kh;
                    const uint64_t da = desc_rows(sA + sa * a_bytes, kr * p.wp + j);
                    const uint64_t db = ptx::desc_k_sw128(sB + sb * HB_BYTES);
#pragma unroll
                    for (int k = 0; k < TC_BK / 16; ++k)
                        ptx::mma_bf16(tmem, da + 2 * k, db + 2 * k, idesc, (bi | k) != 0);
                    ptx::mma_commit(&b_empty[sb]);
                }
                ptx::mma_commit(&a_empty[sa]);
            }
            ptx::mma_commit(&done_bar);
        }
        __syncwarp();
    }

    // ================= epilogue
    ptx::mbar_wait(&done_bar, 0);
    ptx::tc_fence_after();
    const int q = q0 + warp * 32 + lane;
    const int plane = p.hp * p.wp;
    const int n = q / plane;
    const int r = q - n * plane;
    const int oh = r / p.wp;
    const int ow = r - oh * p.wp;
    const bool valid = n < p.n && oh < p.oh && ow < p.ow;
    const int64_t ybase = (int64_t)n * p.co * p.ohw + (int64_t)oh * p.ow + ow;
    store_tile<HBN>(p, tmem, warp, valid, ybase, co0);
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) ptx::tmem_dealloc(tmem, HBN);
}

// Persistent, warp-specialised halo kernel for c_o >= 256 (one CTA per SM,
// 2 + PH_EPI_WARPS warps, N = HBN output channels per tile):
//   warp 0 lane 0 : TMA producer over this CTA's tiles — per 64-channel block
//                   one halo box (A ring, 2 deep), per tap one B tile (B ring as
//                   deep as smem allows);
//   warp 1 lane 0 : tcgen05.mma issuer (M=128, N=HBN: 4 x 128-cycle MMAs per
//                   stage, so per-stage barrier/issue overhead is amortised)
//                   into one of TWO HBN-column TMEM accumulators; MT = 2
//                   stacks two 128-pixel sub-tiles (two halo boxes) on one B
//                   stage, for c_o = 128 layers that cannot use N = 256;
//   warps 2..9    : epilogue of the previous tile while the next one computes
//                   (warp w reads TMEM lanes 32*(w%4)..., half the columns).
#ifndef PH_EPI_WARPS_OVERRIDE  // A/B builds: 4, 8 or 16
constexpr int PH_EPI_WARPS = 16;  // four per TMEM lane quarter, each a quarter of the columns
#else
constexpr int PH_EPI_WARPS = PH_EPI_WARPS_OVERRIDE;
#endif
constexpr int PH_THREADS = 64 + 32 * PH_EPI_WARPS;
constexpr int PH_ACC = 2;
constexpr int PH_B_MAX = 8;

template <int HBN, int MT>
__global__ void __launch_bounds__(PH_THREADS, 1)
conv_tc_halo_persistent_kernel(const __grid_constant__ CUtensorMap tm_a,
                               const __grid_constant__ CUtensorMap tm_b, const TcParams p) {
    constexpr int HB_BYTES = HBN * TC_BK * 2;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    const int a_bytes = p.halo_stage_bytes;
    const int b_stages = p.b_stages;
    uint8_t* sA = smem;
    uint8_t* sB = smem + HALO_A_STAGES * MT * a_bytes;
    __shared__ __align__(8) uint64_t a_full[HALO_A_STAGES], a_empty[HALO_A_STAGES];
    __shared__ __align__(8) uint64_t b_full[PH_B_MAX], b_empty[PH_B_MAX];
    __shared__ __align__(8) uint64_t acc_full[PH_ACC], acc_empty[PH_ACC];
    __shared__ uint32_t tmem_base_sh;

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int items = p.tiles_m * p.tiles_n * p.splits;  // (tile, split) work items

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tm_a);
        ptx::prefetch_tmap(&tm_b);
        for (int s = 0; s < HALO_A_STAGES; ++s) {
            ptx::mbar_init(&a_full[s], 1);
            ptx::mbar_init(&a_empty[s], 1);
        }
        for (int s = 0; s < b_stages; ++s) {
            ptx::mbar_init(&b_full[s], 1);
            ptx::mbar_init(&b_empty[s], 1);
        }
        for (int s = 0; s < PH_ACC; ++s) {
            ptx::mbar_init(&acc_full[s], 1);
            ptx::mbar_init(&acc_empty[s], PH_EPI_WARPS);  // one arrival per epilogue warp
        }
        ptx::fence_mbar_init();
    }
    if (warp == 2) ptx::tmem_alloc(&tmem_base_sh, PH_ACC * MT * HBN);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_base_sh;

    if (warp == 0) {
        if (lane == 0) {
            int ai = 0, bi = 0;
            for (int it = blockIdx.x; it < items; it += gridDim.x) {
                const int t = it / p.splits;
                const int cb0 = (it - t * p.splits) * p.cb_per_split;
                const int cb1 = min(p.cblocks, cb0 + p.cb_per_split);
                const int q0 = (t / p.tiles_n) * (TC_BM * MT);
                const int co0 = (t % p.tiles_n) * HBN;
                for (int cb = cb0; cb < cb1; ++cb, ++ai) {
                    const int sa = ai % HALO_A_STAGES;
                    if (ai >= HALO_A_STAGES)
                        ptx::mbar_wait(&a_empty[sa], ((ai / HALO_A_STAGES) - 1) & 1);
                    ptx::mbar_arrive_expect_tx(&a_full[sa], MT * p.tx_a);
#pragma unroll
                    for (int m = 0; m < MT; ++m)
                        ptx::tma_load_2d(sA + (sa * MT + m) * a_bytes, &tm_a, &a_full[sa], cb * TC_BK,
                                         q0 + m * TC_BM);
                    for (int tap = 0; tap < p.taps; ++tap, ++bi) {
                        const int sb = bi % b_stages;
                        if (bi >= b_stages) ptx::mbar_wait(&b_empty[sb], ((bi / b_stages) - 1) & 1);
                        ptx::mbar_arrive_expect_tx(&b_full[sb], p.tx_b);
                        ptx::tma_load_3d(sB + sb * HB_BYTES, &tm_b, &b_full[sb], cb * TC_BK, co0, tap);
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = ptx::idesc_bf16(TC_BM, HBN);
            int ai = 0, bi = 0, local = 0;
            for (int it = blockIdx.x; it < items; it += gridDim.x, ++local) {
                const int t = it / p.splits;
                const int cb0 = (it - t * p.splits) * p.cb_per_split;
                const int cb1 = min(p.cblocks, cb0 + p.cb_per_split);
                const int acc = local % PH_ACC;
                if (local >= PH_ACC) ptx::mbar_wait(&acc_empty[acc], ((local / PH_ACC) - 1) & 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem + acc * MT * HBN;
                bool first = true;
                for (int cb = cb0; cb < cb1; ++cb, ++ai) {
                    const int sa = ai % HALO_A_STAGES;
                    ptx::mbar_wait(&a_full[sa], (ai / HALO_A_STAGES) & 1);
                    for (int tap = 0; tap < p.taps; ++tap, ++bi) {
                        const int sb = bi % b_stages;
                        ptx::mbar_wait(&b_full[sb], (bi / b_stages) & 1);
                        ptx::tc_fence_after();
                        const int j = tap / p.kh;  // SMM tap order j*kh + k
                        const int kr = tap - j * p.kh;
                        const uint64_t db = ptx::desc_k_sw128(sB + sb * HB_BYTES);
#pragma unroll
                        for (int m = 0; m < MT; ++m) {
                            const uint64_t da = desc_rows(sA + (sa * MT + m) * a_bytes, kr * p.wp + j);
#pragma unroll
                            for (int k = 0; k < TC_BK / 16; ++k)
                                ptx::mma_bf16(d + m * HBN, da + 2 * k, db + 2 * k, idesc,
                                              (first && k == 0) ? 0u : 1u);
                        }
                        first = false;
                        ptx::mma_commit(&b_empty[sb]);
                    }
                    ptx::mma_commit(&a_empty[sa]);
                }
                ptx::mma_commit(&acc_full[acc]);
            }
        }
        __syncwarp();
    } else {
        const int quarter = warp & 3;  // TMEM lane quarter this warp may access
        constexpr int parts = PH_EPI_WARPS / 4;  // column slices per lane quarter
        constexpr int chunks = MT * HBN / 32 / parts;
        const int part = (warp - 2) >> 2;
        const int plane = p.hp * p.wp;
        int local = 0;
        for (int it = blockIdx.x; it < items; it += gridDim.x, ++local) {
            const int t = it / p.splits;
            float* const yo = p.splits > 1 ? p.ws + (int64_t)(it - t * p.splits) * p.y_elems : p.y;
            const int acc = local % PH_ACC;
            ptx::mbar_wait(&acc_full[acc], (local / PH_ACC) & 1);
            ptx::tc_fence_after();
            const int co0 = (t % p.tiles_n) * HBN;
#pragma unroll 1
            for (int c = part * chunks; c < (part + 1) * chunks; ++c) {
                const int m = c / (HBN / 32);  // M sub-tile
                const int cc = c - m * (HBN / 32);
                const int q = (t / p.tiles_n) * (TC_BM * MT) + m * TC_BM + quarter * 32 + lane;
                const int n = q / plane;
                const int r = q - n * plane;
                const int oh = r / p.wp;
                const int ow = r - oh * p.wp;
                const bool valid = n < p.n && oh < p.oh && ow < p.ow;
                const int64_t ybase = (int64_t)n * p.co * p.ohw + (int64_t)oh * p.ow + ow;
                uint32_t v[32];
                ptx::tmem_ld_32x32b_x32(
                    tmem + ((uint32_t)(quarter * 32) << 16) + (acc * MT + m) * HBN + cc * 32, v);
                if (valid) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int co = co0 + cc * 32 + i;
                        if (co < p.co) {
                            SMMC_CHECK_RANGE(ybase + (int64_t)co * p.ohw, 1, p.y_elems);
                            yo[ybase + (int64_t)co * p.ohw] = __uint_as_float(v[i]);
                        }
                    }
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&acc_empty[acc]);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) ptx::tmem_dealloc(tmem, PH_ACC * MT * HBN);
}

// y = ws[0] + ws[1] + ... in split order (deterministic)
__global__ void __launch_bounds__(256) tc_split_reduce_kernel(const float* __restrict__ ws,
                                                              float* __restrict__ y, int64_t total,
                                                              int splits) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if ((total & 3) == 0) {
        const float4* w4 = reinterpret_cast<const float4*>(ws);
        const int64_t t4 = total >> 2;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < t4; i += stride) {
            float4 a = __ldcg(w4 + i);
            for (int z = 1; z < splits; ++z) {
                const float4 v = __ldcg(w4 + z * t4 + i);
                a.x += v.x;
                a.y += v.y;
                a.z += v.z;
                a.w += v.w;
            }
            reinterpret_cast<float4*>(y)[i] = a;
        }
        return;
    }
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        float a = ws[i];
        for (int z = 1; z < splits; ++z) a += ws[z * total + i];
        y[i] = a;
    }
}

__global__ void __launch_bounds__(TC_THREADS, 1)
conv_tc_box_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
                   const TcParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = align1024(smem_raw);
    uint8_t* sA = smem;
    uint8_t* sB = smem + BOX_STAGES * BOX_A_BYTES;
    __shared__ __align__(8) uint64_t full_bar[BOX_STAGES];
    __shared__ __align__(8) uint64_t empty_bar[BOX_STAGES];
    __shared__ __align__(8) uint64_t done_bar;
    __shared__ uint32_t tmem_base_sh;

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int mt = blockIdx.x;
    const int co0 = blockIdx.y * TC_BN;
    const int tw_i = mt % p.tiles_w;
    const int rest = mt / p.tiles_w;
    const int th_i = rest % p.tiles_h;
    const int ow0 = tw_i * p.tw;
    const int oh0 = th_i * p.th;
    const int n0 = (rest / p.tiles_h) * p.nb;
    const int kblocks = p.taps * p.cblocks;

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tm_a);
        ptx::prefetch_tmap(&tm_b);
        for (int s = 0; s < BOX_STAGES; ++s) {
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
            for (int kb = 0; kb < kblocks; ++kb) {
                const int s = kb % BOX_STAGES;
                const int use = kb / BOX_STAGES;
                if (use > 0) ptx::mbar_wait(&empty_bar[s], (use - 1) & 1);
                const int tap = kb / p.cblocks;
                const int c0 = (kb - tap * p.cblocks) * TC_BK;
                const int j = tap / p.kh;
                const int kr = tap - j * p.kh;
                ptx::mbar_arrive_expect_tx(&full_bar[s], p.tx_a + p.tx_b);
                // padded input: output (oh, ow) + tap (k, j) reads X_pad[oh + k][ow + j]
                ptx::tma_load_4d(sA + s * BOX_A_BYTES, &tm_a, &full_bar[s], c0, ow0 + j, oh0 + kr, n0);
                ptx::tma_load_3d(sB + s * TC_B_BYTES, &tm_b, &full_bar[s], c0, co0, tap);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = ptx::idesc_bf16(TC_BM, TC_BN);
            for (int kb = 0; kb < kblocks; ++kb) {
                const int s = kb % BOX_STAGES;
                ptx::mbar_wait(&full_bar[s], (kb / BOX_STAGES) & 1);
                ptx::tc_fence_after();
                const uint64_t da = ptx::desc_k_sw128(sA + s * BOX_A_BYTES);
                const uint64_t db = ptx::desc_k_sw128(sB + s * TC_B_BYTES);
#pragma unroll
                for (int k = 0; k < TC_BK / 16; ++k)
                    ptx::mma_bf16(tmem, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
                ptx::mma_commit(&empty_bar[s]);
            }
            ptx::mma_commit(&done_bar);
        }
        __syncwarp();
    }

    ptx::mbar_wait(&done_bar, 0);
    ptx::tc_fence_after();
    const int row = warp * 32 + lane;
    const int per_img = p.tw * p.th;
    const int nb = row / per_img;
    const int r2 = row - nb * per_img;
    const int hh = r2 / p.tw;
    const int ww = r2 - hh * p.tw;
    const int n = n0 + nb, oh = oh0 + hh, ow = ow0 + ww;
    const bool valid = nb < p.nb && n < p.n && oh < p.oh && ow < p.ow;
    const int64_t ybase = (int64_t)n * p.co * p.ohw + (int64_t)oh * p.ow + ow;
    store_tile(p, tmem, warp, valid, ybase, co0);
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) ptx::tmem_dealloc(tmem, TC_BN);
}

// x fp32 NCHW -> zero-padded bf16 NHWC (n, h + 2p_h, w + 2p_w, c): one block
// per (32 padded columns, 32 channels, padded row, image), smem transpose.
// split = 3 (the fp32-accurate "bf16x3" path): x = hi + lo with hi =
// bf16(x), lo = bf16(x - hi) (|x - hi - lo| <= 2^-16 |x|), written as 3*c
// channels [hi | lo | hi]; paired with weights [hi | hi | lo] the same bf16
// GEMM sums x_hi*w_hi + x_lo*w_hi + x_hi*w_lo in fp32 (TMEM): fp32-grade
// products (the dropped x_lo*w_lo term is ~2^-16 relative) on tcgen05.
__device__ __forceinline__ void split_bf16(float v, __nv_bfloat16& hi, __nv_bfloat16& lo) {
    hi = __float2bfloat16_rn(v);
    lo = __float2bfloat16_rn(v - __bfloat162float(hi));
}

__global__ void __launch_bounds__(256) pack_input_padded_kernel(
    const float* __restrict__ x, __nv_bfloat16* __restrict__ out, int c, int h, int w, int ph, int pw,
    int hp, int wp, int split) {
    // tile: 32 channels x 64 padded columns of one padded row.  Loads are
    // 256-byte rows of one channel; stores are 16-byte runs of 8 channels of
    // one pixel (c % 8 == 0), i.e. whole 32-byte sectors per warp.
    __shared__ float tile[32][65];
    const int t0 = blockIdx.x * 64, c0 = blockIdx.y * 32;
    const int n = blockIdx.z / hp, r = blockIdx.z - n * hp;
    const int ih = r - ph;
    const bool row_in = (unsigned)ih < (unsigned)h;
    const int tid = threadIdx.x;
    {
        const int px = tid & 63, cq = tid >> 6;  // 4 channel quarters of 8
        const int iw = t0 + px - pw;
        const bool col_in = row_in && (unsigned)iw < (unsigned)w;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int cc = c0 + cq * 8 + k;
            float v = 0.0f;
            if (col_in && cc < c) v = __ldg(x + (((int64_t)n * c + cc) * h + ih) * w + iw);
            tile[cq * 8 + k][px] = v;
        }
    }
    __syncthreads();
    const int px = tid >> 2, grp = tid & 3;
    const int t = t0 + px, cc = c0 + grp * 8;
    if (t >= wp || cc >= c) return;
    const int cs = c * split;  // channels per padded pixel
    __nv_bfloat16* o = out + (((int64_t)n * hp + r) * wp + t) * cs + cc;
    __align__(16) __nv_bfloat16 hi[8], lo[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const float v = tile[grp * 8 + k][px];
        if (split == 1)
            hi[k] = __float2bfloat16_rn(v);
        else
            split_bf16(v, hi[k], lo[k]);
    }
    *reinterpret_cast<uint4*>(o) = *reinterpret_cast<const uint4*>(hi);
    if (split != 1) {  // [hi | lo | hi]
        *reinterpret_cast<uint4*>(o + c) = *reinterpret_cast<const uint4*>(lo);
        *reinterpret_cast<uint4*>(o + 2 * c) = *reinterpret_cast<const uint4*>(hi);
    }
}

// W_smm fp32 (c_i, k_w, k_h, c_o) -> bf16 [tap = j*k_h + k][c_o][c_i]
__global__ void pack_weights_kernel(const float* __restrict__ w, __nv_bfloat16* __restrict__ out,
                                    int c, int taps, int co, int split) {
    const int64_t total = (int64_t)taps * co * c;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int ci = (int)(i % c);
        const int64_t rr = i / c;
        const int m = (int)(rr % co);
        const int t = (int)(rr / co);
        const float v = w[((int64_t)ci * taps + t) * co + m];
        if (split == 1) {
            out[i] = __float2bfloat16_rn(v);
        } else {  // [hi | hi | lo] per (tap, c_o) row of 3*c channels
            __nv_bfloat16 hi, lo;
            split_bf16(v, hi, lo);
            __nv_bfloat16* row = out + rr * 3 * c;
            row[ci] = hi;
            row[c + ci] = hi;
            row[2 * c + ci] = lo;
        }
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    });
    return fn;
}

CUresult encode(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims,
                const cuuint64_t* strides, const cuuint32_t* box) {
    const cuuint32_t es[5] = {1, 1, 1, 1, 1};
    return encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims,
                       strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

}  // namespace

TcPlan plan_tc(const smmc_geom& g) {
    TcPlan pl{};
    const int oh = (g.h + 2 * g.p_h - g.k_h) / g.s_h + 1;
    const int ow = (g.w + 2 * g.p_w - g.k_w) / g.s_w + 1;
    const int hp = g.h + 2 * g.p_h, wp = g.w + 2 * g.p_w;
    pl.supported = g.s_h == 1 && g.s_w == 1 && (g.c_i % 8) == 0 && g.c_i >= 8 && g.n > 0;
    const int halo_rows = TC_BM + (g.k_h - 1) * wp + (g.k_w - 1);
    pl.halo = halo_rows <= 256;
    if (const char* f = getenv("SMMC_TC_KERNEL")) pl.halo = pl.halo && f[0] != 'b';  // A/B hook
    pl.halo_rows = halo_rows;
    if (pl.halo) {
        pl.tiles_m = ((int64_t)g.n * hp * wp + TC_BM - 1) / TC_BM;
    } else if (oh * ow <= TC_BM / 2) {
        pl.tw = ow;
        pl.th = oh;
        pl.nb = TC_BM / (oh * ow);
        pl.tiles_m = (g.n + pl.nb - 1) / pl.nb;
    } else {
        pl.tw = ow < TC_BM ? ow : TC_BM;
        pl.th = std::min(TC_BM / pl.tw, oh);
        pl.nb = 1;
        pl.tiles_m = (int64_t)((ow + pl.tw - 1) / pl.tw) * ((oh + pl.th - 1) / pl.th) * g.n;
    }
    // N = 256 runs the persistent warp-specialised kernel (one CTA/SM, TMEM
    // double-buffered so 16 epilogue warps drain one tile while the next one
    // computes). Its 128-cycle MMAs amortise the per-stage barrier/issue
    // overhead that caps the N = 128 kernel; it needs enough tiles to fill
    // 148 SMs twice (measured): conv256@14_n256 74.7 -> 60.7 us,
    // vgg 512@28_n64 217 -> 195 us, 1x1 64->256@56_n256 284 -> 184 us, while
    // small-batch layers (few tiles) lose.
    pl.bn = TC_BN;
    pl.persistent = 0;
    if (pl.halo && g.c_o >= 256) {
        const int64_t tiles256 = pl.tiles_m * ((g.c_o + 255) / 256);
        if (g.c_o % 256 == 0 && tiles256 >= 2 * 148) pl.bn = 256;
        if (const char* f = getenv("SMMC_TC_BN")) pl.bn = atoi(f) == 256 ? 256 : TC_BN;  // A/B hook
    }
    if (pl.halo) {
        // N = 128 tiles go persistent (for the 16-warp epilogue) only when they
        // fit one wave anyway: 512@7_n32 28.6 -> 26.8 us, 256@14_n32 18.5 -> 17.0,
        // but 128@28_n32 (225 tiles) 14.1 -> 17.5 us.
        pl.persistent = pl.bn == 256 || pl.tiles_m * ((g.c_o + TC_BN - 1) / TC_BN) <= 148;
    }
    // N = 128 layers with many tiles (c_o = 128): two stacked 128-pixel
    // sub-tiles share each B stage (8 MMAs per barrier round instead of 4):
    // 128@28_n256 86.9 -> 76.3 us; with fewer tiles the halved tile count loses.
    pl.mt = 1;
    if (pl.halo && pl.bn == TC_BN && (pl.tiles_m / 2) * ((g.c_o + TC_BN - 1) / TC_BN) >= 2 * 148) {
        pl.persistent = 1;
        pl.mt = 2;
    }
    if (const char* f = getenv("SMMC_TC_PERSIST")) {  // A/B hooks
        pl.persistent = pl.halo && (pl.bn == 256 || atoi(f) != 0);
        if (!pl.persistent) pl.mt = 1;
    }
    if (pl.persistent && pl.bn == TC_BN) {
        if (const char* f = getenv("SMMC_TC_MT")) pl.mt = atoi(f) == 2 ? 2 : 1;
    }
    pl.tiles_n = (g.c_o + pl.bn - 1) / pl.bn;
    // few-tile layers (N = 1, 7x7 planes): split the channel blocks across
    // CTAs of the persistent kernel so that ~148 work items run, partial
    // planes summed in split order by a second kernel (needs the workspace
    // of smmc_tc_workspace_bytes)
    const int cblocks = (g.c_i + TC_BK - 1) / TC_BK;
    pl.splits = 1;
    pl.cb_per_split = cblocks;
    const int64_t tiles = pl.tiles_m * pl.tiles_n;
    int want = (pl.halo && pl.mt == 1 && tiles < 148) ? (int)std::min<int64_t>(cblocks, 148 / tiles) : 1;
    if (want == 1 && pl.halo && pl.mt == 1 && tiles < 148) {
        // 75-147 tiles: pick S so that tiles*S fills whole waves of 148
        // (wave count per unit of K, plus a per-split cost); measured on
        // 512@7 N=32, 84 tiles: S=5 66 us vs 85 unsplit (bf16x3)
        double best = 1.0;
        for (int sp = 2; sp <= cblocks; ++sp) {
            const double cost = (double)((tiles * sp + 147) / 148) / sp + 0.02 * sp;
            if (cost < best - 1e-9) {
                best = cost;
                want = sp;
            }
        }
    }
    if (const char* f = getenv("SMMC_TC_SPLIT")) want = pl.halo ? std::max(1, std::min(atoi(f), cblocks)) : 1;
    if (want > 1) {
        pl.cb_per_split = (cblocks + want - 1) / want;
        pl.splits = (cblocks + pl.cb_per_split - 1) / pl.cb_per_split;
        if (pl.splits > 1) {
            pl.persistent = 1;
            pl.mt = 1;
        }
    }
    return pl;
}

size_t tc_workspace_bytes(const smmc_geom& g) {
    const TcPlan pl = plan_tc(g);
    if (!pl.supported || pl.splits <= 1) return 0;
    const int oh = (g.h + 2 * g.p_h - g.k_h) / g.s_h + 1;
    const int ow = (g.w + 2 * g.p_w - g.k_w) / g.s_w + 1;
    return (size_t)pl.splits * g.n * g.c_o * oh * ow * sizeof(float);
}

cudaError_t launch_tc_bf16(const uint16_t* x_pad, const uint16_t* w_tc, float* y, const smmc_geom& g,
                           cudaStream_t s, const char** why, float* ws, size_t ws_bytes) {
    TcPlan pl = plan_tc(g);
    if (pl.splits > 1 && (!ws || ws_bytes < tc_workspace_bytes(g))) {
        pl.splits = 1;  // no workspace: whole K per tile
        pl.cb_per_split = (g.c_i + TC_BK - 1) / TC_BK;
    }
    if (!pl.supported) {
        *why = "bf16 tensor-core variant needs stride 1 and c_i % 8 == 0";
        return cudaErrorNotSupported;
    }
    if (!encode_fn()) {
        *why = "cuTensorMapEncodeTiled unavailable from the driver";
        return cudaErrorNotSupported;
    }
    const int oh = (g.h + 2 * g.p_h - g.k_h) / g.s_h + 1;
    const int ow = (g.w + 2 * g.p_w - g.k_w) / g.s_w + 1;
    const int hp = g.h + 2 * g.p_h, wp = g.w + 2 * g.p_w;
    const int taps = g.k_h * g.k_w;
    TcParams p{};
    p.y = y;
    p.n = g.n;
    p.co = g.c_o;
    p.oh = oh;
    p.ow = ow;
    p.ohw = oh * ow;
    p.hp = hp;
    p.wp = wp;
    p.kh = g.k_h;
    p.kw = g.k_w;
    p.taps = taps;
    p.cblocks = (g.c_i + TC_BK - 1) / TC_BK;
    p.tx_b = TC_B_BYTES;
    p.splits = pl.splits;
    p.cb_per_split = pl.cb_per_split;
    p.ws = ws;
    p.y_elems = (int64_t)g.n * g.c_o * oh * ow;

    CUtensorMap tm_a, tm_b;
    {
        const cuuint64_t dims[3] = {(cuuint64_t)g.c_i, (cuuint64_t)g.c_o, (cuuint64_t)taps};
        const cuuint64_t strides[2] = {(cuuint64_t)g.c_i * 2, (cuuint64_t)g.c_o * g.c_i * 2};
        const cuuint32_t box[3] = {TC_BK, TC_BN, 1};
        if (encode(&tm_b, w_tc, 3, dims, strides, box) != CUDA_SUCCESS) {
            *why = "cuTensorMapEncodeTiled(B) failed";
            return cudaErrorInvalidValue;
        }
    }
    if (pl.halo) {
        p.halo_rows = pl.halo_rows;
        const cuuint64_t dims[2] = {(cuuint64_t)g.c_i, (cuuint64_t)g.n * hp * wp};
        const cuuint64_t strides[1] = {(cuuint64_t)g.c_i * 2};
        const cuuint32_t box[2] = {TC_BK, (cuuint32_t)pl.halo_rows};
        if (encode(&tm_a, x_pad, 2, dims, strides, box) != CUDA_SUCCESS) {
            *why = "cuTensorMapEncodeTiled(A halo) failed";
            return cudaErrorInvalidValue;
        }
        p.tx_a = (uint32_t)pl.halo_rows * TC_BK * 2;
        p.halo_stage_bytes = (int)((p.tx_a + 1023) & ~1023u);
        // N = 256 output channels per tile when c_o allows: 12 KB of smem
        // operand reads per 128-cycle MMA instead of 8 KB per 64 cycles
        const int hbn = pl.bn;
        if (hbn == 256) {
            const cuuint64_t bd[3] = {(cuuint64_t)g.c_i, (cuuint64_t)g.c_o, (cuuint64_t)taps};
            const cuuint64_t bs[2] = {(cuuint64_t)g.c_i * 2, (cuuint64_t)g.c_o * g.c_i * 2};
            const cuuint32_t bb[3] = {TC_BK, 256, 1};
            if (encode(&tm_b, w_tc, 3, bd, bs, bb) != CUDA_SUCCESS) {
                *why = "cuTensorMapEncodeTiled(B256) failed";
                return cudaErrorInvalidValue;
            }
            p.tx_b = 256 * TC_BK * 2;
        }
        if (pl.persistent) {
            constexpr int kPersistSmem = 227 * 1024 - 4096;
            const void* fns[3] = {(const void*)conv_tc_halo_persistent_kernel<256, 1>,
                                  (const void*)conv_tc_halo_persistent_kernel<128, 1>,
                                  (const void*)conv_tc_halo_persistent_kernel<128, 2>};
            for (const void* f : fns) {
                const cudaError_t attr2 = smem_optin(f, kPersistSmem);
                if (attr2 != cudaSuccess) return attr2;
            }
            const int mt = pl.mt;
            p.b_stages = std::min(PH_B_MAX, (kPersistSmem - 1024 - HALO_A_STAGES * mt * p.halo_stage_bytes) /
                                                (int)p.tx_b);
            if (p.b_stages < 2) {
                *why = "tensor-core halo tiles do not fit shared memory";
                return cudaErrorInvalidValue;
            }
            p.tiles_m = (int)((pl.tiles_m + mt - 1) / mt);
            p.tiles_n = pl.tiles_n;
            const int psmem = HALO_A_STAGES * mt * p.halo_stage_bytes + p.b_stages * (int)p.tx_b + 1024;
            int sms = 148, dev = 0;
            if (cudaGetDevice(&dev) == cudaSuccess)
                cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            const int pgrid = (int)std::min<int64_t>((int64_t)p.tiles_m * p.tiles_n * p.splits, sms);
            if (hbn == 256)
                conv_tc_halo_persistent_kernel<256, 1><<<pgrid, PH_THREADS, psmem, s>>>(tm_a, tm_b, p);
            else if (mt == 2)
                conv_tc_halo_persistent_kernel<128, 2><<<pgrid, PH_THREADS, psmem, s>>>(tm_a, tm_b, p);
            else
                conv_tc_halo_persistent_kernel<128, 1><<<pgrid, PH_THREADS, psmem, s>>>(tm_a, tm_b, p);
            if (p.splits > 1) {
                count_launches(1);
                const int64_t t4 = (p.y_elems + 3) / 4;
                const int rblocks = (int)std::min<int64_t>((t4 + 255) / 256, 148 * 8);
                tc_split_reduce_kernel<<<rblocks, 256, 0, s>>>(ws, y, p.y_elems, p.splits);
            }
        } else {
            const int smem = HALO_A_STAGES * p.halo_stage_bytes + HALO_B_STAGES * (int)p.tx_b + 1024;
            const cudaError_t attr = smem_optin(conv_tc_halo_kernel<128>, HALO_SMEM_MAX);
            if (attr != cudaSuccess) return attr;
            dim3 grid((unsigned)pl.tiles_m, (unsigned)pl.tiles_n);
            conv_tc_halo_kernel<128><<<grid, TC_THREADS, smem, s>>>(tm_a, tm_b, p);
        }
    } else {
        p.tw = pl.tw;
        p.th = pl.th;
        p.nb = pl.nb;
        p.tiles_w = (ow + pl.tw - 1) / pl.tw;
        p.tiles_h = (oh + pl.th - 1) / pl.th;
        const cuuint64_t dims[4] = {(cuuint64_t)g.c_i, (cuuint64_t)wp, (cuuint64_t)hp,
                                    (cuuint64_t)g.n};
        const cuuint64_t strides[3] = {(cuuint64_t)g.c_i * 2, (cuuint64_t)wp * g.c_i * 2,
                                       (cuuint64_t)hp * wp * g.c_i * 2};
        const cuuint32_t box[4] = {TC_BK, (cuuint32_t)pl.tw, (cuuint32_t)pl.th, (cuuint32_t)pl.nb};
        if (encode(&tm_a, x_pad, 4, dims, strides, box) != CUDA_SUCCESS) {
            *why = "cuTensorMapEncodeTiled(A box) failed";
            return cudaErrorInvalidValue;
        }
        p.tx_a = (uint32_t)(pl.tw * pl.th * pl.nb) * TC_BK * 2;
        const cudaError_t attr = smem_optin(conv_tc_box_kernel, BOX_SMEM);
        if (attr != cudaSuccess) return attr;
        dim3 grid((unsigned)pl.tiles_m, (unsigned)pl.tiles_n);
        conv_tc_box_kernel<<<grid, TC_THREADS, BOX_SMEM, s>>>(tm_a, tm_b, p);
    }
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_pack_input_nhwc(const float* x, uint16_t* out, const smmc_geom& g,
                                   cudaStream_t s, int split) {
    const int hp = g.h + 2 * g.p_h, wp = g.w + 2 * g.p_w;
    dim3 grid((wp + 63) / 64, (g.c_i + 31) / 32, g.n * hp);
    pack_input_padded_kernel<<<grid, 256, 0, s>>>(x, reinterpret_cast<__nv_bfloat16*>(out),
                                                          g.c_i, g.h, g.w, g.p_h, g.p_w, hp, wp,
                                                          split);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_pack_weights_bf16(const float* w, uint16_t* out, const smmc_geom& g,
                                     cudaStream_t s, int split) {
    const int64_t total = (int64_t)g.k_h * g.k_w * g.c_o * g.c_i;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    pack_weights_kernel<<<blocks, 256, 0, s>>>(w, reinterpret_cast<__nv_bfloat16*>(out), g.c_i,
                                               g.k_h * g.k_w, g.c_o, split);
    count_launches(1);
    return cudaGetLastError();
}

}  // namespace smmc
