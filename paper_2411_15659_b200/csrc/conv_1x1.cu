// conv_1x1.cu — persistent FFMA kernel for 1x1 stride-1 layers (short K).
//
// With k_h = k_w = 1 the SMM update (c, 0, 0) is one scalar weight per
// output channel times the input plane of channel c (smm.py:84-114 with a
// single tap): Y[n, m, p] = sum_c W_smm[c, 0, 0, m] * X[n, c, p].  K = c_i
// is short (64-256: 4-16 blocks of 16), so in the tiled kernel every CTA
// spends as long in its prologue (first loads) and epilogue (tile stores) as
// in its K loop (timeline probe: 3.6 + 2.9 us around an 8.2 us loop on the
// ResNet-50 1x1 64->256 layer; with 4 CTAs per SM the other CTAs mostly
// cover that: measured 643 -> 637 us there, 27.8 -> 26.5 us on the config-3
// 1x1 256->64 layer).  Here a persistent CTA walks its tiles as ONE
// continuous stream of 16-deep blocks through a 4-stage cp.async ring: the
// loads of tile t+1's first blocks are in flight while tile t's last blocks
// compute and its outputs are stored.
//
// Same 8x8 FFMA2 thread tile and the same summation order as conv_ffma's
// tap-major path (channel blocks in order, k steps in order), so results are
// bitwise identical to it.  Input quads of 4 consecutive pixels of one
// channel are 16-byte cp.async copies (h*w % 4 == 0): a quarter of the
// tiled kernel's 4-byte gathers.
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "smmc_internal.cuh"

namespace smmc {
namespace {

constexpr int kBK = 16;
constexpr int kRing = 4;
// A warp = kLanePx pixel groups x kLaneCo channel groups.  8 x 4 (round 2;
// was 4 x 8): a warp's STG.128 of one channel covers 8 quads = 128 contiguous
// bytes, so a tile's 16 stores per thread are 4 full-line writes each instead
// of 8 half-line ones -- ncu had the epilogue's address math waiting on the
// stores' source registers (long-scoreboard, ~15 % of all samples on the
// ResNet-50 64->256 layer).  Both LDS.128 fragments stay <= 128 distinct bytes.
#ifndef SMMC_1X1_LANE_CO
#define SMMC_1X1_LANE_CO 4
#endif
constexpr int kLaneCo = SMMC_1X1_LANE_CO;
constexpr int kLanePx = 32 / kLaneCo;

template <int BM, int BN, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) conv1x1_persistent_kernel(const Problem p) {
    constexpr int TM = 8;
    constexpr int TPX = BM / TM, TCO = BN / 8;
    static_assert(TPX * TCO == THREADS && TCO % kLaneCo == 0 && TPX % kLanePx == 0, "thread tile");
    constexpr int WCO = TCO / kLaneCo;
    constexpr int A_CHUNKS = kBK * BM / 4;   // 16-byte chunks per A stage
    constexpr int B_CHUNKS = kBK * BN / 4;
    static_assert(A_CHUNKS % THREADS == 0 && B_CHUNKS % THREADS == 0, "loader split");
    constexpr int A_PER = A_CHUNKS / THREADS, B_PER = B_CHUNKS / THREADS;

    extern __shared__ __align__(16) float smem[];
    float* As = smem;                          // [kRing][kBK][BM]
    float* Bs = smem + kRing * kBK * BM;       // [kRing][kBK][BN]

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int cg = (warp % WCO) * kLaneCo + (lane % kLaneCo);
    const int pg = (warp / WCO) * kLanePx + (lane / kLaneCo);
    const int KT = p.c / kBK;
    const int64_t tiles = p.tiles;
    // this CTA's tiles: blockIdx.x, +gridDim.x, ...; global block q of the
    // stream = local tile index * KT + channel block
    const int my_tiles = tiles > blockIdx.x ? (int)((tiles - 1 - blockIdx.x) / gridDim.x) + 1 : 0;
    const int nq = my_tiles * KT;

    // loader state (incremental: block kb of local tile lt), per-tile
    // source pointers of this thread's A chunks and B chunks
    int ld_kb = 0, ld_lt = 0, ld_slot = 0;
    const float* a_src[A_PER];
    bool a_ok[A_PER];
    const float* b_src[B_PER];
    int b_bytes[B_PER];
    auto tile_setup = [&](int lt) {
        const int64_t tile = blockIdx.x + (int64_t)lt * gridDim.x;
        const int tm = (int)(tile / p.tiles_n);
        const int m0 = tm * BM;
        const int n0 = (int)(tile - (int64_t)tm * p.tiles_n) * BN;
#pragma unroll
        for (int i = 0; i < A_PER; ++i) {
            const int ch = tid + i * THREADS;        // chunk: row r, pixel quad
            const int r = ch / (BM / 4);
            const int pm = m0 + (ch - r * (BM / 4)) * 4;
            a_ok[i] = pm < p.m;
            const int n = a_ok[i] ? pm / p.ohw : 0;
            const int px = a_ok[i] ? pm - n * p.ohw : 0;
            a_src[i] = p.x + ((int64_t)n * p.c + r) * p.ohw + px;
        }
#pragma unroll
        for (int i = 0; i < B_PER; ++i) {
            const int ch = tid + i * THREADS;
            const int r = ch / (BN / 4);
            const int co = n0 + (ch - r * (BN / 4)) * 4;
            b_bytes[i] = min(max(p.co - co, 0), 4) * 4;
            b_src[i] = p.w + (int64_t)r * p.co + co;
        }
    };
    auto load_next = [&]() {
        if (ld_kb == 0) tile_setup(ld_lt);
        const uint32_t adst = smem_u32(As + ld_slot * kBK * BM);
        const int64_t aoff = (int64_t)ld_kb * kBK * p.ohw;
#pragma unroll
        for (int i = 0; i < A_PER; ++i) {
            const int ch = tid + i * THREADS;
            const int r = ch / (BM / 4);
            const int pq = (ch - r * (BM / 4)) * 4;
#ifdef SMMC_CHECKED
            SMMC_CHECK_SMEM(smem_u32(smem), adst + (r * BM + pq) * 4, 16);
            if (a_ok[i]) SMMC_CHECK_RANGE(a_src[i] + aoff - p.x, 4, (int64_t)p.n * p.c * p.ohw);
#endif
            cp_async16_zfill(adst + (r * BM + pq) * 4, a_ok[i] ? a_src[i] + aoff : p.x, a_ok[i] ? 16 : 0);
        }
        const uint32_t bdst = smem_u32(Bs + ld_slot * kBK * BN);
        const int64_t boff = (int64_t)ld_kb * kBK * p.co;
#pragma unroll
        for (int i = 0; i < B_PER; ++i) {
            const int ch = tid + i * THREADS;
            const int r = ch / (BN / 4);
            const int cq = (ch - r * (BN / 4)) * 4;
#ifdef SMMC_CHECKED
            SMMC_CHECK_SMEM(smem_u32(smem), bdst + (r * BN + cq) * 4, 16);
            if (b_bytes[i]) SMMC_CHECK_RANGE(b_src[i] + boff - p.w, b_bytes[i] / 4, (int64_t)p.c * p.co);
#endif
            cp_async16_zfill(bdst + (r * BN + cq) * 4, b_bytes[i] ? b_src[i] + boff : p.w, b_bytes[i]);
        }
        if (++ld_kb == KT) {
            ld_kb = 0;
            ++ld_lt;
        }
        ld_slot = ld_slot == kRing - 1 ? 0 : ld_slot + 1;
    };

#pragma unroll
    for (int s = 0; s < kRing - 1; ++s) {
        if (s < nq) load_next();
        cp_async_commit();
    }

    uint64_t acc2[TM][4];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc2[i][j] = 0ull;

#ifdef SMMC_CHECKED
    const uint32_t smem0 = smem_u32(smem);
    const int64_t x_elems = (int64_t)p.n * p.c * p.ohw, w_elems = (int64_t)p.c * p.co;
#endif
    const float* a_rd = As + pg * 4;
    const float* b_rd = Bs + cg * 4;
    int slot = 0, kb = 0, lt = 0;
    for (int q = 0; q < nq; ++q) {
        cp_async_wait<kRing - 2>();
        __syncthreads();
        if (q + kRing - 1 < nq) load_next();
        cp_async_commit();
        const float* ap = a_rd + slot * (kBK * BM);
        const float* bp = b_rd + slot * (kBK * BN);
        SMMC_CHECK_SMEM(smem0, smem_u32(ap + (kBK - 1) * BM + BM / 2), 16);
        SMMC_CHECK_SMEM(smem0, smem_u32(bp + (kBK - 1) * BN + BN / 2), 16);
#pragma unroll
        for (int kk = 0; kk < kBK; ++kk) {
            float a[TM];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const float4 v = *reinterpret_cast<const float4*>(ap + kk * BM + h * (BM / 2));
                a[4 * h + 0] = v.x;
                a[4 * h + 1] = v.y;
                a[4 * h + 2] = v.z;
                a[4 * h + 3] = v.w;
            }
            const ulonglong2 b0 = *reinterpret_cast<const ulonglong2*>(bp + kk * BN);
            const ulonglong2 b1 = *reinterpret_cast<const ulonglong2*>(bp + kk * BN + BN / 2);
            const uint64_t b[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc2[i][j] = ffma2_bcast(a[i], b[j], acc2[i][j]);
        }
        slot = slot == kRing - 1 ? 0 : slot + 1;
        if (++kb == KT) {  // last block of this tile: store it, restart
            kb = 0;
            const int64_t tile = blockIdx.x + lt * gridDim.x;
            const int tm = (int)(tile / p.tiles_n);
            const int m0 = tm * BM;
            const int n0 = (int)(tile - (int64_t)tm * p.tiles_n) * BN;
#pragma unroll
            for (int ib = 0; ib < 2; ++ib) {
                const int pbase = m0 + ib * (BM / 2) + pg * 4;
                if (pbase >= p.m) continue;
                const int n = pbase / p.ohw;
                const int rem = pbase - n * p.ohw;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int co = n0 + (j >> 2) * (BN / 2) + cg * 4 + (j & 3);
                    if (co >= p.co) continue;
                    float v[4];
#pragma unroll
                    for (int ii = 0; ii < 4; ++ii) {
                        const float2 pr = unpack2(acc2[ib * 4 + ii][j >> 1]);
                        v[ii] = (j & 1) ? pr.y : pr.x;
                    }
                    SMMC_CHECK_RANGE(((int64_t)n * p.co + co) * p.ohw + rem, 4,
                                     (int64_t)p.n * p.co * p.ohw);
                    *reinterpret_cast<float4*>(p.y + ((int64_t)n * p.co + co) * p.ohw + rem) =
                        make_float4(v[0], v[1], v[2], v[3]);
                }
            }
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc2[i][j] = 0ull;
            ++lt;
        }
    }
    cp_async_wait<0>();
}

// Weight-resident variant (round 2): the CTA's whole weight slice
// W_smm[0:K, n0:n0+BN] (K x BN floats, <= 64 KB) is staged into shared
// memory ONCE, then the CTA walks the pixel tiles of its channel slice
// (blockIdx.y) as one continuous stream of 16-deep input blocks through the
// cp.async ring -- only the input is streamed; no weight tile per block, so
// c_o = 256 runs as one 64 x 256 tile (input read once, not once per
// 128-channel tile).  Same thread tile and summation order as the other
// kernels (bitwise identical results).
template <int BM, int BN, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) conv1x1_wres_kernel(const Problem p) {
    constexpr int TM = 8;
    constexpr int TPX = BM / TM, TCO = BN / 8;
    static_assert(TPX * TCO == THREADS && TCO % kLaneCo == 0 && TPX % kLanePx == 0, "thread tile");
    constexpr int WCO = TCO / kLaneCo;
    constexpr int A_CHUNKS = kBK * BM / 4;
    static_assert(A_CHUNKS % THREADS == 0, "loader split");
    constexpr int A_PER = A_CHUNKS / THREADS;

    extern __shared__ __align__(16) float smem[];
    float* As = smem;                          // [kRing][kBK][BM]
    float* Ws = smem + kRing * kBK * BM;       // [K][BN]

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int cg = (warp % WCO) * kLaneCo + (lane % kLaneCo);
    const int pg = (warp / WCO) * kLanePx + (lane / kLaneCo);
    const int KT = p.c / kBK;
    const int n0 = blockIdx.y * BN;
    const int64_t mtiles = (p.m + BM - 1) / BM;
    const int my_tiles = mtiles > blockIdx.x ? (int)((mtiles - 1 - blockIdx.x) / gridDim.x) + 1 : 0;
    const int nq = my_tiles * KT;

    // weight slice: K rows x BN columns, 16-byte copies (c_o % 4 == 0)
    for (int i = tid; i < p.c * (BN / 4); i += THREADS) {
        const int row = i / (BN / 4), cq = (i - row * (BN / 4)) * 4;
        const int bytes = min(max(p.co - (n0 + cq), 0), 4) * 4;
        SMMC_CHECK_SMEM(smem_u32(smem), smem_u32(Ws + row * BN + cq), 16);
        if (bytes) SMMC_CHECK_RANGE((int64_t)row * p.co + n0 + cq, bytes / 4, (int64_t)p.c * p.co);
        cp_async16_zfill(smem_u32(Ws + row * BN + cq), bytes ? p.w + (int64_t)row * p.co + n0 + cq : p.w,
                         bytes);
    }
    cp_async_commit();

    int ld_kb = 0, ld_lt = 0, ld_slot = 0;
    const float* a_src[A_PER];
    bool a_ok[A_PER];
    auto tile_setup = [&](int lt) {
        const int m0 = (int)((blockIdx.x + (int64_t)lt * gridDim.x) * BM);
#pragma unroll
        for (int i = 0; i < A_PER; ++i) {
            const int ch = tid + i * THREADS;
            const int r = ch / (BM / 4);
            const int pm = m0 + (ch - r * (BM / 4)) * 4;
            a_ok[i] = pm < p.m;
            const int n = a_ok[i] ? pm / p.ohw : 0;
            const int px = a_ok[i] ? pm - n * p.ohw : 0;
            a_src[i] = p.x + ((int64_t)n * p.c + r) * p.ohw + px;
        }
    };
    auto load_next = [&]() {
        if (ld_kb == 0) tile_setup(ld_lt);
        const uint32_t adst = smem_u32(As + ld_slot * kBK * BM);
        const int64_t aoff = (int64_t)ld_kb * kBK * p.ohw;
#pragma unroll
        for (int i = 0; i < A_PER; ++i) {
            const int ch = tid + i * THREADS;
            const int r = ch / (BM / 4);
            const int pq = (ch - r * (BM / 4)) * 4;
            SMMC_CHECK_SMEM(smem_u32(smem), adst + (r * BM + pq) * 4, 16);
            if (a_ok[i]) SMMC_CHECK_RANGE(a_src[i] + aoff - p.x, 4, (int64_t)p.n * p.c * p.ohw);
            cp_async16_zfill(adst + (r * BM + pq) * 4, a_ok[i] ? a_src[i] + aoff : p.x, a_ok[i] ? 16 : 0);
        }
        if (++ld_kb == KT) {
            ld_kb = 0;
            ++ld_lt;
        }
        ld_slot = ld_slot == kRing - 1 ? 0 : ld_slot + 1;
    };

#pragma unroll
    for (int s = 0; s < kRing - 1; ++s) {
        if (s < nq) load_next();
        cp_async_commit();
    }

    uint64_t acc2[TM][4];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc2[i][j] = 0ull;

    const float* a_rd = As + pg * 4;
    const float* w_rd = Ws + cg * 4;
    int slot = 0, kb = 0, lt = 0;
    for (int q = 0; q < nq; ++q) {
        cp_async_wait<kRing - 2>();  // (the weight group is the oldest: complete first)
        __syncthreads();
        if (q + kRing - 1 < nq) load_next();
        cp_async_commit();
        const float* ap = a_rd + slot * (kBK * BM);
        const float* bp = w_rd + kb * kBK * BN;
#pragma unroll
        for (int kk = 0; kk < kBK; ++kk) {
            float a[TM];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const float4 v = *reinterpret_cast<const float4*>(ap + kk * BM + h * (BM / 2));
                a[4 * h + 0] = v.x;
                a[4 * h + 1] = v.y;
                a[4 * h + 2] = v.z;
                a[4 * h + 3] = v.w;
            }
            const ulonglong2 b0 = *reinterpret_cast<const ulonglong2*>(bp + kk * BN);
            const ulonglong2 b1 = *reinterpret_cast<const ulonglong2*>(bp + kk * BN + BN / 2);
            const uint64_t b[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc2[i][j] = ffma2_bcast(a[i], b[j], acc2[i][j]);
        }
        slot = slot == kRing - 1 ? 0 : slot + 1;
        if (++kb == KT) {  // last block of this tile: store it, restart
            kb = 0;
            const int m0 = (int)((blockIdx.x + (int64_t)lt * gridDim.x) * BM);
#pragma unroll
            for (int ib = 0; ib < 2; ++ib) {
                const int pbase = m0 + ib * (BM / 2) + pg * 4;
                if (pbase >= p.m) continue;
                const int n = pbase / p.ohw;
                const int rem = pbase - n * p.ohw;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int co = n0 + (j >> 2) * (BN / 2) + cg * 4 + (j & 3);
                    if (co >= p.co) continue;
                    float v[4];
#pragma unroll
                    for (int ii = 0; ii < 4; ++ii) {
                        const float2 pr = unpack2(acc2[ib * 4 + ii][j >> 1]);
                        v[ii] = (j & 1) ? pr.y : pr.x;
                    }
                    SMMC_CHECK_RANGE(((int64_t)n * p.co + co) * p.ohw + rem, 4,
                                     (int64_t)p.n * p.co * p.ohw);
                    *reinterpret_cast<float4*>(p.y + ((int64_t)n * p.co + co) * p.ohw + rem) =
                        make_float4(v[0], v[1], v[2], v[3]);
                }
            }
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc2[i][j] = 0ull;
            ++lt;
        }
    }
    cp_async_wait<0>();
}

// Narrow-c_o variant (round 2, last session): c_o <= 64 with a long K (the
// config-3 1x1 256->64 layer).  Tiled kernels quantise that layer's 25088
// pixels into 64- or 128-pixel CTA tiles (392 tiles = 2.65 rounds of 148 SMs,
// or 196 tiles on 296 slots) and pay a CTA barrier per 16-deep block.  Here
// the unit of work is a WARP tile of 16 pixels x 64 channels over the whole K:
// one CTA per SM takes a contiguous, balanced run of warp tiles (1568 tiles /
// 148 SMs = 10-11 warps per CTA, 96 % balance), the weight matrix
// W_smm[0:K, 0:64] is staged once per CTA, and every warp streams ITS OWN 16
// pixels of the input through a private cp.async ring -- no CTA barrier after
// the weight stage, only __syncwarp.  Thread tile 4 px x 8 c_o (a warp = 4
// pixel quads x 8 channel groups).  Each output is one fma chain over
// k = 0..K-1 in order, as in the kernels above (bitwise identical to their
// unsplit plans).  (Measured and dropped: a warp pair per tile splitting K,
// +1.2 us; an 8 x 8 thread tile with the half-warps on even / odd channels,
// same time -- the loop runs the FMA pipe at 71 % on schedulers with 3 warps
// either way.)
//
// Programmatic dependent launch: the kernel is launched with the stream-
// serialization attribute and releases its dependents at once, so the next
// grid's launch latency overlaps this grid (back-to-back launches 22.6 ->
// 21.0 us; no effect when another kernel sits between).  Measured and not
// kept: staging the weights before griddepcontrol.wait (-0.4 us, but unsafe
// when the previous kernel of the stream wrote them), and sizing for two
// co-resident CTAs (4-stage rings, 80 registers: +0.9 us).
template <int ST, int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB)
conv1x1_narrow_kernel(const Problem p, const int64_t wtiles) {
    constexpr int BN = 64, WPX = 16, STAGE = kBK * WPX;
    extern __shared__ __align__(16) float smem[];
    float* Ws = smem;                                   // [K][64]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    float* ring = smem + p.c * BN + warp * (ST * STAGE);  // this warp's [ST][16 ch][16 px]
    const int cg = lane & 7, pq = lane >> 3;
    const int KT = p.c / kBK;

    // launched with programmatic stream serialization: release the dependents at
    // once (their launch overlaps this grid), wait for the previous grid before
    // the first global read (weights or input may be its output)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int i = tid; i < p.c * (BN / 4); i += blockDim.x) {
        const int row = i / (BN / 4), cq = (i - row * (BN / 4)) * 4;
        const int bytes = min(max(p.co - cq, 0), 4) * 4;
        SMMC_CHECK_SMEM(smem_u32(smem), smem_u32(Ws + row * BN + cq), 16);
        if (bytes) SMMC_CHECK_RANGE((int64_t)row * p.co + cq, bytes / 4, (int64_t)p.c * p.co);
        cp_async16_zfill(smem_u32(Ws + row * BN + cq), bytes ? p.w + (int64_t)row * p.co + cq : p.w, bytes);
    }
    cp_async_commit();

    // this CTA's run of warp tiles, dealt round-robin to its warps
    const int64_t t0 = wtiles * blockIdx.x / gridDim.x, t1 = wtiles * (blockIdx.x + 1) / gridDim.x;
    const int mine = t1 - t0 > warp ? (int)((t1 - t0 - 1 - warp) / nwarps) + 1 : 0;
    const int nq = mine * KT;

    // loader: lane = (channel lr of 8, pixel quad lq of 4), two channels per
    // lane and block; running source pointer, one step of 16 channels per block
    const int lq = lane & 3, lr = lane >> 2;
    const int64_t kstep = (int64_t)kBK * p.ohw;
    const uint32_t ring_u32 = smem_u32(ring) + (lr * WPX + lq * 4) * 4;
    int ld_left = 0, ld_lt = 0, ld_slot = 0;
    const float* a_src = p.x;
    int a_bytes = 0;
    auto load_next = [&]() {
        if (ld_left == 0) {
            const int64_t pm = (t0 + warp + (int64_t)ld_lt * nwarps) * WPX + lq * 4;
            const bool ok = pm < p.m;
            const int n = ok ? (int)(pm / p.ohw) : 0;
            const int px = ok ? (int)(pm - (int64_t)n * p.ohw) : 0;
            a_src = p.x + ((int64_t)n * p.c + lr) * p.ohw + px;
            a_bytes = ok ? 16 : 0;
            ld_left = KT;
            ++ld_lt;
        }
        const uint32_t dst = ring_u32 + ld_slot * (STAGE * 4);
#ifdef SMMC_CHECKED
        SMMC_CHECK_SMEM(smem_u32(smem), dst + 8 * WPX * 4, 16);
        if (a_bytes) SMMC_CHECK_RANGE(a_src + 8 * (int64_t)p.ohw - p.x, 4, (int64_t)p.n * p.c * p.ohw);
#endif
        cp_async16_zfill(dst, a_src, a_bytes);
        cp_async16_zfill(dst + 8 * WPX * 4, a_src + 8 * (int64_t)p.ohw, a_bytes);
        a_src += kstep;
        --ld_left;
        ld_slot = ld_slot == ST - 1 ? 0 : ld_slot + 1;
    };
#pragma unroll
    for (int s = 0; s < ST - 1; ++s) {
        if (s < nq) load_next();
        cp_async_commit();
    }
    cp_async_wait<ST - 1>();  // the weight group is the oldest: this thread's part has landed
    __syncthreads();          // ... and everyone else's

    uint64_t acc2[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc2[i][j] = 0ull;

    const float* a_rd = ring + pq * 4;
    const float* w_rd = Ws + cg * 4;
    int slot = 0, kb = 0, lt = 0;
    for (int q = 0; q < nq; ++q) {
        cp_async_wait<ST - 2>();
        __syncwarp();
        if (q + ST - 1 < nq) load_next();
        cp_async_commit();
        const float* ap = a_rd + slot * STAGE;
        const float* bp = w_rd + kb * (kBK * BN);
        SMMC_CHECK_SMEM(smem_u32(smem), smem_u32(ap + (kBK - 1) * WPX), 16);
        SMMC_CHECK_SMEM(smem_u32(smem), smem_u32(bp + (kBK - 1) * BN + BN / 2), 16);
#pragma unroll
        for (int kk = 0; kk < kBK; ++kk) {
            const float4 v = *reinterpret_cast<const float4*>(ap + kk * WPX);
            const float a[4] = {v.x, v.y, v.z, v.w};
            const ulonglong2 b0 = *reinterpret_cast<const ulonglong2*>(bp + kk * BN);
            const ulonglong2 b1 = *reinterpret_cast<const ulonglong2*>(bp + kk * BN + BN / 2);
            const uint64_t b[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc2[i][j] = ffma2_bcast(a[i], b[j], acc2[i][j]);
        }
        slot = slot == ST - 1 ? 0 : slot + 1;
        if (++kb == KT) {  // last block of this warp tile: store it, restart
            kb = 0;
            const int64_t pm = (t0 + warp + (int64_t)lt * nwarps) * WPX + pq * 4;
            if (pm < p.m) {
                const int n = (int)(pm / p.ohw);
                const int rem = (int)(pm - (int64_t)n * p.ohw);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int co = (j >> 2) * (BN / 2) + cg * 4 + (j & 3);
                    if (co >= p.co) continue;
                    float o[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const float2 pr = unpack2(acc2[i][j >> 1]);
                        o[i] = (j & 1) ? pr.y : pr.x;
                    }
                    SMMC_CHECK_RANGE(((int64_t)n * p.co + co) * p.ohw + rem, 4,
                                     (int64_t)p.n * p.co * p.ohw);
                    *reinterpret_cast<float4*>(p.y + ((int64_t)n * p.co + co) * p.ohw + rem) =
                        make_float4(o[0], o[1], o[2], o[3]);
                }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc2[i][j] = 0ull;
            ++lt;
        }
    }
    cp_async_wait<0>();
}

int narrow_mode() {  // A/B hook: 0 = tile kernels only, 2 = warp-tile kernel whenever the channels fit
    const char* fn = getenv("SMMC_1X1_NARROW");
    return fn ? atoi(fn) : 1;
}
// Where the warp-tile kernel pays (tools/narrow_n_probe.py, B200): the CTA
// holds `per` warps, ceil(per / 4) on its fullest scheduler.  Taken when the
// schedulers are >= 80 % evenly filled (per = 4, 7, 8, 10, 11, 12: 1.02-1.20x
// the tile kernels), or with 2-3 warp tiles per SM, where CTA tiles leave most
// SMs idle (1.15-1.33x).  Not for per = 1 (no gain), 5, 6, 9 (2,2,1,1-style
// fills: 0.86-0.99x) or per > 12 (second round of tiles: 0.81-0.91x).
bool narrow_eligible(int c_i, int c_o, int64_t m, int sm_count) {
    const int mode = narrow_mode();
    if (!mode || c_o <= 32 || c_o > 64 || c_i < 64 || c_i > 384) return false;
    if (mode == 2) return true;
    const int64_t wtiles = (m + 15) / 16;
    if (wtiles < 2 * (int64_t)sm_count) return false;
    const int per = (int)((wtiles + sm_count - 1) / sm_count);
    if (per > 12) return false;
    return per <= 3 || 5 * per >= 4 * 4 * ((per + 3) / 4);
}

template <int ST, int MAXT, int MINB>
cudaError_t launch_narrow_t(const Problem& p, int grid, int warps, int smem, int64_t wtiles,
                            cudaStream_t s) {
    auto kern = conv1x1_narrow_kernel<ST, MAXT, MINB>;
    const cudaError_t attr = smem_optin(kern, 227 * 1024);
    if (attr != cudaSuccess) return attr;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(warps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = getenv("SMMC_NO_PDL") ? 0 : 1;  // A/B hook
    return cudaLaunchKernelEx(&cfg, kern, p, wtiles);
}

// One CTA per SM over balanced runs of warp tiles, a warp per tile (up to 16
// warps; longer runs are walked round-robin).
cudaError_t launch_1x1_narrow(const Problem& p, int sm_count, cudaStream_t s) {
    const int64_t wtiles = ((int64_t)p.m + 15) / 16;
    const int grid = (int)std::min<int64_t>(wtiles, sm_count);
    const int per = (int)((wtiles + grid - 1) / grid);
    const char* fwp = getenv("SMMC_1X1_NARROW_WARPS");  // A/B hook: warps per CTA
    const int warps = fwp ? std::max(1, std::min(atoi(fwp), 16)) : std::min(per, 16);
    const int fixed = p.c * 64 * (int)sizeof(float);
    const int stage = kBK * 16 * (int)sizeof(float);
    const int st = std::min(6, (227 * 1024 - fixed) / (warps * stage));
    if (st < 4) return cudaErrorInvalidConfiguration;
    const int smem = fixed + warps * st * stage;
    switch (st) {
        case 4: return launch_narrow_t<4, 512, 1>(p, grid, warps, smem, wtiles, s);
        case 5: return launch_narrow_t<5, 512, 1>(p, grid, warps, smem, wtiles, s);
        default: return launch_narrow_t<6, 512, 1>(p, grid, warps, smem, wtiles, s);
    }
}

template <int BM, int BN, int T, int MINB>
cudaError_t launch_1x1_wres(const Problem& p, int sm_count, cudaStream_t s) {
    const int smem = (kRing * kBK * BM + p.c * BN) * (int)sizeof(float);
    auto kern = conv1x1_wres_kernel<BM, BN, T, MINB>;
    const cudaError_t attr = smem_optin(kern, 227 * 1024);
    if (attr != cudaSuccess) return attr;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, T, smem) != cudaSuccess || occ < 1)
        return cudaErrorInvalidConfiguration;
    const int ntiles = (p.co + BN - 1) / BN;
    const int64_t mtiles = ((int64_t)p.m + BM - 1) / BM;
    dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(mtiles, (int64_t)sm_count * occ / ntiles)),
              (unsigned)ntiles);
    kern<<<grid, T, smem, s>>>(p);
    return cudaGetLastError();
}

template <int BM, int BN, int T, int MINB>
cudaError_t launch_1x1(const Problem& p, int sm_count, cudaStream_t s) {
    constexpr int smem = kRing * kBK * (BM + BN) * (int)sizeof(float);
    auto kern = conv1x1_persistent_kernel<BM, BN, T, MINB>;
    const cudaError_t attr = smem_optin(kern, smem);
    if (attr != cudaSuccess) return attr;
    const int grid = (int)std::min<int64_t>(p.tiles, (int64_t)sm_count * MINB);
    kern<<<grid, T, smem, s>>>(p);
    return cudaGetLastError();
}

}  // namespace

bool conv1x1_eligible(const smmc_geom& g) {
    return g.k_h == 1 && g.k_w == 1 && g.s_h == 1 && g.s_w == 1 && g.p_h == 0 && g.p_w == 0 &&
           (g.c_i % kBK) == 0 && ((g.h * g.w) & 3) == 0 && (g.c_o & 3) == 0;
}

const char* conv1x1_describe(const smmc_geom& g, int sm_count) {
    return narrow_eligible(g.c_i, g.c_o, (int64_t)g.n * g.h * g.w, sm_count)
               ? ", persistent 1x1 warp-tile stream (16 px x 64 c_o per warp, weights resident, "
                 "per-warp 16-byte cp.async rings, one CTA per SM)"
               : ", persistent 1x1 block stream (16-byte loads)";
}

// bn = 64 (128 x 64 tiles) for c_o <= 64, else 64 x 128 tiles; 4 CTAs per SM.
// (64 x 256 tiles, 256 threads, 2 CTAs/SM — the input read once instead of
// twice for c_o = 256 — measured 2x slower on the 64->256 layer, dropped.)
cudaError_t launch_conv1x1(const Problem& p, int bn, int sm_count, cudaStream_t s) {
    cudaError_t e;
    const char* f = getenv("SMMC_1X1_WRES");  // A/B hook: 0 = streamed-weight kernel
    const bool wres_ok = (!f || atoi(f) != 0) && p.c <= 256;
    if (narrow_eligible(p.c, p.co, p.m, sm_count))
        e = launch_1x1_narrow(p, sm_count, s);
    else if (wres_ok && p.co > 128 && p.c * 256 * (int)sizeof(float) <= 96 * 1024)
        e = launch_1x1_wres<64, 256, 256, 2>(p, sm_count, s);
    else if (wres_ok && p.co <= 64 && p.c * 64 * (int)sizeof(float) <= 96 * 1024)
        e = launch_1x1_wres<128, 64, 128, 2>(p, sm_count, s);
    else
        e = bn == 64 ? launch_1x1<128, 64, 128, 4>(p, sm_count, s)
                     : launch_1x1<64, 128, 128, 4>(p, sm_count, s);
    count_launches(1);
    return e;
}

}  // namespace smmc
