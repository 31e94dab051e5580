// conv_ffma.cu — the product kernel: register-tiled fp32 FFMA SMM-Conv for sm_100a.
//
// The reference computes, per sample, for every (c, j) an extracted zero-packed
// slice T_j^c (smm.py:56-73), then for every kernel row k the shifted window of
// that slice times one scalar weight per output channel is accumulated into
// the whole output plane (smm.py:84-114).  Each output element therefore sees
// K = c_i*k_w*k_h scalar-times-window updates; the weight of update (c, j, k)
// for channel m is W_smm[c, j, k, m] (smm.py:164-167).
//
// On B200 the loop nest is inverted so that the output, not the input, stays
// on chip:
//   * a CTA owns BM output pixels (flattened over n, oh, ow) x BN output
//     channels; every thread keeps an 8x8 pixel x channel tile of fp32
//     accumulators in registers for the whole K loop (no re-streaming of the
//     output plane per update, which is what bounds the CPU path);
//   * the K loop walks BK updates at a time.  The zero-packed slice becomes a
//     BK x BM shared-memory tile filled by predicated cp.async with zero-fill
//     (src-size 0 for padding taps) — no global scratch, no padded copy;
//   * "shifting" is index arithmetic in the loader: tap (j, k) of pixel
//     (oh, ow) reads x[c, oh*s_h + k - p_h, ow*s_w + j - p_w];
//   * the scalar weights of BK updates for BN channels are rows of W_smm,
//     staged by 16-byte cp.async into a BK x BN tile and read back as
//     broadcast LDS.128;
//   * a STAGES-deep cp.async ring overlaps the loads of block t+STAGES-1 with
//     the FMAs of block t.  Per k step a thread issues 4 LDS.128 + 32 FFMA2
//     (Blackwell packed fp32 FMA: one scalar pixel value times a pair of
//     channel weights), i.e. 64 FMAs in 36 issue slots.
//
// K order.  When c_i % BK == 0 ("cvec") a BK block is one tap (j, k) x BK
// consecutive input channels: a thread's A elements in a block share one
// padding test and one running pointer (advanced by BK*h*w per block), and the
// weight rows are W_smm[c0:c0+BK, j, k, :].  Otherwise (the c_i = 3 stems) a
// block is BK consecutive updates in the reference's own (c, j, k) order.
//
// Split K (small problems; wave-quantisation-aware planner, see plan_ffma):
//   reduce_mode 1 — each split stores its partial tile to the workspace; the
//     last CTA to arrive on the tile's counter sums all partials in split
//     order 0..S-1 and writes y (used for S <= 4);
//   reduce_mode 2 — splits write partial NCHW planes and a second, fully
//     parallel kernel sums them in split order (large S, tiny M).
// Both orders are fixed, so results are bitwise run-to-run deterministic; no
// float atomics anywhere.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include <cooperative_groups.h>

#include <array>
#include <map>
#include <mutex>

#include "smmc_internal.cuh"

namespace smmc {
namespace {

constexpr int kStages = 4;
// A warp = kLanePx pixel groups x kLaneCo channel groups of 8 x 8 thread tiles.
// 8 x 4 (round 2; round 1: 4 x 8): a warp's STG.128 of one channel covers 8
// pixel quads = one full 128-byte line (was two half lines), the A fragment
// LDS.128 reads 128 contiguous bytes and the B fragment 4 broadcast quads.
#ifndef SMMC_LANE_CO
#define SMMC_LANE_CO 4
#endif
constexpr int kLaneCo = SMMC_LANE_CO;
constexpr int kLanePx = 32 / kLaneCo;

#ifdef SMMC_PROBE_TL
// Timing probe (A/B builds only, -DSMMC_PROBE_TL=1): per-CTA globaltimer
// stamps [entry, first stage landed, K loop done, exit, smid, warp groups
// summed, split barrier passed (mode 5), -] for
// tools/timeline_probe.py.
__device__ unsigned long long g_tl[16384 * 8];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define TL_STAMP(slot, val)                                                                   \
    do {                                                                                      \
        const unsigned bid_ = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z); \
        if (threadIdx.x == 0 && bid_ < 16384) g_tl[bid_ * 8 + (slot)] = (val);                \
    } while (0)
#else
#define TL_STAMP(slot, val) \
    do {                    \
    } while (0)
#endif

// G > 1 (warp-group split-K, small problems): the CTA runs G groups of
// THREADS threads on the same tile, group g over the g-th 1/G of the CTA's
// tap blocks with its own cp.async ring and named barrier; at the end the
// groups' partial tiles are summed in group order through shared memory
// (deterministic) and group 0 carries on with the split-K epilogue.  More
// warps per SM without more global partials or a second reduction level.
// 64x64 warp-group tiles (the N = 1 plans) run a 3-stage ring per group and
// are register-capped for 2 CTAs per SM, so the next launch's CTAs fit beside
// a running grid (programmatic dependent launch, reduce mode 5).
template <int BM, int BN, int G>
constexpr int ring_stages() {
    return (BM == 64 && BN == 64 && G > 1) ? 3 : kStages;
}
template <int BM, int BN, int THREADS, int G, int MINB>
constexpr int min_blocks() {
    return G > 1 ? ((BM == 64 && BN == 64 && THREADS * G <= 256) ? 2 : 1) : (BN == 32 ? 8 : MINB);
}

template <int BM, int BN, int THREADS, int MINB, int TM, int BK, int KH, int KW, int SH, int SW,
          bool CVEC, bool SK, int G = 1>
__global__ void __launch_bounds__(THREADS * G, (min_blocks<BM, BN, THREADS, G, MINB>()))
    conv_ffma_kernel(const Problem p) {
    constexpr int STAGES = ring_stages<BM, BN, G>();
    constexpr int NQ = TM / 4;             // 4-pixel blocks per thread, BM/NQ apart
    constexpr int TPX = BM / TM;           // pixel groups
    constexpr int TCO = BN / 8;            // channel groups (4 + 4 channels each)
    static_assert(TPX * TCO == THREADS, "thread tile must cover the CTA tile");
    static_assert(TCO % kLaneCo == 0 && TPX % kLanePx == 0, "warp = kLanePx pixel groups x kLaneCo channel groups");
    // A loader: a thread owns one pixel column of the tile and every KSTEP-th
    // k row of a block -- or, for narrow-channel tiles with fewer threads than
    // pixels (128 x 32 on 64 threads), PXC pixel columns and every k row.
    constexpr int PXC = BM > THREADS ? BM / THREADS : 1;
    static_assert(PXC == 1 ? THREADS % BM == 0 : BM % THREADS == 0, "loader maps whole pixel columns to threads");
    static_assert(PXC == 1 || CVEC, "multi-column loader: tap-major K order only");
    constexpr int KSTEP = PXC == 1 ? THREADS / BM : 1;  // k rows apart for one thread's A loads
    constexpr int A_PER = BK / KSTEP;                   // k rows per pixel column per thread
    constexpr int B_CHUNKS = BK * BN / 4;  // 16-byte chunks per B tile
    constexpr int B_PER = (B_CHUNKS + THREADS - 1) / THREADS;
    constexpr bool B_FULL = (B_CHUNKS % THREADS) == 0;
    constexpr int B_ROWS_PER_PASS = THREADS / (BN / 4);
    constexpr uint32_t AS_STAGE = BK * BM * 4;
    constexpr uint32_t BS_STAGE = BK * BN * 4;

    extern __shared__ __align__(16) float smem[];
    constexpr int RING_F = STAGES * BK * (BM + BN);  // floats per group ring
    static_assert(!(SK && G > 1), "warp-group split-K is for classic grids");
    const int grp = G > 1 ? (int)threadIdx.x / THREADS : 0;
    float* As = smem + grp * RING_F;                 // [STAGES][BK][BM]
    float* Bs = As + STAGES * BK * BM;               // [STAGES][BK][BN]
    __shared__ int s_last;
    auto group_sync = [&]() {
        if constexpr (G > 1)
            asm volatile("bar.sync %0, %1;" ::"r"(grp + 1), "r"(THREADS) : "memory");
        else
            __syncthreads();
    };

    const int tid = G > 1 ? (int)threadIdx.x - grp * THREADS : (int)threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
#ifdef SMMC_PROBE_TL
    TL_STAMP(0, gtimer());
    {
        unsigned sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        TL_STAMP(4, sm);
    }
    bool tl_first = true;
#endif
    constexpr int WCO = TCO / kLaneCo;
    const int cg = (warp % WCO) * kLaneCo + (lane % kLaneCo);
    const int pg = (warp / WCO) * kLanePx + (lane / kLaneCo);

    // ---- work decomposition.  Modes 0-2: one (tile, split) per CTA from the
    // 3-D grid.  Mode 3 (stream-K): CTA b walks iterations [b*I, (b+1)*I) of
    // the linearised (tile, tap-block) space, tile-major, so it finishes the
    // tail of one tile and starts the next; tiles cut between CTAs are summed
    // by their last arriving CTA in segment order.
    constexpr bool sk = SK;  // stream-K instantiation (reduce_mode 3)
    const int KT = p.kt_total;
    int it = sk ? blockIdx.x * p.sk_iters : 0;
    const int it_end = sk ? (int)min((int64_t)p.tiles * KT, (int64_t)it + p.sk_iters) : 0;
    for (;;) {
    int m0, n0, kt_beg, ktiles, slot, nslots;
    int64_t tile;
    if (sk) {
        tile = it / KT;
        kt_beg = it - (int)tile * KT;
        ktiles = min(KT - kt_beg, it_end - it);
        const int tm = (int)(tile / p.tiles_n);
        m0 = tm * BM;
        n0 = (int)(tile - (int64_t)tm * p.tiles_n) * BN;
        const int first = (int)((tile * KT) / p.sk_iters);
        const int last = (int)((tile * KT + KT - 1) / p.sk_iters);
        slot = blockIdx.x - first;
        nslots = last - first + 1;
    } else {
        m0 = blockIdx.x * BM;
        n0 = blockIdx.y * BN;
        tile = (int64_t)blockIdx.x * gridDim.y + blockIdx.y;
        slot = blockIdx.z;
        nslots = p.splits;
        kt_beg = slot * p.kt_per_split;
        ktiles = min(KT - kt_beg, p.kt_per_split);
        if (G > 1) {  // this group's share of the CTA's tap blocks
            const int per_g = (ktiles + G - 1) / G;
            kt_beg += grp * per_g;
            ktiles = max(0, min(ktiles - grp * per_g, per_g));
        }
    }

    const int kh = KH ? KH : p.kh;
    const int kw = KW ? KW : p.kw;
    const int sh = SH ? SH : p.sh;
    const int sw = SW ? SW : p.sw;
    const int taps = kh * kw;

    // ---- per-thread loader geometry: one fixed output pixel column
    const int lp = tid % BM;
    const int lk0 = tid / BM;
    const int pm = m0 + lp;
    const bool pvalid = pm < p.m;
    int ih0 = 0, iw0 = 0;
    int64_t xoff0 = 0;
    if (pvalid) {
        const int n = pm / p.ohw;
        const int rem = pm - n * p.ohw;
        const int oh = rem / p.ow;
        const int ow = rem - oh * p.ow;
        ih0 = oh * sh - p.ph;
        iw0 = ow * sw - p.pw;
        xoff0 = (int64_t)n * p.c * p.hw + (int64_t)ih0 * p.w_in + iw0;
    }
    // extra pixel columns of a narrow-channel tile's loader thread (PXC > 1: fewer
    // threads than pixels; column c is pixel tid + c*THREADS, every k row)
    bool xpvalid[PXC];
    int64_t xxoff0[PXC];
    int xih0[PXC], xiw0[PXC];
#pragma unroll
    for (int c = 1; c < PXC; ++c) {
        const int pmc = m0 + tid + c * THREADS;
        xpvalid[c] = pmc < p.m;
        xih0[c] = xiw0[c] = 0;
        xxoff0[c] = 0;
        if (xpvalid[c]) {
            const int n = pmc / p.ohw;
            const int rem = pmc - n * p.ohw;
            const int oh = rem / p.ow;
            const int ow = rem - oh * p.ow;
            xih0[c] = oh * sh - p.ph;
            xiw0[c] = ow * sw - p.pw;
            xxoff0[c] = (int64_t)n * p.c * p.hw + (int64_t)xih0[c] * p.w_in + xiw0[c];
        }
    }
    const float* __restrict__ xg = p.x;
    const float* __restrict__ wg = p.w;
#ifdef SMMC_CHECKED
    const int64_t x_elems = (int64_t)p.n * p.c * p.hw;
    const int64_t w_elems = (int64_t)p.k * p.co;
    const uint32_t smem0 = smem_u32(smem);
#endif
    const uint32_t as_base = smem_u32(As + lk0 * BM + lp);
    const uint32_t bs_base = smem_u32(Bs);
    const bool b_vec = (p.co & 3) == 0;

    // B chunk of this thread (first pass): row brow, columns bcol..bcol+3
    const int brow = tid / (BN / 4);
    const int bcol = (tid % (BN / 4)) * 4;
    const int bco = n0 + bcol;
    const int b_bytes = min(max(p.co - bco, 0), 4) * 4;

    // ---- cvec loader state (tap-major K order)
    uint32_t rowmask = 0, colmask = 0;
    const bool masks = kh <= 32 && kw <= 32;
    if (masks && pvalid) {
        for (int r = 0; r < kh; ++r) rowmask |= (uint32_t)((unsigned)(ih0 + r) < (unsigned)p.h) << r;
        for (int j = 0; j < kw; ++j)
            colmask |= (uint32_t)((unsigned)(iw0 + j) < (unsigned)p.w_in) << j;
    }
    uint32_t xrowmask[PXC], xcolmask[PXC];
#pragma unroll
    for (int c = 1; c < PXC; ++c) {
        xrowmask[c] = xcolmask[c] = 0;
        if (masks && xpvalid[c]) {
            for (int r = 0; r < kh; ++r)
                xrowmask[c] |= (uint32_t)((unsigned)(xih0[c] + r) < (unsigned)p.h) << r;
            for (int j = 0; j < kw; ++j)
                xcolmask[c] |= (uint32_t)((unsigned)(xiw0[c] + j) < (unsigned)p.w_in) << j;
        }
    }
    // generic path: an odometer over this thread's next update index
    // kidx = (c*kw + j)*kh + k (the reference's order) and its input offset
    // c*h*w + k*w + j, advanced by +1 update with compares instead of divisions
    int od_k = 0, od_j = 0, od_kidx = 0;
    int64_t od_off = 0;
    if (!CVEC && masks) {
        od_kidx = kt_beg * BK + lk0;
        const int c = od_kidx / taps;
        const int tap = od_kidx - c * taps;
        od_j = tap / kh;
        od_k = tap - od_j * kh;
        od_off = (int64_t)c * p.hw + od_k * p.w_in + od_j;
    }
    auto od_step = [&]() {
        ++od_kidx;
        ++od_k;
        od_off += p.w_in;
        if (od_k == kh) {
            od_k = 0;
            od_off += 1 - (int64_t)kh * p.w_in;
            if (++od_j == kw) {
                od_j = 0;
                od_off += p.hw - kw;
            }
        }
    };
    const int cblocks = p.c / BK;
    const int64_t a_blk = (int64_t)BK * p.hw;             // A pointer step per channel block
    const int64_t a_elem = (int64_t)KSTEP * p.hw;         // between one thread's A elements
    const int64_t b_blk = (int64_t)BK * taps * p.co;      // B pointer step per channel block
    const int64_t b_pass = (int64_t)B_ROWS_PER_PASS * taps * p.co;
    int ld_tap = 0, ld_cb = 0;
    bool a_ok = false;
    const float* a_ptr = xg;
    bool xa_ok[PXC];
    const float* xa_ptr[PXC];
#pragma unroll
    for (int c = 1; c < PXC; ++c) {
        xa_ok[c] = false;
        xa_ptr[c] = xg;
    }
    const float* b_ptr = wg;
    auto set_tap = [&]() {
        const int j = ld_tap / kh;
        const int kr = ld_tap - j * kh;
        a_ok = (rowmask >> kr) & (colmask >> j) & 1u;
        a_ptr = xg + xoff0 + (int64_t)(ld_cb * BK + lk0) * p.hw + kr * p.w_in + j;
#pragma unroll
        for (int c = 1; c < PXC; ++c) {
            xa_ok[c] = (xrowmask[c] >> kr) & (xcolmask[c] >> j) & 1u;
            xa_ptr[c] = xg + xxoff0[c] + (int64_t)(ld_cb * BK) * p.hw + kr * p.w_in + j;
        }
        b_ptr = wg + ((int64_t)(ld_cb * BK + brow) * taps + ld_tap) * p.co + bco;
    };
    if (CVEC) {
        ld_tap = kt_beg / cblocks;
        ld_cb = kt_beg - ld_tap * cblocks;
        set_tap();
    }

    auto load_stage = [&](int slot, int kt) {
        if (CVEC) {
            const uint32_t adst = as_base + slot * AS_STAGE;
#pragma unroll
            for (int i = 0; i < A_PER; ++i) {
                SMMC_CHECK_SMEM(smem0, adst + i * KSTEP * BM * 4, 4);
                if (a_ok) SMMC_CHECK_RANGE(a_ptr + i * a_elem - xg, 1, x_elems);
                cp_async4_zfill(adst + i * KSTEP * BM * 4, a_ok ? a_ptr + i * a_elem : xg, a_ok);
            }
#pragma unroll
            for (int c = 1; c < PXC; ++c) {
#pragma unroll
                for (int i = 0; i < A_PER; ++i) {
                    SMMC_CHECK_SMEM(smem0, adst + (c * THREADS + i * BM) * 4, 4);
                    if (xa_ok[c]) SMMC_CHECK_RANGE(xa_ptr[c] + i * a_elem - xg, 1, x_elems);
                    cp_async4_zfill(adst + (c * THREADS + i * BM) * 4, xa_ok[c] ? xa_ptr[c] + i * a_elem : xg,
                                    xa_ok[c]);
                }
            }
            const uint32_t bdst = bs_base + slot * BS_STAGE + (brow * BN + bcol) * 4;
#pragma unroll
            for (int i = 0; i < B_PER; ++i) {
                if (!B_FULL && tid + i * THREADS >= B_CHUNKS) break;
                const uint32_t dst = bdst + i * B_ROWS_PER_PASS * BN * 4;
                const float* src = b_ptr + i * b_pass;
                SMMC_CHECK_SMEM(smem0, dst, 16);
                if (b_bytes) SMMC_CHECK_RANGE(src - wg, b_bytes / 4, w_elems);
                if (b_vec) {
                    cp_async16_zfill(dst, b_bytes ? src : wg, b_bytes);
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const bool okb = bco + e < p.co;
                        cp_async4_zfill(dst + e * 4, okb ? src + e : wg, okb);
                    }
                }
            }
            if (++ld_cb == cblocks) {
                ld_cb = 0;
                ++ld_tap;
                if (ld_tap < taps) set_tap();
            } else {
                a_ptr += a_blk;
#pragma unroll
                for (int c = 1; c < PXC; ++c) xa_ptr[c] += a_blk;
                b_ptr += b_blk;
            }
        } else {
            // reference (c, j, k) order: kidx = (c*kw + j)*kh + k
            const int kb = (kt_beg + kt) * BK;
            if (masks) {
#pragma unroll
                for (int i = 0; i < A_PER; ++i) {
                    const bool ok = pvalid && od_kidx < p.k && ((rowmask >> od_k) & (colmask >> od_j) & 1u);
                    SMMC_CHECK_SMEM(smem0, as_base + slot * AS_STAGE + i * KSTEP * BM * 4, 4);
                    if (ok) SMMC_CHECK_RANGE(xoff0 + od_off, 1, x_elems);
                    cp_async4_zfill(as_base + slot * AS_STAGE + i * KSTEP * BM * 4,
                                    ok ? xg + xoff0 + od_off : xg, ok);
#pragma unroll
                    for (int st = 0; st < KSTEP; ++st) od_step();
                }
            } else {
#pragma unroll
            for (int i = 0; i < A_PER; ++i) {
                const int kk = lk0 + i * KSTEP;
                const int kidx = kb + kk;
                const int c = kidx / taps;
                const int tap = kidx - c * taps;
                const int j = tap / kh;
                const int kr = tap - j * kh;
                const int ih = ih0 + kr;
                const int iw = iw0 + j;
                const bool ok = pvalid && kidx < p.k && (unsigned)ih < (unsigned)p.h &&
                                (unsigned)iw < (unsigned)p.w_in;
                const float* src = ok ? xg + xoff0 + (int64_t)c * p.hw + kr * p.w_in + j : xg;
                if (ok) SMMC_CHECK_RANGE(src - xg, 1, x_elems);
                cp_async4_zfill(as_base + slot * AS_STAGE + i * KSTEP * BM * 4, src, ok);
            }
            }
#pragma unroll
            for (int i = 0; i < B_PER; ++i) {
                const int q = tid + i * THREADS;
                if (!B_FULL && q >= B_CHUNKS) break;
                const int row = q / (BN / 4);
                const int col = (q % (BN / 4)) * 4;
                const int kidx = kb + row;
                const int co = n0 + col;
                const uint32_t dst = bs_base + slot * BS_STAGE + (row * BN + col) * 4;
                SMMC_CHECK_SMEM(smem0, dst, 16);
                if (b_vec) {
                    const int bytes = (kidx < p.k) ? min(max(p.co - co, 0), 4) * 4 : 0;
                    if (bytes) SMMC_CHECK_RANGE((int64_t)kidx * p.co + co, bytes / 4, w_elems);
                    cp_async16_zfill(dst, bytes ? wg + (int64_t)kidx * p.co + co : wg, bytes);
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const bool okb = kidx < p.k && co + e < p.co;
                        cp_async4_zfill(dst + e * 4, okb ? wg + (int64_t)kidx * p.co + co + e : wg,
                                        okb);
                    }
                }
            }
        }
    };

    // accumulators as FFMA2 lane pairs: acc2[i][jp] = (channel 2jp, 2jp+1) of pixel i
    uint64_t acc2[TM][4];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc2[i][j] = 0ull;

    TL_STAMP(7, gtimer());
    // mode 5 grids are launched with programmatic stream serialization: the
    // launch and the setup above overlap the previous grid's tail; wait for
    // its completion (and memory) before the first global read
    if (!sk && p.reduce_mode == 5) asm volatile("griddepcontrol.wait;" ::: "memory");
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < ktiles) load_stage(s, s);
        cp_async_commit();
    }

    const float* a_rd = As + pg * 4;
    const float* b_rd = Bs + cg * 4;
    for (int kt = 0; kt < ktiles; ++kt) {
        cp_async_wait<STAGES - 2>();
        group_sync();
#ifdef SMMC_PROBE_TL
        if (kt == 0 && tl_first) TL_STAMP(1, gtimer());
#endif
        {
            const int nk = kt + STAGES - 1;
            if (nk < ktiles) load_stage(nk % STAGES, nk);
            cp_async_commit();
        }
        const int slot = kt % STAGES;
        const float* ap = a_rd + slot * (BK * BM);
        const float* bp = b_rd + slot * (BK * BN);
        SMMC_CHECK_SMEM(smem0, smem_u32(ap + (BK - 1) * BM + (NQ - 1) * (BM / NQ)), 16);
        SMMC_CHECK_SMEM(smem0, smem_u32(bp + (BK - 1) * BN + BN / 2), 16);
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            float a[TM];
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const float4 aq = *reinterpret_cast<const float4*>(ap + kk * BM + q * (BM / NQ));
                a[4 * q + 0] = aq.x;
                a[4 * q + 1] = aq.y;
                a[4 * q + 2] = aq.z;
                a[4 * q + 3] = aq.w;
            }
            const ulonglong2 b0 = *reinterpret_cast<const ulonglong2*>(bp + kk * BN);
            const ulonglong2 b1 = *reinterpret_cast<const ulonglong2*>(bp + kk * BN + BN / 2);
            const uint64_t b[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc2[i][j] = ffma2_bcast(a[i], b[j], acc2[i][j]);
        }
    }
    cp_async_wait<0>();
    // single-wave grid: the next grid may start its setup on freed resources
    if (!sk && p.reduce_mode == 5) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#ifdef SMMC_PROBE_TL
    if (tl_first) TL_STAMP(2, gtimer());
    tl_first = false;
#endif

    float acc[TM][8];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float2 v = unpack2(acc2[i][j]);
            acc[i][2 * j] = v.x;
            acc[i][2 * j + 1] = v.y;
        }

    // ---- warp groups: sum the G partial tiles in group order (groups >= 1
    // park theirs in the drained rings, [g-1][2*TM float4][THREADS])
    const bool lead = grp == 0;
    if constexpr (G > 1) {
        __syncthreads();  // every group is done with its ring
        float4* red = reinterpret_cast<float4*>(smem);
        if (!lead) {
#pragma unroll
            for (int g = 0; g < 2 * TM; ++g) {
                SMMC_CHECK_SMEM(smem0, smem_u32(red + ((grp - 1) * 2 * TM + g) * THREADS + tid), 16);
                red[((grp - 1) * 2 * TM + g) * THREADS + tid] =
                    make_float4(acc[g >> 1][(g & 1) * 4 + 0], acc[g >> 1][(g & 1) * 4 + 1],
                                acc[g >> 1][(g & 1) * 4 + 2], acc[g >> 1][(g & 1) * 4 + 3]);
            }
        }
        __syncthreads();
        if (lead) {
            for (int z = 1; z < G; ++z)
#pragma unroll
                for (int g = 0; g < 2 * TM; ++g) {
                    const float4 v = red[((z - 1) * 2 * TM + g) * THREADS + tid];
                    acc[g >> 1][(g & 1) * 4 + 0] += v.x;
                    acc[g >> 1][(g & 1) * 4 + 1] += v.y;
                    acc[g >> 1][(g & 1) * 4 + 2] += v.z;
                    acc[g >> 1][(g & 1) * 4 + 3] += v.w;
                }
        }
        __syncthreads();  // partials read before smem is reused below
    }
    TL_STAMP(5, gtimer());

    // ---- split-K / stream-K: deterministic last-arriver fixup
    bool store = true;
    if ((p.reduce_mode == 1 && p.splits > 1) || (sk && nslots > 1)) {
        const int stride_slots = sk ? p.sk_maxseg : p.splits;
        float* part = p.ws + (tile * stride_slots) * (BM * BN);
        // layout [slot][2*TM float4 groups][THREADS]: warp stores are contiguous
        float4* mine = reinterpret_cast<float4*>(part + (int64_t)slot * (BM * BN));
        SMMC_CHECK_RANGE(part - p.ws, (int64_t)nslots * BM * BN, p.ws_floats);
        SMMC_CHECK_RANGE(tile * 4, 4, (const char*)p.ws - (const char*)p.counters);  // counter region
        if (lead)
#pragma unroll
        for (int g = 0; g < 2 * TM; ++g)
            mine[g * THREADS + tid] = make_float4(acc[g >> 1][(g & 1) * 4 + 0], acc[g >> 1][(g & 1) * 4 + 1],
                                                  acc[g >> 1][(g & 1) * 4 + 2], acc[g >> 1][(g & 1) * 4 + 3]);
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) s_last = atomicAdd(p.counters + tile, 1) == nslots - 1;
        __syncthreads();
        store = s_last && lead;
        if (store) {
            __threadfence();
            // P_0 + P_1 + ... in slot order (own partial re-read too);
            // 8 independent loads in flight per round
            const float4* base = reinterpret_cast<const float4*>(part) + tid;
#pragma unroll
            for (int h = 0; h < TM / 4; ++h) {
                float4 s4[8];
#pragma unroll
                for (int g = 0; g < 8; ++g) s4[g] = __ldcg(base + (h * 8 + g) * THREADS);
                for (int z = 1; z < nslots; ++z) {
                    float4 v[8];
#pragma unroll
                    for (int g = 0; g < 8; ++g)
                        v[g] = __ldcg(base + (int64_t)z * (BM * BN / 4) + (h * 8 + g) * THREADS);
#pragma unroll
                    for (int g = 0; g < 8; ++g) {
                        s4[g].x += v[g].x;
                        s4[g].y += v[g].y;
                        s4[g].z += v[g].z;
                        s4[g].w += v[g].w;
                    }
                }
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    const int gg = h * 8 + g;
                    acc[gg >> 1][(gg & 1) * 4 + 0] = s4[g].x;
                    acc[gg >> 1][(gg & 1) * 4 + 1] = s4[g].y;
                    acc[gg >> 1][(gg & 1) * 4 + 2] = s4[g].z;
                    acc[gg >> 1][(gg & 1) * 4 + 3] = s4[g].w;
                }
            }
            if (tid == 0) p.counters[tile] = 0;  // re-arm for the next launch
        }
    }

    // ---- split-K inside a thread-block cluster (reduce_mode 4): the S CTAs
    // of a tile (cluster dims 1 x 1 x S) park their partial tiles in their own
    // shared memory (the drained cp.async ring), then CTA r sums slice r of
    // the tile over ranks 0..S-1 in order through distributed shared memory
    // and stores it — no workspace, no counters, no second kernel, and the
    // reduction runs on all S SMs at once (deterministic: fixed rank order).
    if (!sk && p.reduce_mode == 4) {
        cooperative_groups::cluster_group cluster = cooperative_groups::this_cluster();
        constexpr int LD = BM + 4;  // channel-major [BN][BM+4]: float4 rows, fewer conflicts
        float* part = smem;
        __syncthreads();  // every warp is done reading the ring
        if (lead)
#pragma unroll
        for (int ib = 0; ib < NQ; ++ib)
#pragma unroll
            for (int jb = 0; jb < 2; ++jb)
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const int cl = jb * (BN / 2) + cg * 4 + jj;
                    const int j = jb * 4 + jj;
                    SMMC_CHECK_SMEM(smem0, smem_u32(part + cl * LD + ib * (BM / NQ) + pg * 4), 16);
                    *reinterpret_cast<float4*>(part + cl * LD + ib * (BM / NQ) + pg * 4) =
                        make_float4(acc[ib * 4 + 0][j], acc[ib * 4 + 1][j], acc[ib * 4 + 2][j],
                                    acc[ib * 4 + 3][j]);
                }
        cluster.sync();
        const int S = (int)cluster.num_blocks();
        const int r = (int)cluster.block_rank();
        constexpr int T4 = BN * BM / 4;  // float4s per tile
        const bool vec_ok = (p.ohw & 3) == 0;
        for (int e = r * T4 / S + (int)threadIdx.x; e < (r + 1) * T4 / S; e += THREADS * G) {
            const int cl = e / (BM / 4);
            const int px = (e - cl * (BM / 4)) * 4;
            const int off = cl * LD + px;
            SMMC_CHECK_SMEM(smem0, smem_u32(part + off), 16);
            SMMC_ASSERT(S <= 8);
            // all S (<= 8) remote loads in flight, then the fixed-order sum
            float4 v[8];
#pragma unroll
            for (int z = 0; z < 8; ++z)
                if (z < S) v[z] = *reinterpret_cast<const float4*>(cluster.map_shared_rank(part, z) + off);
            float4 a4 = v[0];
#pragma unroll
            for (int z = 1; z < 8; ++z)
                if (z < S) {
                    a4.x += v[z].x;
                    a4.y += v[z].y;
                    a4.z += v[z].z;
                    a4.w += v[z].w;
                }
            const int co = n0 + cl;
            const int pbase = m0 + px;
            if (co >= p.co || pbase >= p.m) continue;
            const int n = pbase / p.ohw;
            const int rem = pbase - n * p.ohw;
            if (vec_ok && pbase + 3 < p.m) {
                SMMC_CHECK_RANGE(((int64_t)n * p.co + co) * p.ohw + rem, 4, (int64_t)p.n * p.co * p.ohw);
                *reinterpret_cast<float4*>(p.y + ((int64_t)n * p.co + co) * p.ohw + rem) = a4;
            } else {
                const float v4[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
                for (int ii = 0; ii < 4; ++ii) {
                    const int pp = pbase + ii;
                    if (pp >= p.m) break;
                    const int nn = pp / p.ohw;
                    SMMC_CHECK_RANGE(((int64_t)nn * p.co + co) * p.ohw + (pp - nn * p.ohw), 1,
                                     (int64_t)p.n * p.co * p.ohw);
                    p.y[((int64_t)nn * p.co + co) * p.ohw + (pp - nn * p.ohw)] = v4[ii];
                }
            }
        }
        cluster.sync();  // peers may still be reading this CTA's partial
        TL_STAMP(3, gtimer());
        return;
    }

    // ---- reduce_mode 5: split-K reduced inside this launch by ALL S CTAs of
    // the tile (the grid is launched cooperatively, so every CTA is resident).
    // Each split publishes its partial tile (tile-contiguous: 2*TM float4
    // groups x THREADS, group g of lead thread t = 4 pixels of one channel)
    // to the L2-resident workspace, arrives on the tile counter with a
    // release reduction and waits (acquire) for all S arrivals; then CTA s
    // sums slice s of the tile over splits 0..S-1 in order with all its
    // threads and stores it.  One launch, no serial fixup, no second kernel;
    // the last CTA to leave re-arms the two tile counters.  (Measured, N = 1
    // layers: a variant that kept the own split in registers and staged the
    // S-1 others into shared memory with cp.async on the lead threads only
    // was 2 us slower; programmatic dependent launch on these single-wave
    // grids changed nothing -- the next grid's CTAs do not fit beside them.)
    if (!sk && p.reduce_mode == 5) {
        constexpr int NG = 2 * TM;        // float4 groups per thread
        constexpr int POS = NG * THREADS;  // float4 positions per partial tile
        float4* wsq = reinterpret_cast<float4*>(p.ws) + tile * (int64_t)nslots * POS;
        auto quad = [&](int g) {
            return make_float4(acc[(g >> 3) * 4 + 0][g & 7], acc[(g >> 3) * 4 + 1][g & 7],
                               acc[(g >> 3) * 4 + 2][g & 7], acc[(g >> 3) * 4 + 3][g & 7]);
        };
        if (lead) {
            float4* dst = wsq + (int64_t)slot * POS + tid;
            SMMC_CHECK_RANGE((const float*)(dst + (NG - 1) * THREADS) - p.ws, 4, p.ws_floats);
#pragma unroll
            for (int g = 0; g < NG; ++g)
                __stcg(dst + g * THREADS, quad(g));
        }
        int* ctr = p.counters + 2 * tile;  // [arrive, depart]
        SMMC_CHECK_RANGE((const char*)(ctr + 1) - (const char*)p.counters, 4,
                         (const char*)p.ws - (const char*)p.counters);  // counter region
        __syncthreads();
        if (threadIdx.x == 0) {
            // release: this CTA's partial stores (ordered before it by the
            // barrier) are visible to whoever acquires the count
            asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(ctr) : "memory");
            int seen;
            for (;;) {
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(seen) : "l"(ctr) : "memory");
                if (seen >= nslots) break;
                __nanosleep(32);
            }
        }
        __syncthreads();
        TL_STAMP(6, gtimer());
        // every thread of the CTA: slice [q0, q1) of the tile's float4
        // positions (q = g * THREADS + t), splits summed in order 0..S-1 with
        // 8 loads in flight per round; position q is thread t's float4 g
        const int q0 = (int)((int64_t)slot * POS / nslots);
        const int q1 = (int)((int64_t)(slot + 1) * POS / nslots);
        const bool vec_ok = (p.ohw & 3) == 0;
        for (int q = q0 + (int)threadIdx.x; q < q1; q += THREADS * G) {
            const int gq = q / THREADS, t = q - gq * THREADS;
            float4 a4 = __ldcg(wsq + q);
            for (int z0 = 1; z0 < nslots; z0 += 8) {
                float4 v[8];
#pragma unroll
                for (int z = 0; z < 8; ++z)
                    if (z0 + z < nslots) v[z] = __ldcg(wsq + (int64_t)(z0 + z) * POS + q);
#pragma unroll
                for (int z = 0; z < 8; ++z)
                    if (z0 + z < nslots) {
                        a4.x += v[z].x;
                        a4.y += v[z].y;
                        a4.z += v[z].z;
                        a4.w += v[z].w;
                    }
            }
            const int tw = t >> 5, tl = t & 31;
            const int tcg = (tw % WCO) * kLaneCo + (tl % kLaneCo);
            const int tpg = (tw / WCO) * kLanePx + (tl / kLaneCo);
            const int ib = gq >> 3, j = gq & 7;
            const int co = n0 + (j >> 2) * (BN / 2) + tcg * 4 + (j & 3);
            const int pbase = m0 + ib * (BM / NQ) + tpg * 4;
            if (co >= p.co || pbase >= p.m) continue;
            const int n = pbase / p.ohw;
            const int rem = pbase - n * p.ohw;
            if (vec_ok && pbase + 3 < p.m) {
                SMMC_CHECK_RANGE(((int64_t)n * p.co + co) * p.ohw + rem, 4, (int64_t)p.n * p.co * p.ohw);
                *reinterpret_cast<float4*>(p.y + ((int64_t)n * p.co + co) * p.ohw + rem) = a4;
            } else {
                const float v4[4] = {a4.x, a4.y, a4.z, a4.w};
                int nn = n, rr = rem;
#pragma unroll
                for (int ii = 0; ii < 4; ++ii) {
                    if (pbase + ii >= p.m) break;
                    SMMC_CHECK_RANGE(((int64_t)nn * p.co + co) * p.ohw + rr, 1, (int64_t)p.n * p.co * p.ohw);
                    p.y[((int64_t)nn * p.co + co) * p.ohw + rr] = v4[ii];
                    if (++rr == p.ohw) {
                        rr = 0;
                        ++nn;
                    }
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0 && atomicAdd(ctr + 1, 1) == nslots - 1) {
            // every split has passed the arrival wait: re-arm for the next launch
            ctr[0] = 0;
            ctr[1] = 0;
        }
        TL_STAMP(3, gtimer());
        return;
    }

    // ---- reduce_mode 2: this split's partial tile, tile-contiguous
    // [tile][split][16 float4 = (pixel quad, channel)][THREADS] (coalesced, no
    // index math); splitk_reduce_kernel sums the splits in order and places
    // the result (NCHW, gather replicas) — also with a single split when the
    // output goes to gather replicas
    if (!sk && p.reduce_mode == 2) {
        if (lead) {
            float4* dst =
                reinterpret_cast<float4*>(p.ws) + ((tile * p.splits + slot) * (2 * TM)) * THREADS + tid;
            SMMC_CHECK_RANGE((const float*)(dst + (2 * TM - 1) * THREADS) - p.ws, 4, p.ws_floats);
#pragma unroll
            for (int ib = 0; ib < NQ; ++ib)
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    dst[(ib * 8 + j) * THREADS] = make_float4(acc[ib * 4 + 0][j], acc[ib * 4 + 1][j],
                                                              acc[ib * 4 + 2][j], acc[ib * 4 + 3][j]);
        }
        TL_STAMP(3, gtimer());
        return;
    }

    // ---- epilogue: NCHW stores
    float* out = p.y;
    const bool vec_ok = (p.ohw & 3) == 0;
#pragma unroll
    for (int ib = 0; ib < NQ && store && lead; ++ib) {
        const int pbase = m0 + ib * (BM / NQ) + pg * 4;
        if (pbase >= p.m) continue;
        const int n = pbase / p.ohw;
        const int rem = pbase - n * p.ohw;
        const bool full4 = vec_ok && (pbase + 3 < p.m);  // same sample when ohw % 4 == 0
#pragma unroll
        for (int jb = 0; jb < 2; ++jb) {
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                const int co = n0 + jb * (BN / 2) + cg * 4 + jj;
                if (co >= p.co) continue;
                const int j = jb * 4 + jj;
                if (full4) {
                    SMMC_CHECK_RANGE(((int64_t)n * p.co + co) * p.ohw + rem, 4, (int64_t)p.n * p.co * p.ohw);
                    float4 v = make_float4(acc[ib * 4 + 0][j], acc[ib * 4 + 1][j],
                                           acc[ib * 4 + 2][j], acc[ib * 4 + 3][j]);
                    *reinterpret_cast<float4*>(out + ((int64_t)n * p.co + co) * p.ohw + rem) = v;
                } else {  // quad may cross a sample boundary (ohw % 4 != 0)
                    int nn = n, rr = rem;
#pragma unroll
                    for (int ii = 0; ii < 4; ++ii) {
                        if (pbase + ii >= p.m) break;
                        SMMC_CHECK_RANGE(((int64_t)nn * p.co + co) * p.ohw + rr, 1, (int64_t)p.n * p.co * p.ohw);
                        out[((int64_t)nn * p.co + co) * p.ohw + rr] = acc[ib * 4 + ii][j];
                        if (++rr == p.ohw) {
                            rr = 0;
                            ++nn;
                        }
                    }
                }
            }
        }
    }
    if (!sk) break;
    it += ktiles;
    if (it >= it_end) break;
    __syncthreads();  // smem ring and s_last are reused by the next segment
    }  // segment loop
    TL_STAMP(3, gtimer());
}

// reduce_modes 1 and 3: the per-tile arrival counters must read zero at
// kernel start.  An SM kernel rather than cudaMemsetAsync: the host entry's
// copy engines are busy with the H2D/D2H pipeline, and a memset queued behind
// them delayed every conv by 15-50 us (CUPTI timeline, tools/e2e_timeline.py).
__global__ void __launch_bounds__(256) zero_counters_kernel(int* __restrict__ c, int n) {
    // (the checked build validates the counter range on the host, conv_device_placed)
    for (int i = blockIdx.x * 256 + threadIdx.x; i < n; i += gridDim.x * 256) c[i] = 0;
}

// reduce_mode 2: y = sum over splits (in split order) of the partial tiles
// written by the conv epilogue ([tile][split][16][threads] float4s, each 4
// consecutive pixels of one channel), placed into NCHW (and into every
// replica of the fused c_o-shard gather).  One thread per float4 position
// with all of its split loads in flight (one memory round trip).
struct ReduceOut {
    float* ys[kMaxOut];
    int n_out, co, co_total, co_base, ohw;
    int m, bm, bn, threads, wco, tiles_n;
    int nq;  // pixel quads per thread (float4 groups per thread = 8 * nq)
    int vec;  // every replica 16-byte aligned and ohw % 4 == 0 (float4 stores)
    int64_t ws_floats, y_elems;  // bounds of the checked build
};

constexpr int kMaxSplits = 32;

__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float* __restrict__ ws,
                                                            const ReduceOut ro, int64_t positions,
                                                            int splits) {
    const float4* w4 = reinterpret_cast<const float4*>(ws);
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < positions;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int t = (int)(q % ro.threads);
        const int64_t r = q / ro.threads;
        const int ng = 8 * ro.nq;
        const int64_t tile = r / ng;
        const int g = (int)(r - tile * ng);
        // (thread, g) -> pixel quad and channel, as in the conv epilogue
        const int warp = t >> 5, lane = t & 31;
        const int cg = (warp % ro.wco) * kLaneCo + (lane % kLaneCo);
        const int pg = (warp / ro.wco) * kLanePx + (lane / kLaneCo);
        const int ib = g >> 3, j = g & 7;
        const int tm = (int)(tile / ro.tiles_n);
        const int tn = (int)(tile - (int64_t)tm * ro.tiles_n);
        const int pbase = tm * ro.bm + ib * (ro.bm / ro.nq) + pg * 4;
        const int co = tn * ro.bn + (j >> 2) * (ro.bn / 2) + cg * 4 + (j & 3);
        if (co >= ro.co || pbase >= ro.m) continue;
        const float4* src = w4 + (tile * splits * ng + g) * ro.threads + t;
        const int64_t zstride = (int64_t)ng * ro.threads;
        SMMC_CHECK_RANGE((const float*)(src + (splits - 1) * zstride) - ws, 4, ro.ws_floats);
        SMMC_ASSERT(splits <= kMaxSplits);
        float4 v[kMaxSplits];
#pragma unroll
        for (int z = 0; z < kMaxSplits; ++z)
            if (z < splits) v[z] = __ldcg(src + z * zstride);
        float4 a = v[0];
#pragma unroll
        for (int z = 1; z < kMaxSplits; ++z)
            if (z < splits) {
                a.x += v[z].x;
                a.y += v[z].y;
                a.z += v[z].z;
                a.w += v[z].w;
            }
        const int n = pbase / ro.ohw;
        const int rem = pbase - n * ro.ohw;
        if (ro.vec && pbase + 3 < ro.m) {  // same sample: ohw % 4 == 0
            const int64_t d = ((int64_t)n * ro.co_total + ro.co_base + co) * ro.ohw + rem;
            SMMC_CHECK_RANGE(d, 4, ro.y_elems);
#pragma unroll
            for (int o = 0; o < kMaxOut; ++o)
                if (o < ro.n_out) *reinterpret_cast<float4*>(ro.ys[o] + d) = a;
        } else {
            const float av[4] = {a.x, a.y, a.z, a.w};
            int nn = n, rr = rem;
#pragma unroll
            for (int ii = 0; ii < 4; ++ii) {
                if (pbase + ii >= ro.m) break;
                const int64_t d = ((int64_t)nn * ro.co_total + ro.co_base + co) * ro.ohw + rr;
                SMMC_CHECK_RANGE(d, 1, ro.y_elems);
#pragma unroll
                for (int o = 0; o < kMaxOut; ++o)
                    if (o < ro.n_out) ro.ys[o][d] = av[ii];
                if (++rr == ro.ohw) {
                    rr = 0;
                    ++nn;
                }
            }
        }
    }
}

struct TileCfg {
    int bm, bn, threads, per_sm, tm;
    int model;  // considered by the cost model (else tuning table / forced plans only)
};
constexpr TileCfg kTiles[] = {
    {128, 128, 256, 2, 8, 1},   // 0
    {128, 64, 128, 4, 8, 1},    // 1
    {256, 64, 256, 2, 8, 1},    // 2
    {64, 128, 128, 4, 8, 1},    // 3
    {64, 64, 64, 8, 8, 0},      // 4: small problems (N = 1), with warp groups / in-kernel split reduce
    {128, 32, 64, 5, 8, 1},     // 5: c_o (mod 64) <= 32, tap-major layers only (the paper's c_o = 32
                                //    sweeps): half the padded channels of a 64-wide tile; 64 threads
                                //    load two pixel columns each
    // 4 x 8 thread tiles (64 registers, 8 CTAs/SM: latency hiding by
    // occupancy) were measured 1-13 % slower on the c_i = 3 stems and 1x1
    // layers (A/B, round 1) and are not instantiated.
    // 16 x 8 thread tiles (TM = 16, 216 registers) were measured slower on
    // every BASELINE layer (A/B, profiles/r01): more warps beat more ILP here.
};
constexpr int kNumTiles = sizeof(kTiles) / sizeof(kTiles[0]);
constexpr int kBKCvec = 16;
#ifndef SMMC_BK_GENERIC  // A/B builds
#define SMMC_BK_GENERIC 8  // 16 measured: 11x11 s4 -4 %, VGG conv1_1 +14 % (round 1)
#endif
constexpr int kBKGeneric = SMMC_BK_GENERIC;

template <int BM, int BN, int T, int MINB, int TM, int BK, int KH, int KW, int SH, int SW,
          bool CVEC, bool SK = false, int G = 1>
cudaError_t launch_one(const Problem& p, dim3 grid, cudaStream_t s) {
    if constexpr (G == 1)
        if (!SK && p.reduce_mode == 3)
            return launch_one<BM, BN, T, MINB, TM, BK, KH, KW, SH, SW, CVEC, true>(p, grid, s);
    constexpr int ring = G * ring_stages<BM, BN, G>() * BK * (BM + BN) * (int)sizeof(float);
    constexpr int part = BN * (BM + 4) * (int)sizeof(float);  // reduce_mode 4 partial tile
    constexpr int smem_max = ring > part ? ring : part;
    auto kern = conv_ffma_kernel<BM, BN, T, MINB, TM, BK, KH, KW, SH, SW, CVEC, SK, G>;
    const cudaError_t attr_err = smem_optin(kern, smem_max);
    if (attr_err != cudaSuccess) return attr_err;
    if (!SK && p.reduce_mode == 5) {  // every CTA must be resident: cooperative launch
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(T * G);
        cfg.dynamicSmemBytes = ring;
        cfg.stream = s;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = getenv("SMMC_NO_PDL") ? 1 : 2;  // A/B hook
        return cudaLaunchKernelEx(&cfg, kern, p);
    }
    if (!SK && p.reduce_mode == 4) {  // the S splits of a tile form one cluster
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(T * G);
        cfg.dynamicSmemBytes = smem_max;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 1;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = grid.z;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kern, p);
    }
    kern<<<grid, T * G, ring, s>>>(p);
    return cudaGetLastError();
}

// warp-group split-K instantiations (3x3 stride-1 and generic tap-major)
template <int BM, int BN, int T, int G>
cudaError_t launch_tile_groups(const Problem& p, int tap_kind, dim3 grid, cudaStream_t s) {
    constexpr int C = kBKCvec;
    if (tap_kind == 1) return launch_one<BM, BN, T, 1, 8, C, 3, 3, 1, 1, true, false, G>(p, grid, s);
    return launch_one<BM, BN, T, 1, 8, C, 0, 0, 0, 0, true, false, G>(p, grid, s);
}

template <int BM, int BN, int T, int MINB, int TM = 8>
cudaError_t launch_tile(const Problem& p, int tap_kind, bool cvec, dim3 grid, cudaStream_t s) {
    constexpr int C = kBKCvec, G = kBKGeneric;
    if (cvec) {
        switch (tap_kind) {
            case 1: return launch_one<BM, BN, T, MINB, TM, C, 3, 3, 1, 1, true>(p, grid, s);
            case 2: return launch_one<BM, BN, T, MINB, TM, C, 1, 1, 1, 1, true>(p, grid, s);
            case 5: return launch_one<BM, BN, T, MINB, TM, C, 5, 5, 1, 1, true>(p, grid, s);
            default: return launch_one<BM, BN, T, MINB, TM, C, 0, 0, 0, 0, true>(p, grid, s);
        }
    }
    switch (tap_kind) {
        case 1: return launch_one<BM, BN, T, MINB, TM, G, 3, 3, 1, 1, false>(p, grid, s);
        case 3: return launch_one<BM, BN, T, MINB, TM, G, 7, 7, 2, 2, false>(p, grid, s);
        case 4: return launch_one<BM, BN, T, MINB, TM, G, 11, 11, 4, 4, false>(p, grid, s);
        default: return launch_one<BM, BN, T, MINB, TM, G, 0, 0, 0, 0, false>(p, grid, s);
    }
}

int tap_kind_of(const smmc_geom& g) {
    if (g.k_h == 3 && g.k_w == 3 && g.s_h == 1 && g.s_w == 1) return 1;
    if (g.k_h == 1 && g.k_w == 1 && g.s_h == 1 && g.s_w == 1) return 2;
    if (g.k_h == 7 && g.k_w == 7 && g.s_h == 2 && g.s_w == 2) return 3;
    if (g.k_h == 11 && g.k_w == 11 && g.s_h == 4 && g.s_w == 4) return 4;
    if (g.k_h == 5 && g.k_w == 5 && g.s_h == 1 && g.s_w == 1) return 5;
    return 0;
}

}  // namespace

// Measured-best (tile variant, splits) for the BASELINE.json layer shapes on
// B200 (tools/plan_table_sweep.py; profiles/r01/plan_sweep.json).  splits = 0
// selects stream-K.  Shapes not listed use the cost model below.
struct TunedPlan {
    int n, c_i, h, w, c_o, k, s, p;
    int variant, splits;
    int groups = 1;
    int reduce = 0;  // 0: by split count (last arriver / reduce kernel / cluster); 5: in-kernel
};
void set_workspace_layout(FfmaPlan& b);
constexpr TunedPlan kTuned[] = {
    // N=1: 64x64 tiles, warp-group split-K inside the CTA (third field:
    // groups) and split-K across CTAs reduced in-kernel (fourth field 5) or
    // in a cluster (splits <= 8); 20 back-to-back launches in a graph
    // (tools/n1_sweep.py, profiles/r02/n1_sweep.log; round-1 plans in brackets)
    {1, 64, 56, 56, 64, 3, 1, 1, 4, 3, 4, 5},   // 11.8 us (1,4,3 cluster: 12.8)
    {1, 128, 28, 28, 128, 3, 1, 1, 4, 5, 4},    // 12.1 us (1,8,2 cluster: 12.7)
    {1, 256, 14, 14, 256, 3, 1, 1, 4, 9, 4, 5}, // 12.9 us (1,16,2 reduce kernel: 14.1)
    {1, 512, 7, 7, 512, 3, 1, 1, 4, 18, 4, 5},  // 14.1 us (3,32,2 reduce kernel: 15.1)
    {32, 64, 56, 56, 64, 3, 1, 1, 2, 0},       // 160.0 us (168.0)
    {8, 96, 27, 27, 256, 5, 1, 2, 3, 4},       // 150.1 us (154.2)
    {256, 128, 28, 28, 128, 3, 1, 1, 0, 1},    // 1083.9 us (1119.4)
    {8, 512, 7, 7, 512, 3, 1, 1, 3, 5, 2, 5},  // 53.0 us (3,24 reduce kernel: 56.4; model 76.3)
    {64, 128, 56, 56, 256, 3, 1, 1, 3, 1},     // 2136.5 us (2154.1)
    {64, 256, 56, 56, 256, 3, 1, 1, 3, 1},     // 4206.0 us (4249.3)
    {64, 256, 28, 28, 512, 3, 1, 1, 0, 3},     // 2122.6 us (2164.0)
    {8, 3, 227, 227, 96, 11, 4, 0, 1, 1},      // 73.5 us (73.9)
#ifdef SMMC_TABLE_1X1_N8  // (A/B: the round-2 tiled plan; the warp-tile 1x1 kernel replaced it)
    {8, 256, 56, 56, 64, 1, 1, 0, 4, 1, 2},    // 25.5 us (persistent 1x1 kernel: 26.8)
#endif
};

// ---- measured plan choices (autotuner, smmc_autotune_f32)
thread_local bool tl_force_on = false;
thread_local PlanChoice tl_force{};
std::mutex g_rec_mu;
using GeomKey = std::array<int, 11>;
std::map<GeomKey, PlanChoice> g_recorded;
GeomKey geom_key(const smmc_geom& g) {
    return {g.n, g.c_i, g.h, g.w, g.c_o, g.k_h, g.k_w, g.s_h, g.s_w, g.p_h, g.p_w};
}

int64_t best_cost_waves(const FfmaPlan& b, int64_t m, int c_o, int sm_count) {
    const int per_sm = kTiles[b.variant].per_sm;
    const int64_t tiles = ((m + b.bm - 1) / b.bm) * ((c_o + b.bn - 1) / b.bn);
    const int64_t slots = (int64_t)sm_count * per_sm;
    return (tiles * std::max(b.splits, 1) + slots - 1) / slots;
}

// Wave-quantisation-aware choice of CTA tile and split-K factor.  Cost model:
// a wave of `slots` CTAs runs per_sm CTAs per SM, so its time is proportional
// to per_sm * BM * BN * (work per CTA in 8-deep tap blocks, plus a prologue /
// epilogue term and ~3 blocks of partial-tile traffic when split), with a
// small per-split overhead.
static FfmaPlan plan_ffma_impl(const smmc_geom& g, int sm_count, bool allow_stem) {  // NOLINT
    FfmaPlan best{};
    double best_cost = 1e300;
    const int oh = (g.h + 2 * g.p_h - g.k_h) / g.s_h + 1;
    const int ow = (g.w + 2 * g.p_w - g.k_w) / g.s_w + 1;
    const int64_t m = (int64_t)g.n * oh * ow;
    const int taps = g.k_h * g.k_w;
    const bool cvec = (g.c_i % kBKCvec) == 0 && g.k_h <= 32 && g.k_w <= 32;
    const int bk = cvec ? kBKCvec : kBKGeneric;
    const int kt_total = cvec ? taps * (g.c_i / bk) : (g.c_i * taps + bk - 1) / bk;
    const double blk = bk / 8.0;  // work of one tap block in 8-deep units
    // the 32-channel tile: tap-major layers whose last 64-channel tile is at most half full
    const bool narrow_ok = cvec && (g.c_o % 64) != 0 && (g.c_o % 64) <= 32 && !getenv("SMMC_NO_BN32");
    for (int v = 0; v < kNumTiles; ++v) {
        const TileCfg t = kTiles[v];
        if (!t.model || (v == 5 && !narrow_ok)) continue;
        const int64_t mt = (m + t.bm - 1) / t.bm;
        const int64_t nt = (g.c_o + t.bn - 1) / t.bn;
        const int64_t tiles = mt * nt;
        const int64_t slots = (int64_t)sm_count * t.per_sm;
        const double tile_area = (double)t.per_sm * t.bm * t.bn;
        // (a) classic grid: one (tile, split) per CTA
        const int max_s = std::max(1, std::min(32, kt_total / 2));
        for (int s = 1; s <= max_s; ++s) {
            const int per = (kt_total + s - 1) / s;
            const int sp = (kt_total + per - 1) / per;  // effective splits
            if (sp != s) continue;
            const int64_t ctas = tiles * sp;
            const int64_t waves = (ctas + slots - 1) / slots;
            const double work = per * blk + 1.0 + (sp > 1 ? 3.0 : 0.0);
            const double cost = (double)waves * tile_area * work * (1.0 + 0.02 * (sp - 1));
            if (cost < best_cost * 0.999) {
                best_cost = cost;
                best = FfmaPlan{};
                best.variant = v;
                best.bm = t.bm;
                best.bn = t.bn;
                best.threads = t.threads;
                best.splits = sp;
                best.kt_per_split = per;
                best.tiles = tiles;
                best.tiles_n = (int)nt;
                best.reduce_mode = sp > 1 ? (sp <= 4 ? 1 : 2) : 0;
            }
        }
    }
    // (b) stream-K: one persistent wave, every CTA the same number (>= 8) of tap
    // blocks, tiles cut between CTAs fixed up by the last arriver.  Only worth
    // it when the best classic grid runs <= 2 waves (quantisation loss is
    // large) and it is clearly cheaper; A/B on B200: +5-6 % on conv64@56 and
    // conv512@7 at N=32, but slower than split-K on many-wave layers.
    const int64_t best_waves = best_cost_waves(best, m, g.c_o, sm_count);
    const double classic_cost = best_cost;
    // (tap-major layers only: on the c_i = 3 stems stream-K measured 8-24 %
    // slower than the classic grid; forced plans still reach it)
    for (int v = 0; v < kNumTiles && cvec && best_waves <= 2; ++v) {
        const TileCfg t = kTiles[v];
        if (!t.model || v == 5) continue;  // (stream-K: not instantiated for the 32-channel tile)
        const int64_t nt = (g.c_o + t.bn - 1) / t.bn;
        const int64_t tiles = ((m + t.bm - 1) / t.bm) * nt;
        const int64_t slots = (int64_t)sm_count * t.per_sm;
        const int64_t W = tiles * kt_total;
        if (W >= (int64_t)INT32_MAX) continue;
        int64_t ctas = std::min<int64_t>(slots, W / 32);  // >= 32 tap blocks per CTA
        if (ctas < 1) continue;
        const int iters = (int)((W + ctas - 1) / ctas);
        ctas = (W + iters - 1) / iters;
        const double segs = (double)iters / kt_total + 1.0;  // tiles touched per CTA
        const double work = iters * blk + segs * 1.0 + 3.0;
        const double cost = (double)t.per_sm * t.bm * t.bn * work;
        if (cost < classic_cost * 0.93 && cost < best_cost) {
            best_cost = cost;
            best = FfmaPlan{};
            best.variant = v;
            best.bm = t.bm;
            best.bn = t.bn;
            best.threads = t.threads;
            best.splits = 1;
            best.kt_per_split = kt_total;
            best.tiles = tiles;
            best.tiles_n = (int)nt;
            best.reduce_mode = 3;
            best.sk_ctas = (int)ctas;
            best.sk_iters = iters;
            int maxseg = 1;
            for (int64_t tt = 0; tt < tiles; ++tt) {
                const int64_t first = (tt * kt_total) / iters;
                const int64_t last = (tt * kt_total + kt_total - 1) / iters;
                maxseg = std::max(maxseg, (int)(last - first + 1));
            }
            best.sk_maxseg = maxseg;
        }
    }
    // (c) one-wave problems (the preset networks at batch 1: 0.1-4 GFLOP): when the
    // best classic plan is a split grid of at most one wave, split-K reduced
    // IN the kernel by all split CTAs (mode 5, no second launch) on a grid of
    // about one CTA per SM with warp groups inside the CTA.  The rule follows
    // what smmc_autotune_f32 picks on those layers (profiles/r02/harness/
    // autotune_probe.log): the tile that pads M x N least at the fullest
    // single wave, 4 warp groups when a split keeps >= 12 tap blocks, else 2.
    int rule_v = -1, rule_s = 0, rule_g = 1;
    if (cvec && best.reduce_mode != 3 && best.splits > 1 && best_waves <= 1 && !conv1x1_eligible(g) &&
        !getenv("SMMC_NO_SMALL_RULE")) {  // (A/B hook)
        // the classic plan's own fill x useful area is the bar to beat (VGG conv4_x at
        // batch 1: 572 CTAs on 592 slots at 94 % useful area stays classic; 56 tiles x 2
        // in-kernel splits on 148 SMs measured 9-19 % slower)
        const TileCfg bt = kTiles[best.variant];
        const double classic_fill =
            std::min(1.0, (double)(best.tiles * best.splits) / ((double)sm_count * bt.per_sm));
        // (a classic plan of more than 4 splits also pays a second launch that re-reads
        // all S partial tiles: YOLOv3-tiny conv4/conv5 20 -> 15.5 us at equal fill)
        const double classic_score = classic_fill * (double)m * g.c_o / ((double)best.tiles * bt.bm * bt.bn) *
                                     (best.splits > 4 ? 0.8 : 1.0);
        double best_score = classic_score;
        const int order[3] = {1, 3, 4};  // 128x64, 64x128, 64x64
        for (int v : order) {
            const TileCfg t = kTiles[v];
            const int64_t tiles = ((m + t.bm - 1) / t.bm) * ((g.c_o + t.bn - 1) / t.bn);
            int64_t sp = std::min<int64_t>({(int64_t)sm_count / std::max<int64_t>(tiles, 1), 32, kt_total / 2});
            if (sp < 2) continue;
            const double fill = (double)(tiles * sp) / sm_count;
            const double useful = (double)m * g.c_o / ((double)tiles * t.bm * t.bn);
            const double score = fill * useful;
            if (score > best_score * 1.02) {
                best_score = score;
                rule_v = v;
                rule_s = (int)sp;
            }
        }
        if (rule_v >= 0) {
            const int per = (kt_total + rule_s - 1) / rule_s;
            rule_g = per >= 12 ? 4 : 2;
        }
    }
    // measured-best plans for known shapes (tuning table), then the
    // SMMC_FORCE_PLAN="variant,splits" experiment hook (splits 0 = stream-K)
    int fv = -1, fs = -1, fg = 1, fr = 0;
    if (rule_v >= 0) {
        fv = rule_v;
        fs = rule_s;
        fg = rule_g;
        fr = 5;
    }
    const bool use_table = !getenv("SMMC_NO_TABLE");  // A/B hook: cost model / 1x1 kernel only
    for (const TunedPlan& e : kTuned) {
        if (use_table && e.n == g.n && e.c_i == g.c_i && e.h == g.h && e.w == g.w && e.c_o == g.c_o &&
            e.k == g.k_h && g.k_w == g.k_h && e.s == g.s_h && g.s_w == g.s_h && e.p == g.p_h &&
            g.p_w == g.p_h) {
            fv = e.variant;
            fs = e.splits;
            fg = e.groups;
            fr = e.reduce;
        }
    }
    const bool table_hit = fv >= 0;  // a tuning-table hit also overrides the 1x1 kernel choice
    bool env_forced = false;
    if (const char* f = getenv("SMMC_FORCE_PLAN")) {  // "variant,splits[,groups[,reduce]]"
        int v = -1, sp = -1, gr = 1, rd = 0;
        if (sscanf(f, "%d,%d,%d,%d", &v, &sp, &gr, &rd) >= 2) {
            fv = v;
            fs = sp;
            fg = gr;
            fr = rd;
            env_forced = true;
        }
    }
    // a plan pinned by the autotuner for this thread, else the measured winner
    // recorded for this geometry (not for the replicated-output gather plans)
    {
        PlanChoice pc{};
        bool have = false;
        if (tl_force_on) {
            pc = tl_force;
            have = true;
        } else if (!env_forced && allow_stem) {
            have = plan_recorded(g, &pc);
        }
        if (have) {
            fv = pc.variant;
            fs = pc.splits;
            fg = pc.groups;
            fr = pc.reduce;
            env_forced = true;
            if (fv < 0) {  // "tiled kernel, cost-model plan" (no_stem only)
                fs = -1;
                allow_stem = false;
            }
        }
    }
    if ((fv == 4 || fv == 5) && (!cvec || fs == 0)) fv = -1;  // 64x64 / 128x32 tiles: tap-major split grids only
    // warp groups: tap-major blocks, classic split grid, instantiated
    // (variant, G) pairs only
    const bool groups_ok = cvec && fs > 0 &&
                           ((fg == 2 && (fv == 0 || fv == 1 || fv == 3 || fv == 4)) ||
                            ((fg == 3 || fg == 4) && (fv == 1 || fv == 3)) || (fg == 4 && fv == 4));
    if (!groups_ok) fg = 1;
    if (fv >= 0 && fv < kNumTiles && fs >= 0) {
        const TileCfg t = kTiles[fv];
        best = FfmaPlan{};
        best.variant = fv;
        best.bm = t.bm;
        best.bn = t.bn;
        best.threads = t.threads;
        best.tiles_n = (int)((g.c_o + t.bn - 1) / t.bn);
        best.tiles = ((m + t.bm - 1) / t.bm) * best.tiles_n;
        if (fs == 0) {
            const int64_t W = best.tiles * kt_total;
            int64_t ctas = std::max<int64_t>(1, std::min<int64_t>((int64_t)sm_count * t.per_sm, W / 8));
            best.sk_iters = (int)((W + ctas - 1) / ctas);
            best.sk_ctas = (int)((W + best.sk_iters - 1) / best.sk_iters);
            best.splits = 1;
            best.kt_per_split = kt_total;
            best.reduce_mode = 3;
            int maxseg = 1;
            for (int64_t tt = 0; tt < best.tiles; ++tt)
                maxseg = std::max(maxseg, (int)((tt * kt_total + kt_total - 1) / best.sk_iters -
                                                (tt * kt_total) / best.sk_iters + 1));
            best.sk_maxseg = maxseg;
        } else {
            fs = std::min(fs, kMaxSplits);
            best.kt_per_split = (kt_total + fs - 1) / fs;
            best.splits = (kt_total + best.kt_per_split - 1) / best.kt_per_split;
            best.reduce_mode = best.splits > 1 ? (best.splits <= 4 ? 1 : 2) : 0;
            if (fr == 5 && best.splits > 1) best.reduce_mode = 5;
            best.groups = fg;
        }
    }
    if (best.groups < 1) best.groups = 1;
    // split-K with 2..8 splits on an under-filled GPU (at most half the CTA
    // slots): reduce inside a thread-block cluster (reduce_mode 4) instead of
    // global partials (modes 1, 2).  On fuller grids a cluster's CTAs idle at
    // the reduction waiting for each other and co-scheduling clusters costs
    // slots (measured: conv256@14 N=32, 294 CTAs, 147 -> 211 us; conv128@28
    // N=32, 588 CTAs, 152 -> 184 us); N=1 layers gain (20.0 -> 19.1 us).
    int per_sm_best = kTiles[best.variant].per_sm;
    if (best.groups > 1) per_sm_best = 2;  // one G-group CTA per SM: allow a full wave
    if ((best.reduce_mode == 1 || best.reduce_mode == 2) && best.splits >= 2 && best.splits <= 8 &&
        2 * best.tiles * best.splits <= (int64_t)sm_count * per_sm_best) {
        const char* f = getenv("SMMC_CLUSTER_RED");  // A/B hook
        if (!f || atoi(f) != 0) best.reduce_mode = 4;
    }
    // (d) a split of more than 4 whose whole grid is co-resident (one wave at the
    // tile's design occupancy, which its launch bounds and ring size guarantee):
    // reduce in the kernel (mode 5) instead of the second launch -- same tile,
    // same splits, same summation order per output.  VGG-16 at batch 1: conv3_1
    // 53.9 -> 43.8 us, conv3_2 87.3 -> 77.8, conv4_1 53.6 -> 49.6, conv4_2 90.1 -> 86.5.
    if (best.reduce_mode == 2 && !env_forced && !table_hit && best.groups == 1 && best.variant != 5 &&
        best.tiles * best.splits <= (int64_t)sm_count * kTiles[best.variant].per_sm &&
        !getenv("SMMC_NO_INKERNEL_RULE"))  // (A/B hook)
        best.reduce_mode = 5;
    // 1x1 layers: the persistent block-stream kernel (no split, no
    // workspace); the tiled kernel with the same tile is its fallback for
    // operands that are not 16-byte aligned
    const char* f1 = getenv("SMMC_1X1");  // A/B hook: 0 = tiled kernel
    if (conv1x1_eligible(g) && (!f1 || atoi(f1) != 0) && !env_forced && !table_hit) {
        const int v = g.c_o <= 64 ? 1 : 3;  // 128x64 or 64x128
        const TileCfg t = kTiles[v];
        best = FfmaPlan{};
        best.variant = v;
        best.bm = t.bm;
        best.bn = t.bn;
        best.threads = t.threads;
        best.tiles_n = (int)((g.c_o + t.bn - 1) / t.bn);
        best.tiles = ((m + t.bm - 1) / t.bm) * best.tiles_n;
        best.splits = 1;
        best.kt_per_split = kt_total;
        best.reduce_mode = 0;
        best.groups = 1;
        best.persist1x1 = t.bn;
    }
    // c_i <= 4 stems: the direct register-window kernel (weights resident in
    // smem, no zero-packed A tiles); the tiled kernel stays the fallback for
    // the fused gather and for forced plans
    if (allow_stem && !env_forced && stem_kind(g, sm_count)) {
        const int kind = stem_kind(g, sm_count);
        best = FfmaPlan{};
        best.bm = 128;  // nominal pixels per CTA (the stem kernel tiles rows itself)
        best.bn = stem_bn(g, kind);
        best.threads = 128;
        best.tiles_n = (g.c_o + best.bn - 1) / best.bn;
        best.tiles = ((m + best.bm - 1) / best.bm) * best.tiles_n;
        best.splits = 1;
        best.kt_per_split = kt_total;
        best.reduce_mode = 0;
        best.groups = 1;
        best.stem = kind;
    }
    best.bk = bk;
    best.kt_total = kt_total;
    best.cvec = cvec ? 1 : 0;
    best.tap_kind = tap_kind_of(g);
    set_workspace_layout(best);
    return best;
}

// [counter region][partial tiles] (see kCounterRegion).
void set_workspace_layout(FfmaPlan& b) {
    b.ws_counter_offset = 0;
    b.ws_partial_offset = 0;
    b.ws_bytes = 0;
    b.zero_counters = 0;
    if (b.reduce_mode == 0 || b.reduce_mode == 4) return;
    const int slots_per_tile = b.reduce_mode == 3 ? b.sk_maxseg : b.splits;
    const size_t part = (size_t)b.tiles * slots_per_tile * b.bm * b.bn * sizeof(float);
    const size_t counters = b.reduce_mode == 2 ? 0 : (size_t)b.tiles * (b.reduce_mode == 5 ? 2 : 1) * sizeof(int);
    size_t region = kCounterRegion;
    if (counters > kCounterRegion) {  // rare: more tiles than the resident region holds
        region = (counters + 255) & ~(size_t)255;
        b.zero_counters = 1;
    }
    b.ws_partial_offset = region;
    b.ws_bytes = region + part;
}

// Plan for the fused c_o-shard gather: the product plan recast to reduce
// mode 2, so the conv kernel keeps its single-output epilogue and the (already
// needed, or one extra tiny) placement pass splitk_reduce_kernel writes the
// replicas — local and NVLink peer memory — in split order.
FfmaPlan plan_ffma(const smmc_geom& g, int sm_count) { return plan_ffma_impl(g, sm_count, true); }

void plan_force(const PlanChoice* c) {
    tl_force_on = c != nullptr;
    if (c) tl_force = *c;
}

void plan_record(const smmc_geom& g, const PlanChoice* c) {
    std::lock_guard<std::mutex> lk(g_rec_mu);
    if (c)
        g_recorded[geom_key(g)] = *c;
    else
        g_recorded.erase(geom_key(g));
}

void plan_record_clear() {
    std::lock_guard<std::mutex> lk(g_rec_mu);
    g_recorded.clear();
}

bool plan_recorded(const smmc_geom& g, PlanChoice* out) {
    std::lock_guard<std::mutex> lk(g_rec_mu);
    auto it = g_recorded.find(geom_key(g));
    if (it == g_recorded.end()) return false;
    if (out) *out = it->second;
    return true;
}

// Candidates for the autotuner: in-kernel-split grids (reduce mode 5) of the
// small tiles sized to about 0.5, 0.75, 1, 1.5 and 2 CTAs per SM with 2 or 4
// warp groups, stream-K on two tiles, classic splits of the cost model's tile,
// and the tiled kernel where the default is a stem / 1x1 kernel.
int plan_candidates(const smmc_geom& g, int sm_count, PlanChoice* out, int max_out) {
    const int oh = (g.h + 2 * g.p_h - g.k_h) / g.s_h + 1, ow = (g.w + 2 * g.p_w - g.k_w) / g.s_w + 1;
    const int64_t m = (int64_t)g.n * oh * ow;
    const bool cvec = g.c_i % kBKCvec == 0;
    const int bk = cvec ? kBKCvec : kBKGeneric;
    const int kt = (g.c_i * g.k_h * g.k_w + bk - 1) / bk;
    int n = 0;
    auto add = [&](int v, int sp, int gr, int rd, int ns) {
        for (int i = 0; i < n; ++i)
            if (out[i].variant == v && out[i].splits == sp && out[i].groups == gr && out[i].reduce == rd &&
                out[i].no_stem == ns)
                return;
        if (n < max_out) out[n++] = PlanChoice{v, sp, gr, rd, ns};
    };
    const FfmaPlan def = plan_ffma(g, sm_count);
    if (def.stem || def.persist1x1) add(-1, -1, 1, 0, 1);
    struct V { int v, bm, bn, g0, g1; };
    const V vs[] = {{3, 64, 128, 2, 2}, {4, 64, 64, 2, 4}, {1, 128, 64, 2, 4}};
    const int targets[] = {sm_count / 2, sm_count * 3 / 4, sm_count, sm_count * 3 / 2, sm_count * 2};
    for (const V& v : vs) {
        const int64_t tiles = ((m + v.bm - 1) / v.bm) * ((g.c_o + v.bn - 1) / v.bn);
        for (int t : targets) {
            const int64_t sp = t / std::max<int64_t>(tiles, 1);
            if (sp < 2 || sp > 32) continue;
            for (int gr = v.g0; gr <= v.g1; gr += 2) {
                if (!cvec) {  // generic K order: no warp groups, 64x64 tile not instantiated
                    if (v.v != 4) add(v.v, (int)sp, 1, 5, 1);
                } else if (kt / sp >= gr) {
                    add(v.v, (int)sp, gr, 5, 1);
                }
            }
        }
    }
    if (cvec) {
        add(3, 0, 1, 0, 1);
        add(1, 0, 1, 0, 1);
    }
    if (cvec && (g.c_o % 64) != 0 && (g.c_o % 64) <= 32) {  // the 128x32 tile, 2-4 CTAs per SM
        const int64_t tiles = ((m + 127) / 128) * ((g.c_o + 31) / 32);
        add(5, 1, 1, 0, 1);
        for (int t : {sm_count, sm_count * 2, sm_count * 4}) {
            const int64_t sp = t / std::max<int64_t>(tiles, 1);
            if (sp >= 2 && sp <= 32 && kt / sp >= 1) add(5, (int)sp, 1, 5, 1);
        }
    }
    return n;
}

FfmaPlan plan_ffma_gather(const smmc_geom& g, int sm_count) {
    // the gather epilogue lives in the tiled kernel: plan without the stem kernel
    FfmaPlan pl = plan_ffma_impl(g, sm_count, false);
    const int64_t m = (int64_t)g.n * ((g.h + 2 * g.p_h - g.k_h) / g.s_h + 1) *
                      ((g.w + 2 * g.p_w - g.k_w) / g.s_w + 1);
    if (pl.reduce_mode == 3) {  // stream-K -> classic split grid of similar size
        const int64_t want = std::max<int64_t>(1, pl.sk_ctas / std::max<int64_t>(1, pl.tiles));
        const int sp = (int)std::min<int64_t>(want, pl.kt_total);
        pl.kt_per_split = (pl.kt_total + sp - 1) / sp;
        pl.splits = (pl.kt_total + pl.kt_per_split - 1) / pl.kt_per_split;
        pl.sk_ctas = pl.sk_iters = pl.sk_maxseg = 0;
    }
    (void)m;
    pl.persist1x1 = 0;
    pl.reduce_mode = 2;
    set_workspace_layout(pl);
    return pl;
}

cudaError_t launch_ffma(const Problem& p, const FfmaPlan& pl, cudaStream_t s) {
    dim3 grid((p.m + pl.bm - 1) / pl.bm, (p.co + pl.bn - 1) / pl.bn, pl.splits);
    if (pl.reduce_mode == 3) grid = dim3((unsigned)pl.sk_ctas, 1, 1);
    if (pl.zero_counters && (pl.reduce_mode == 1 || pl.reduce_mode == 3 || pl.reduce_mode == 5)) {
        const int nc = (int)pl.tiles * (pl.reduce_mode == 5 ? 2 : 1);
        zero_counters_kernel<<<(int)std::min<int64_t>((nc + 255) / 256, 148), 256, 0, s>>>(p.counters, nc);
        count_launches(1);
    }
    cudaError_t e;
    if (pl.stem) {  // stem plans come from plan_ffma only (never the replicated-output gather)
        if (p.n_out != 1) return cudaErrorInvalidConfiguration;
        return launch_stem(p, pl.stem, s);
    }
    if (pl.persist1x1 && p.n_out == 1 &&
        !(((uintptr_t)p.x | (uintptr_t)p.w | (uintptr_t)p.y) & 15)) {
        int dev = 0, sms = 148;
        if (cudaGetDevice(&dev) == cudaSuccess)
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        return launch_conv1x1(p, pl.persist1x1, sms, s);
    }
    if (pl.groups > 1) {
        const int key = pl.variant * 8 + pl.groups;
        switch (key) {
            case 0 * 8 + 2: e = launch_tile_groups<128, 128, 256, 2>(p, pl.tap_kind, grid, s); break;
            case 1 * 8 + 2: e = launch_tile_groups<128, 64, 128, 2>(p, pl.tap_kind, grid, s); break;
            case 1 * 8 + 3: e = launch_tile_groups<128, 64, 128, 3>(p, pl.tap_kind, grid, s); break;
            case 3 * 8 + 3: e = launch_tile_groups<64, 128, 128, 3>(p, pl.tap_kind, grid, s); break;
            case 1 * 8 + 4: e = launch_tile_groups<128, 64, 128, 4>(p, pl.tap_kind, grid, s); break;
            case 3 * 8 + 2: e = launch_tile_groups<64, 128, 128, 2>(p, pl.tap_kind, grid, s); break;
            case 3 * 8 + 4: e = launch_tile_groups<64, 128, 128, 4>(p, pl.tap_kind, grid, s); break;
            case 4 * 8 + 2: e = launch_tile_groups<64, 64, 64, 2>(p, pl.tap_kind, grid, s); break;
            case 4 * 8 + 4: e = launch_tile_groups<64, 64, 64, 4>(p, pl.tap_kind, grid, s); break;
            default: return cudaErrorInvalidConfiguration;
        }
    } else
    switch (pl.variant) {
        case 0: e = launch_tile<128, 128, 256, 2>(p, pl.tap_kind, pl.cvec, grid, s); break;
        case 1: e = launch_tile<128, 64, 128, 4>(p, pl.tap_kind, pl.cvec, grid, s); break;
        case 2: e = launch_tile<256, 64, 256, 2>(p, pl.tap_kind, pl.cvec, grid, s); break;
        case 4: e = launch_tile_groups<64, 64, 64, 1>(p, pl.tap_kind, grid, s); break;
        case 5: e = launch_tile_groups<128, 32, 64, 1>(p, pl.tap_kind, grid, s); break;
        default: e = launch_tile<64, 128, 128, 4>(p, pl.tap_kind, pl.cvec, grid, s); break;
    }
    count_launches(1);
    if (e != cudaSuccess || pl.reduce_mode != 2) return e;
    if (p.splits > kMaxSplits) return cudaErrorInvalidConfiguration;
    const int64_t positions = pl.tiles * 2 * kTiles[pl.variant].tm * pl.threads;
    const int blocks = (int)std::min<int64_t>((positions + 255) / 256, 148 * 16);
    ReduceOut ro{};
    ro.m = p.m;
    ro.bm = pl.bm;
    ro.bn = pl.bn;
    ro.threads = pl.threads;
    ro.wco = pl.bn / (8 * kLaneCo);
    ro.nq = kTiles[pl.variant].tm / 4;
    ro.tiles_n = pl.tiles_n;
    for (int o = 0; o < p.n_out; ++o) ro.ys[o] = p.ys[o];
    ro.n_out = p.n_out;
    ro.co = p.co;
    ro.co_total = p.co_total;
    ro.co_base = p.co_base;
    ro.ohw = p.ohw;
    ro.vec = (p.ohw & 3) == 0;
    ro.ws_floats = p.ws_floats;
    ro.y_elems = (int64_t)p.n * p.co_total * p.ohw;
    for (int o = 0; o < p.n_out; ++o) ro.vec &= ((uintptr_t)p.ys[o] & 15) == 0;
    splitk_reduce_kernel<<<blocks, 256, 0, s>>>(p.ws, ro, positions, p.splits);
    count_launches(1);
    return cudaGetLastError();
}

#ifdef SMMC_PROBE_TL
extern "C" __attribute__((visibility("default"))) int smmc_probe_timeline(unsigned long long* host,
                                                                         int n) {
    if (!host) {  // clear
        static unsigned long long zeros[16384 * 8];
        return (int)cudaMemcpyToSymbol(g_tl, zeros, sizeof(zeros));
    }
    return (int)cudaMemcpyFromSymbol(host, g_tl, sizeof(unsigned long long) * 8 * std::min(n, 16384));
}
#endif

int ffma_launches(const FfmaPlan& pl) {
    if (pl.stem || pl.persist1x1) return 1;
    return (pl.reduce_mode == 2 ? 2 : 1) + (pl.zero_counters ? 1 : 0);
}

}  // namespace smmc
