// conv_ffma.cu — the product kernel: register-tiled fp32 FFMA SMM-Conv for sm_100a.
//
// The reference computes, per sample, for every (c, j) an extracted zero-packed
// slice T_j^c (smm.py:56-73), then for every kernel row k the shifted window of
// that slice times one scalar weight per output channel is accumulated into
// the whole output plane (smm.py:84-114).  Each output element therefore sees
// K = c_i*k_w*k_h scalar-times-window updates, indexed in the reference's
// (c, j, k) order by kidx = (c*k_w + j)*k_h + k — exactly the row index of the
// repacked weights W_smm viewed as a [K][c_o] matrix (smm.py:164-167).
//
// On B200 the loop nest is inverted so that the output, not the input, stays
// on chip:
//   * a CTA owns BM output pixels (flattened over n, oh, ow) x BN output
//     channels; every thread keeps an 8x8 pixel x channel tile of fp32
//     accumulators in registers for the whole K loop (no re-streaming of the
//     output plane per update, which is what bounds the CPU path);
//   * the K loop walks BK taps at a time.  The "zero-packed slice" becomes a
//     BK x BM shared-memory tile filled by predicated cp.async with zero-fill
//     (src-size 0 for padding taps) — no global scratch, no padded copy;
//   * "shifting" is index arithmetic in the loader: tap (j, k) of pixel
//     (oh, ow) reads x[c, oh*s_h + k - p_h, ow*s_w + j - p_w];
//   * the scalar weights W_smm[c, j, k, :] are rows of the [K][c_o] matrix,
//     staged by 16-byte cp.async into a BK x BN tile, and read back as
//     broadcast LDS.128;
//   * a STAGES-deep cp.async ring overlaps the loads of tap block t+STAGES-1
//     with the FFMAs of block t.
// Per k step a thread issues 4 LDS.128 and 64 FFMA.
//
// Small problems (few pixel x channel tiles) split K across CTAs; each split
// writes a full partial output plane to the workspace and a second kernel sums
// the planes in split order, so results stay run-to-run deterministic (no
// atomics).
#include <algorithm>

#include "smmc_internal.cuh"

namespace smmc {
namespace {

constexpr int kBK = 8;
constexpr int kStages = 4;

template <int BM, int BN, int THREADS, int KH, int KW, int SH, int SW>
__global__ void __launch_bounds__(THREADS, (THREADS >= 256 ? 2 : 3))
conv_ffma_kernel(const Problem p) {
    constexpr int BK = kBK;
    constexpr int STAGES = kStages;
    constexpr int TPX = BM / 8;            // pixel groups (4 + 4 pixels each)
    constexpr int TCO = BN / 8;            // channel groups (4 + 4 channels each)
    static_assert(TPX * TCO == THREADS, "thread tile must cover the CTA tile");
    static_assert(TCO % 8 == 0 && TPX % 4 == 0, "warp = 4 pixel groups x 8 channel groups");
    static_assert(THREADS % BM == 0, "loader maps one pixel column per thread");
    constexpr int KSTEP = THREADS / BM;    // taps apart for one thread's A loads
    constexpr int A_PER = BK * BM / THREADS;
    constexpr int B_CHUNKS = BK * BN / 4;  // 16-byte chunks per B tile
    static_assert(B_CHUNKS % THREADS == 0, "B loader");
    constexpr int B_PER = B_CHUNKS / THREADS;

    __shared__ __align__(16) float As[STAGES][BK][BM];
    __shared__ __align__(16) float Bs[STAGES][BK][BN];

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    constexpr int WCO = TCO / 8;
    const int cg = (warp % WCO) * 8 + (lane & 7);
    const int pg = (warp / WCO) * 4 + (lane >> 3);

    const int m0 = blockIdx.x * BM;
    const int n0 = blockIdx.y * BN;
    const int split = blockIdx.z;
    const int kbeg = split * p.k_per_split;
    const int kend = min(p.k, kbeg + p.k_per_split);
    const int ktiles = (kend - kbeg + BK - 1) / BK;

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
    const bool b_vec = (p.co & 3) == 0;

    auto load_stage = [&](int slot, int kt) {
        const int kb = kbeg + kt * BK;
        // A: zero-packed, shifted input taps (the SMM slice, built in smem)
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
            const bool ok = pvalid && kidx < kend && (unsigned)ih < (unsigned)p.h &&
                            (unsigned)iw < (unsigned)p.w_in;
            const float* src = ok ? p.x + xoff0 + (int64_t)c * p.hw + kr * p.w_in + j : p.x;
            cp_async4_zfill(smem_u32(&As[slot][kk][lp]), src, ok);
        }
        // B: scalar weights W_smm[c, j, k, n0:n0+BN] (rows of [K][c_o])
#pragma unroll
        for (int i = 0; i < B_PER; ++i) {
            const int q = tid + i * THREADS;
            const int row = q / (BN / 4);
            const int col = (q % (BN / 4)) * 4;
            const int kidx = kb + row;
            const int co = n0 + col;
            if (b_vec) {
                int bytes = (kidx < kend) ? min(max(p.co - co, 0), 4) * 4 : 0;
                const float* src = bytes ? p.w + (int64_t)kidx * p.co + co : p.w;
                cp_async16_zfill(smem_u32(&Bs[slot][row][col]), src, bytes);
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const bool ok = kidx < kend && co + e < p.co;
                    const float* src = ok ? p.w + (int64_t)kidx * p.co + co + e : p.w;
                    cp_async4_zfill(smem_u32(&Bs[slot][row][col + e]), src, ok);
                }
            }
        }
    };

    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < ktiles) load_stage(s, s);
        cp_async_commit();
    }

    for (int kt = 0; kt < ktiles; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        {
            const int nk = kt + STAGES - 1;
            if (nk < ktiles) load_stage(nk % STAGES, nk);
            cp_async_commit();
        }
        const int slot = kt % STAGES;
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            const float4 a0 = *reinterpret_cast<const float4*>(&As[slot][kk][pg * 4]);
            const float4 a1 = *reinterpret_cast<const float4*>(&As[slot][kk][BM / 2 + pg * 4]);
            const float4 b0 = *reinterpret_cast<const float4*>(&Bs[slot][kk][cg * 4]);
            const float4 b1 = *reinterpret_cast<const float4*>(&Bs[slot][kk][BN / 2 + cg * 4]);
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
    }
    cp_async_wait<0>();

    // ---- epilogue: NCHW stores (split-K: partial plane `split` of the workspace)
    float* out = p.splits > 1 ? p.ws + (int64_t)split * ((int64_t)p.m * p.co) : p.y;
    const bool vec_ok = (p.ohw & 3) == 0;
#pragma unroll
    for (int ib = 0; ib < 2; ++ib) {
        const int pbase = m0 + ib * (BM / 2) + pg * 4;
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
                    float4 v = make_float4(acc[ib * 4 + 0][j], acc[ib * 4 + 1][j],
                                           acc[ib * 4 + 2][j], acc[ib * 4 + 3][j]);
                    *reinterpret_cast<float4*>(out + ((int64_t)n * p.co + co) * p.ohw + rem) = v;
                } else {
#pragma unroll
                    for (int ii = 0; ii < 4; ++ii) {
                        const int pp = pbase + ii;
                        if (pp >= p.m) break;
                        const int nn = pp / p.ohw;
                        const int rr = pp - nn * p.ohw;
                        out[((int64_t)nn * p.co + co) * p.ohw + rr] = acc[ib * 4 + ii][j];
                    }
                }
            }
        }
    }
}

// y = sum over splits of the partial planes, in split order (deterministic).
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, float* __restrict__ y,
                                     int64_t total, int splits) {
    const int64_t total4 = total >> 2;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total4; i += stride) {
        float4 s = reinterpret_cast<const float4*>(ws)[i];
        for (int z = 1; z < splits; ++z) {
            const float4 v = reinterpret_cast<const float4*>(ws + (int64_t)z * total)[i];
            s.x += v.x;
            s.y += v.y;
            s.z += v.z;
            s.w += v.w;
        }
        reinterpret_cast<float4*>(y)[i] = s;
    }
    for (int64_t i = (total4 << 2) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += stride) {
        float s = ws[i];
        for (int z = 1; z < splits; ++z) s += ws[(int64_t)z * total + i];
        y[i] = s;
    }
}

struct TileCfg {
    int bm, bn, threads;
};
constexpr TileCfg kTiles[] = {
    {128, 128, 256},  // 0: wide channel dimension
    {128, 64, 128},   // 1: c_o <= 64
};

template <int BM, int BN, int T>
cudaError_t launch_tile(const Problem& p, int tap_kind, dim3 grid, cudaStream_t s) {
    switch (tap_kind) {
        case 1: conv_ffma_kernel<BM, BN, T, 3, 3, 1, 1><<<grid, T, 0, s>>>(p); break;
        case 2: conv_ffma_kernel<BM, BN, T, 1, 1, 1, 1><<<grid, T, 0, s>>>(p); break;
        case 3: conv_ffma_kernel<BM, BN, T, 7, 7, 2, 2><<<grid, T, 0, s>>>(p); break;
        case 4: conv_ffma_kernel<BM, BN, T, 11, 11, 4, 4><<<grid, T, 0, s>>>(p); break;
        case 5: conv_ffma_kernel<BM, BN, T, 5, 5, 1, 1><<<grid, T, 0, s>>>(p); break;
        default: conv_ffma_kernel<BM, BN, T, 0, 0, 0, 0><<<grid, T, 0, s>>>(p); break;
    }
    return cudaGetLastError();
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

FfmaPlan plan_ffma(const smmc_geom& g, int sm_count) {
    FfmaPlan pl{};
    const int oh = (g.h + 2 * g.p_h - g.k_h) / g.s_h + 1;
    const int ow = (g.w + 2 * g.p_w - g.k_w) / g.s_w + 1;
    const int64_t m = (int64_t)g.n * oh * ow;
    const int k = g.c_i * g.k_h * g.k_w;
    pl.variant = g.c_o <= 64 ? 1 : 0;
    const TileCfg t = kTiles[pl.variant];
    pl.bm = t.bm;
    pl.bn = t.bn;
    pl.bk = kBK;
    pl.threads = t.threads;
    pl.tap_kind = tap_kind_of(g);
    const int64_t tiles = ((m + t.bm - 1) / t.bm) * ((g.c_o + t.bn - 1) / t.bn);
    const int ktiles = (k + kBK - 1) / kBK;
    const int resident = t.threads >= 256 ? 2 : 3;
    const int64_t target = (int64_t)sm_count * resident;
    int splits = 1;
    if (tiles < target) {
        splits = (int)((target + tiles - 1) / tiles);
        splits = std::min(splits, std::max(1, ktiles / 4));  // >= 4 tap blocks per split
        splits = std::min(splits, 32);
    }
    int kt_per = (ktiles + splits - 1) / splits;
    pl.k_per_split = kt_per * kBK;
    pl.splits = (ktiles + kt_per - 1) / kt_per;
    return pl;
}

cudaError_t launch_ffma(const Problem& p, const FfmaPlan& pl, cudaStream_t s) {
    dim3 grid((p.m + pl.bm - 1) / pl.bm, (p.co + pl.bn - 1) / pl.bn, pl.splits);
    cudaError_t e;
    if (pl.variant == 0)
        e = launch_tile<128, 128, 256>(p, pl.tap_kind, grid, s);
    else
        e = launch_tile<128, 64, 128>(p, pl.tap_kind, grid, s);
    count_launches(1);
    return e;
}

cudaError_t launch_splitk_reduce(const Problem& p, cudaStream_t s) {
    const int64_t total = (int64_t)p.m * p.co;
    int blocks = (int)std::min<int64_t>((total / 4 + 255) / 256 + 1, 148 * 8);
    splitk_reduce_kernel<<<blocks, 256, 0, s>>>(p.ws, p.y, total, p.splits);
    count_launches(1);
    return cudaGetLastError();
}

}  // namespace smmc
