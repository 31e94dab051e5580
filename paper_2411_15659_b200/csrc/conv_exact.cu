// conv_exact.cu — bitwise-reproducing SMM-Conv kernel + the slice/FMA helpers.
//
// SMMC_MODE_EXACT reproduces the reference's smm_conv_single bit for bit
// (smm.py:226-251 with _fma_channel_range, smm.py:84-114): for every output
// element the updates arrive in (c, j, k) order — input channel, kernel
// column, kernel row — each a separately rounded multiply followed by a
// separately rounded add, starting from +0.  Padded taps are skipped: in the
// reference they add w*0 = +-0 to an accumulator that can never be -0 (it
// starts at +0 and round-to-nearest addition only yields -0 from -0 + -0), so
// skipping them is bit-neutral.  The compiler must not contract mul+add into
// FFMA, hence the explicit __fmul_rn/__fadd_rn.
//
// Each thread owns one output pixel and MB output channels: the (c, j, k)
// input value is loaded once and scaled by MB weights (the reference's
// "for m" loop in _fma_channel_range), which keeps this verification mode
// within a small factor of the fast path for the test sizes.
#include "smmc_internal.cuh"

namespace smmc {
namespace {

constexpr int kExactMB = 8;

template <int MB>
__global__ void __launch_bounds__(128) conv_exact_kernel(Problem p) {
    const int pix = blockIdx.x * blockDim.x + threadIdx.x;
    if (pix >= p.m) return;
    const int m0 = blockIdx.y * MB;
    const int n = pix / p.ohw;
    const int rem = pix - n * p.ohw;
    const int oh = rem / p.ow;
    const int ow = rem - oh * p.ow;
    const int ih0 = oh * p.sh - p.ph;
    const int iw0 = ow * p.sw - p.pw;
    const float* xs = p.x + (int64_t)n * p.c * p.hw;

    float acc[MB];
#pragma unroll
    for (int i = 0; i < MB; ++i) acc[i] = 0.0f;
    const int mcount = min(MB, p.co - m0);

    for (int c = 0; c < p.c; ++c) {
        const float* xc = xs + (int64_t)c * p.hw;
        for (int j = 0; j < p.kw; ++j) {
            const int iw = iw0 + j;
            const bool col_ok = (unsigned)iw < (unsigned)p.w_in;
            const float* wcj = p.w + ((int64_t)(c * p.kw + j) * p.kh) * p.co + m0;
            for (int k = 0; k < p.kh; ++k) {
                const int ih = ih0 + k;
                if (!col_ok || (unsigned)ih >= (unsigned)p.h) continue;
                SMMC_CHECK_RANGE(xc + (int64_t)ih * p.w_in + iw - p.x, 1, (int64_t)p.n * p.c * p.hw);
                SMMC_CHECK_RANGE(wcj + (int64_t)k * p.co - p.w, mcount, (int64_t)p.k * p.co);
                const float xv = __ldg(xc + (int64_t)ih * p.w_in + iw);
                const float* wk = wcj + (int64_t)k * p.co;
#pragma unroll
                for (int i = 0; i < MB; ++i) {
                    if (i < mcount) acc[i] = __fadd_rn(acc[i], __fmul_rn(__ldg(wk + i), xv));
                }
            }
        }
    }
    float* yp = p.y + ((int64_t)n * p.co + m0) * p.ohw + rem;
#pragma unroll
    for (int i = 0; i < MB; ++i)
        if (i < mcount) {
            SMMC_CHECK_RANGE(yp + (int64_t)i * p.ohw - p.y, 1, (int64_t)p.n * p.co * p.ohw);
            yp[(int64_t)i * p.ohw] = acc[i];
        }
}

// buf[r, t] = x[c, r - p_h, j + t*s_w - p_w] or 0 — smm.py:56-73
__global__ void extract_slice_kernel(const float* __restrict__ x, int h, int w, int c, int j,
                                     int sw, int ph, int pw, int hp, int ow,
                                     float* __restrict__ buf) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= hp * ow) return;
    const int r = idx / ow;
    const int t = idx - r * ow;
    const int sr = r - ph;
    const int sc = j + t * sw - pw;
    float v = 0.0f;
    if ((unsigned)sr < (unsigned)h && (unsigned)sc < (unsigned)w)
        v = x[((int64_t)c * h + sr) * w + sc];
    buf[idx] = v;
}

// dst += alpha * src, unfused — smm.py:76-81
__global__ void scalar_matrix_fma_kernel(float alpha, const float* __restrict__ src, int64_t ss,
                                         float* __restrict__ dst, int64_t ds, int rows, int cols) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)rows * cols) return;
    const int r = (int)(idx / cols);
    const int t = (int)(idx - (int64_t)r * cols);
    float* d = dst + r * ds + t;
    *d = __fadd_rn(*d, __fmul_rn(alpha, src[r * ss + t]));
}

}  // namespace

cudaError_t launch_exact(const Problem& p, cudaStream_t s) {
    dim3 block(128);
    dim3 grid((p.m + 127) / 128, (p.co + kExactMB - 1) / kExactMB);
    conv_exact_kernel<kExactMB><<<grid, block, 0, s>>>(p);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_extract_slice(const float* x, const smmc_geom& g, int c, int j, float* buf,
                                 cudaStream_t s) {
    const int ow = (g.w + 2 * g.p_w - g.k_w) / g.s_w + 1;
    const int hp = g.h + 2 * g.p_h;
    const int total = hp * ow;
    extract_slice_kernel<<<(total + 255) / 256, 256, 0, s>>>(x, g.h, g.w, c, j, g.s_w, g.p_h,
                                                             g.p_w, hp, ow, buf);
    count_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_scalar_matrix_fma(float alpha, const float* src, int64_t ss, float* dst,
                                     int64_t ds, int rows, int cols, cudaStream_t s) {
    const int64_t total = (int64_t)rows * cols;
    if (total == 0) return cudaSuccess;
    scalar_matrix_fma_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(alpha, src, ss, dst,
                                                                             ds, rows, cols);
    count_launches(1);
    return cudaGetLastError();
}

}  // namespace smmc

// ---------------------------------------------------------------------------
// GPU im2col comparator (the paper's baseline): the explicit
// lowered matrix of the reference's im2col_pack (im2col.py:22-42), per sample
// [c_i*k_h*k_w][out_h*out_w] with row (c*k_h + k)*k_w + j, zero-filled padding.
// Its size is exactly the scratch SMM-Conv avoids.
namespace smmc {
namespace {

__global__ void im2col_pack_kernel(const float* __restrict__ x, float* __restrict__ low, int n,
                                   int c, int h, int w, int kh, int kw, int sh, int sw, int ph,
                                   int pw, int oh, int ow) {
    const int64_t ohw = (int64_t)oh * ow;
    const int64_t rows = (int64_t)c * kh * kw;
    const int64_t total = (int64_t)n * rows * ohw;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t col = i % ohw;
        const int64_t r = (i / ohw) % rows;
        const int64_t s = i / (ohw * rows);
        const int j = (int)(r % kw);
        const int k = (int)((r / kw) % kh);
        const int cc = (int)(r / ((int64_t)kw * kh));
        const int orow = (int)(col / ow), ocol = (int)(col % ow);
        const int ih = orow * sh + k - ph, iw = ocol * sw + j - pw;
        float v = 0.0f;
        if ((unsigned)ih < (unsigned)h && (unsigned)iw < (unsigned)w)
            v = __ldg(x + ((s * c + cc) * h + ih) * (int64_t)w + iw);
        low[i] = v;
    }
}

}  // namespace

cudaError_t launch_im2col_pack(const float* x, float* low, const smmc_geom& g, int oh, int ow,
                               cudaStream_t s) {
    const int64_t total = (int64_t)g.n * g.c_i * g.k_h * g.k_w * oh * ow;
    if (total == 0) return cudaSuccess;
    const int blocks = (int)((total + 255) / 256 < 148 * 32 ? (total + 255) / 256 : 148 * 32);
    im2col_pack_kernel<<<blocks, 256, 0, s>>>(x, low, g.n, g.c_i, g.h, g.w, g.k_h, g.k_w, g.s_h,
                                              g.s_w, g.p_h, g.p_w, oh, ow);
    count_launches(1);
    return cudaGetLastError();
}

}  // namespace smmc
