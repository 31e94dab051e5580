/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Not part of the product: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library, and only as the checker or the CPU baseline.
 *
 * A plain-C restatement of the reference's SMM-Conv CPU path
 * (/root/reference/pkg/src/smmconv/smm.py), kept bit-exact with it:
 *
 *   extract_slice   smm.py:56-73    buf[r,t] = x[c, r-p_h, j+t*s_w-p_w] or 0
 *   fma_channel     smm.py:84-114   for k: for m in [m0,m1): out[m] += W[c,j,k,m] * window_k
 *                                   (one rounded multiply, one rounded add; no contraction —
 *                                   build with -ffp-contract=off, never -ffast-math)
 *   smm_single      smm.py:226-251  zero out; for c: for j: extract; fma over all m
 *   smm_parallel    smm.py:254-306  Algorithm 2: d workers, worker n owns slice buffer n and
 *                                   output channels [n*ceil(c_o/d), ...); (c,j) pairs processed in
 *                                   groups of d — phase 1 each worker extracts one pair, barrier,
 *                                   phase 2 each worker applies every buffer of the group, in
 *                                   global pair order, to its own channel block, barrier.
 *   Per output element the update sequence is identical for every d, so the
 *   result is bitwise equal to smm_single (smm.py:20-26).
 *
 * Pinned against the reference's own outputs in tests/golden/ (see
 * tests/golden/make_golden.py and tests/test_oracle.py).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct oracle_geom {
    int32_t n, c_i, h, w, c_o, k_h, k_w, s_h, s_w, p_h, p_w;
} oracle_geom;

static int out_h_of(const oracle_geom* g) { return (g->h + 2 * g->p_h - g->k_h) / g->s_h + 1; }
static int out_w_of(const oracle_geom* g) { return (g->w + 2 * g->p_w - g->k_w) / g->s_w + 1; }

/* smm.py:56-73 */
static void extract_slice(const float* x, float* buf, int c, int j, const oracle_geom* g) {
    const int hp = g->h + 2 * g->p_h;
    const int ow = out_w_of(g);
    for (int rr = 0; rr < hp; ++rr) {
        const int sr = rr - g->p_h;
        float* row = buf + (size_t)rr * ow;
        if (sr < 0 || sr >= g->h) {
            for (int t = 0; t < ow; ++t) row[t] = 0.0f;
            continue;
        }
        const float* xr = x + ((size_t)c * g->h + sr) * g->w;
        for (int t = 0; t < ow; ++t) {
            const int sc = j + t * g->s_w - g->p_w;
            row[t] = (sc < 0 || sc >= g->w) ? 0.0f : xr[sc];
        }
    }
}

/* smm.py:84-114; w_kj is the (k_h, c_o) slice W_smm[c, j]. */
static void fma_channel_range(const float* buf, const float* w_kj, float* out, int m0, int m1,
                              const oracle_geom* g) {
    const int oh = out_h_of(g), ow = out_w_of(g);
    const size_t plane = (size_t)oh * ow;
    if (g->s_h == 1) {
        for (int k = 0; k < g->k_h; ++k) {
            const float* src = buf + (size_t)k * ow;
            for (int m = m0; m < m1; ++m) {
                const float alpha = w_kj[(size_t)k * g->c_o + m];
                float* dst = out + (size_t)m * plane;
                for (size_t i = 0; i < plane; ++i) dst[i] = dst[i] + alpha * src[i];
            }
        }
    } else {
        for (int k = 0; k < g->k_h; ++k) {
            for (int m = m0; m < m1; ++m) {
                const float alpha = w_kj[(size_t)k * g->c_o + m];
                float* dst = out + (size_t)m * plane;
                for (int r = 0; r < oh; ++r) {
                    const float* src = buf + (size_t)(k + r * g->s_h) * ow;
                    float* d = dst + (size_t)r * ow;
                    for (int t = 0; t < ow; ++t) d[t] = d[t] + alpha * src[t];
                }
            }
        }
    }
}

/* smm.py:226-251, one sample. */
static int smm_single(const float* x, const float* w_smm, float* out, const oracle_geom* g) {
    const int oh = out_h_of(g), ow = out_w_of(g);
    const size_t hp = (size_t)(g->h + 2 * g->p_h);
    float* buf = (float*)malloc(hp * ow * sizeof(float));
    if (!buf) return 1;
    memset(out, 0, (size_t)g->c_o * oh * ow * sizeof(float));
    const size_t wpair = (size_t)g->k_h * g->c_o;
    for (int c = 0; c < g->c_i; ++c)
        for (int j = 0; j < g->k_w; ++j) {
            extract_slice(x, buf, c, j, g);
            fma_channel_range(buf, w_smm + ((size_t)c * g->k_w + j) * wpair, out, 0, g->c_o, g);
        }
    free(buf);
    return 0;
}

typedef struct par_ctx {
    const float* x;
    const float* w_smm;
    float* out;
    const oracle_geom* g;
    float* bufs;
    size_t buf_elems;
    int d;
    int chunk;
    pthread_barrier_t bar;
} par_ctx;

typedef struct par_arg {
    par_ctx* ctx;
    int n;
} par_arg;

/* smm.py:277-296 */
static void* par_worker(void* p) {
    par_arg* a = (par_arg*)p;
    par_ctx* cx = a->ctx;
    const oracle_geom* g = cx->g;
    const int d = cx->d, n = a->n;
    int m0 = n * cx->chunk;
    if (m0 > g->c_o) m0 = g->c_o;
    int m1 = m0 + cx->chunk;
    if (m1 > g->c_o) m1 = g->c_o;
    const int n_pairs = g->c_i * g->k_w;
    const size_t wpair = (size_t)g->k_h * g->c_o;
    for (int g0 = 0; g0 < n_pairs; g0 += d) {
        const int g1 = g0 + d < n_pairs ? g0 + d : n_pairs;
        if (g0 + n < g1) {
            const int pair = g0 + n;
            extract_slice(cx->x, cx->bufs + (size_t)n * cx->buf_elems, pair / g->k_w,
                          pair % g->k_w, g);
        }
        pthread_barrier_wait(&cx->bar); /* phase 1 writes before phase 2 reads */
        if (m1 > m0)
            for (int idx = g0; idx < g1; ++idx)
                fma_channel_range(cx->bufs + (size_t)(idx - g0) * cx->buf_elems,
                                  cx->w_smm + (size_t)idx * wpair, cx->out, m0, m1, g);
        pthread_barrier_wait(&cx->bar); /* phase 2 reads before the next refill */
    }
    return NULL;
}

/* smm.py:254-306, one sample. */
static int smm_parallel(const float* x, const float* w_smm, float* out, const oracle_geom* g,
                        int d) {
    if (d < 1) return 2;
    if (d == 1) return smm_single(x, w_smm, out, g);
    const int oh = out_h_of(g), ow = out_w_of(g);
    par_ctx cx;
    cx.x = x;
    cx.w_smm = w_smm;
    cx.out = out;
    cx.g = g;
    cx.d = d;
    cx.chunk = (g->c_o + d - 1) / d;
    cx.buf_elems = (size_t)(g->h + 2 * g->p_h) * ow;
    cx.bufs = (float*)malloc((size_t)d * cx.buf_elems * sizeof(float));
    if (!cx.bufs) return 1;
    memset(out, 0, (size_t)g->c_o * oh * ow * sizeof(float));
    pthread_barrier_init(&cx.bar, NULL, (unsigned)d);
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * d);
    par_arg* args = (par_arg*)malloc(sizeof(par_arg) * d);
    for (int i = 0; i < d; ++i) {
        args[i].ctx = &cx;
        args[i].n = i;
        pthread_create(&th[i], NULL, par_worker, &args[i]);
    }
    for (int i = 0; i < d; ++i) pthread_join(th[i], NULL);
    pthread_barrier_destroy(&cx.bar);
    free(args);
    free(th);
    free(cx.bufs);
    return 0;
}

/* ---------------------------------------------------------------- exports */

int oracle_out_hw(const oracle_geom* g, int32_t* oh, int32_t* ow) {
    *oh = out_h_of(g);
    *ow = out_w_of(g);
    return 0;
}

/* Batch (n, c_i, h, w) -> (n, c_o, oh, ow): Conv2D.transform's per-sample loop
 * (estimator.py:123-124) around smm_parallel (threads > 1) or smm_single. */
int oracle_smm_conv(const float* x, const float* w_smm, float* y, const oracle_geom* g,
                    int threads) {
    const size_t xs = (size_t)g->c_i * g->h * g->w;
    const size_t ys = (size_t)g->c_o * out_h_of(g) * out_w_of(g);
    for (int i = 0; i < g->n; ++i) {
        int st = threads > 1 ? smm_parallel(x + i * xs, w_smm, y + i * ys, g, threads)
                             : smm_single(x + i * xs, w_smm, y + i * ys, g);
        if (st) return st;
    }
    return 0;
}

/* The zero-packed slice of sample 0 (extract_slice, smm.py:190-203). */
int oracle_extract_slice(const float* x, const oracle_geom* g, int c, int j, float* buf) {
    extract_slice(x, buf, c, j, g);
    return 0;
}

/* Secondary oracle: the reference's naive direct conv (reference.py:18-38),
 * (c, k, j) order, float32 accumulator, padded taps skipped; weights OIHW. */
int oracle_conv_ref(const float* x, const float* w_oihw, float* y, const oracle_geom* g) {
    const int oh = out_h_of(g), ow = out_w_of(g);
    const size_t xs = (size_t)g->c_i * g->h * g->w;
    const size_t ys = (size_t)g->c_o * oh * ow;
    for (int s = 0; s < g->n; ++s)
        for (int m = 0; m < g->c_o; ++m)
            for (int r = 0; r < oh; ++r)
                for (int t = 0; t < ow; ++t) {
                    float acc = 0.0f;
                    for (int c = 0; c < g->c_i; ++c)
                        for (int k = 0; k < g->k_h; ++k) {
                            const int rr = r * g->s_h + k - g->p_h;
                            if (rr < 0 || rr >= g->h) continue;
                            for (int j = 0; j < g->k_w; ++j) {
                                const int xx = t * g->s_w + j - g->p_w;
                                if (xx < 0 || xx >= g->w) continue;
                                const float wv =
                                    w_oihw[(((size_t)m * g->c_i + c) * g->k_h + k) * g->k_w + j];
                                acc = acc + wv * x[s * xs + ((size_t)c * g->h + rr) * g->w + xx];
                            }
                        }
                    y[s * ys + ((size_t)m * oh + r) * ow + t] = acc;
                }
    return 0;
}
