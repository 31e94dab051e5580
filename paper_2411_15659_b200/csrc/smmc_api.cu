// smmc_api.cu — the extern "C" boundary (include/smmc.h): validation, kernel
// planning, status/error mapping and the host-buffer staging path.
#include <cuda.h>
#include <sys/mman.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "smmc_internal.cuh"

namespace smmc {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
}  // namespace

void set_error(const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
}

void count_launches(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }

cudaError_t smem_optin(const void* fn, int bytes) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> done;  // (kernel, device) -> bytes set
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_pair(fn, dev);
    auto it = done.find(key);
    if (it != done.end() && it->second >= bytes) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done[key] = bytes;
    return e;
}

namespace {

// ConvGeometry.__post_init__ (geometry.py:32-50), plus batch and int32 range.
int check_geom(const smmc_geom* g, int* oh, int* ow) {
    if (!g) {
        set_error("geometry pointer is NULL");
        return SMMC_EGEOM;
    }
    if (g->n < 0) {
        set_error("batch size must be >= 0, got %d", g->n);
        return SMMC_EGEOM;
    }
    if (g->c_i < 1 || g->c_o < 1 || g->h < 1 || g->w < 1 || g->k_h < 1 || g->k_w < 1) {
        set_error("channel counts, spatial and kernel sizes must be >= 1");
        return SMMC_EGEOM;
    }
    if (g->s_h < 1 || g->s_w < 1) {
        set_error("strides must be >= 1");
        return SMMC_EGEOM;
    }
    if (g->p_h < 0 || g->p_w < 0) {
        set_error("paddings must be >= 0");
        return SMMC_EGEOM;
    }
    const int64_t hp = (int64_t)g->h + 2 * (int64_t)g->p_h;
    const int64_t wp = (int64_t)g->w + 2 * (int64_t)g->p_w;
    if (g->k_h > hp || g->k_w > wp) {
        set_error("kernel %dx%d exceeds padded input %lldx%lld", g->k_h, g->k_w, (long long)hp,
                  (long long)wp);
        return SMMC_EGEOM;
    }
    const int64_t o_h = (hp - g->k_h) / g->s_h + 1;
    const int64_t o_w = (wp - g->k_w) / g->s_w + 1;
    if (o_h < 1 || o_w < 1) {
        set_error("output would be empty for this geometry");
        return SMMC_EGEOM;
    }
    const int64_t m = (int64_t)g->n * o_h * o_w;
    const int64_t k = (int64_t)g->c_i * g->k_h * g->k_w;
    const int64_t xs = (int64_t)g->c_i * g->h * g->w;
    if (m > INT32_MAX || k > INT32_MAX || xs > INT32_MAX || o_h * o_w > INT32_MAX) {
        set_error("problem too large for 32-bit pixel/tap indexing");
        return SMMC_EUNSUPPORTED;
    }
    if (oh) *oh = (int)o_h;
    if (ow) *ow = (int)o_w;
    return SMMC_OK;
}

int sm_count_for(int device) {
    static std::mutex mu;
    static std::vector<int> cache;
    std::lock_guard<std::mutex> lk(mu);
    if (device >= (int)cache.size()) cache.resize(device + 1, 0);
    if (!cache[device]) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v <= 0)
            v = 148;
        cache[device] = v;
    }
    return cache[device];
}

int current_device() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) d = 0;
    return d;
}

int cuda_status(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return SMMC_OK;
    set_error("%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
    // reported here: clear the runtime's (non-sticky) last-error slot so the
    // next launch's cudaGetLastError() does not return this stale failure
    (void)cudaGetLastError();
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) return SMMC_ENODEVICE;
    return SMMC_ECUDA;
}

int check_mode(int mode) {
    if (mode != SMMC_MODE_FFMA && mode != SMMC_MODE_EXACT) {
        set_error("unknown mode %d (0 = ffma, 1 = exact)", mode);
        return SMMC_EUNSUPPORTED;
    }
    return SMMC_OK;
}

size_t workspace_for(const smmc_geom& g, int mode, int sm_count) {
    if (mode != SMMC_MODE_FFMA || g.n == 0) return 0;
    return plan_ffma(g, sm_count).ws_bytes;
}

// Per-device staging buffers for the *_host entry points.
constexpr int kMaxChunks = 64;  // ~4 MB chunks up to 64 per call (fill/drain of the copy pipeline)

struct HostPool {
    std::mutex mu;
    cudaStream_t stream = nullptr;                      // compute
    cudaStream_t s_in = nullptr, s_out = nullptr;       // H2D / D2H copy engines
    cudaEvent_t ev_in[kMaxChunks] = {}, ev_done[kMaxChunks] = {};
    void* buf[4] = {nullptr, nullptr, nullptr, nullptr};
    size_t cap[4] = {0, 0, 0, 0};
};

int ensure_streams(HostPool& hp) {
    if (hp.stream) return SMMC_OK;
    int st;
    if ((st = cuda_status(cudaStreamCreateWithFlags(&hp.stream, cudaStreamNonBlocking),
                          "cudaStreamCreate")) ||
        (st = cuda_status(cudaStreamCreateWithFlags(&hp.s_in, cudaStreamNonBlocking),
                          "cudaStreamCreate")) ||
        (st = cuda_status(cudaStreamCreateWithFlags(&hp.s_out, cudaStreamNonBlocking),
                          "cudaStreamCreate")))
        return st;
    for (int i = 0; i < kMaxChunks; ++i) {
        if ((st = cuda_status(cudaEventCreateWithFlags(&hp.ev_in[i], cudaEventDisableTiming),
                              "cudaEventCreate")) ||
            (st = cuda_status(cudaEventCreateWithFlags(&hp.ev_done[i], cudaEventDisableTiming),
                              "cudaEventCreate")))
            return st;
    }
    return SMMC_OK;
}

// A free (unlocked) staging pool of `device`, returned LOCKED: concurrent
// host-entry calls from several threads (independent layers) each get their
// own streams and buffers and overlap on the copy engines, up to
// kMaxPools per device; beyond that callers queue on a pool.
constexpr int kMaxPools = 4;
HostPool& acquire_pool(int device) {
    static std::mutex mu;
    static std::vector<std::vector<HostPool*>> pools;
    HostPool* wait_on = nullptr;
    {
        std::lock_guard<std::mutex> lk(mu);
        if (device >= (int)pools.size()) pools.resize(device + 1);
        auto& v = pools[device];
        for (HostPool* hp : v)
            if (hp->mu.try_lock()) return *hp;
        if ((int)v.size() < kMaxPools) {
            HostPool* hp = new HostPool();
            hp->mu.lock();
            v.push_back(hp);
            return *hp;
        }
        static unsigned rr = 0;
        wait_on = v[rr++ % v.size()];
    }
    wait_on->mu.lock();
    return *wait_on;
}

void destroy_pool(HostPool& hp) {
    for (int i = 0; i < 4; ++i)
        if (hp.buf[i]) cudaFree(hp.buf[i]);
    for (int i = 0; i < kMaxChunks; ++i) {
        if (hp.ev_in[i]) cudaEventDestroy(hp.ev_in[i]);
        if (hp.ev_done[i]) cudaEventDestroy(hp.ev_done[i]);
    }
    if (hp.stream) cudaStreamDestroy(hp.stream);
    if (hp.s_in) cudaStreamDestroy(hp.s_in);
    if (hp.s_out) cudaStreamDestroy(hp.s_out);
}

int ensure(HostPool& hp, int i, size_t bytes) {
    if (hp.cap[i] >= bytes) return SMMC_OK;
    if (hp.buf[i]) cudaFree(hp.buf[i]);
    hp.buf[i] = nullptr;
    hp.cap[i] = 0;
    if (bytes == 0) return SMMC_OK;
    int st = cuda_status(cudaMalloc(&hp.buf[i], bytes), "cudaMalloc(staging)");
    if (st) return st;
    hp.cap[i] = bytes;
    if (i != 3) return SMMC_OK;
    // the workspace's counter region must start at zero (kernels leave it
    // zeroed).  Ordered on the pool's COMPUTE stream: the pool streams are
    // non-blocking, so a plain cudaMemset (legacy default stream) is not
    // ordered before the conv that uses the buffer -- on a first call with
    // page-locked inputs (fast async H2D) the conv's partial tiles could be
    // zeroed behind its back (seen once as a wrong 512@7 N=1 host-entry
    // result on a fresh box)
#ifdef SMMC_AB_LEGACY_MEMSET  // A/B build reproducing the round-1 race
    return cuda_status(cudaMemset(hp.buf[i], 0, bytes), "cudaMemset(workspace)");
#else
    return cuda_status(cudaMemsetAsync(hp.buf[i], 0, bytes, hp.stream), "cudaMemsetAsync(workspace)");
#endif
}

// Restores the caller's current device on every return path of a host entry.
struct DeviceGuard {
    int prev = -1;
    DeviceGuard() {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// On any early return after work was enqueued on a pool's streams, drain
// them before the pool lock is released: in-flight copies may still read
// the caller's host input / write its host output and the pool buffers.
// Declared after the pool's lock_guard so it runs first.
struct PoolDrain {
    HostPool& hp;
    bool done = false;
    explicit PoolDrain(HostPool& h) : hp(h) {}
    int finish(int st) {
        done = true;
        return st;
    }
    ~PoolDrain() {
        if (done) return;
        if (hp.s_in) cudaStreamSynchronize(hp.s_in);
        if (hp.stream) cudaStreamSynchronize(hp.stream);
        if (hp.s_out) cudaStreamSynchronize(hp.s_out);
    }
};

int select_device(int device) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        set_error("no CUDA device available (%s); this library has no CPU fallback",
                  e == cudaSuccess ? "0 devices" : cudaGetErrorString(e));
        return SMMC_ENODEVICE;
    }
    if (device < 0 || device >= count) {
        set_error("device %d out of range [0, %d)", device, count);
        return SMMC_EINDEX;
    }
    return cuda_status(cudaSetDevice(device), "cudaSetDevice");
}

// Where the epilogue puts the output: n_out replicas of a co_total-channel
// tensor, this problem's channels at offset co_base (fused c_o-shard gather).
struct OutPlace {
    float* const* ys;
    int n_out;
    int co_total;
    int co_base;
};

int conv_device_placed(const float* x, const float* w, const OutPlace& op, const smmc_geom* g,
                       int mode, void* ws, size_t ws_bytes, cudaStream_t stream) {
    int oh = 0, ow = 0;
    int st = check_geom(g, &oh, &ow);
    if (st) return st;
    if ((st = check_mode(mode))) return st;
    if (g->n == 0) return SMMC_OK;
    if (op.n_out < 1 || op.n_out > kMaxOut || !op.ys) {
        set_error("n_out must be in [1, %d]", kMaxOut);
        return SMMC_ESHAPE;
    }
    if (op.co_base < 0 || op.co_total < g->c_o || op.co_base > op.co_total - g->c_o) {
        set_error("channel window [%d, %d) outside a %d-channel output", op.co_base,
                  op.co_base + g->c_o, op.co_total);
        return SMMC_ESHAPE;
    }
    if (!x || !w) {
        set_error("x, w_smm and y must be non-NULL device pointers");
        return SMMC_ESHAPE;
    }
    // x is read with 4-byte copies; w with 16-byte copies; y with float4
    // stores when a channel plane is a multiple of 4 pixels
    const bool y_vec = ((oh * ow) & 3) == 0;
    uintptr_t a16 = (uintptr_t)w, a4 = (uintptr_t)x;
    for (int o = 0; o < op.n_out; ++o) {
        if (!op.ys[o]) {
            set_error("x, w_smm and y must be non-NULL device pointers");
            return SMMC_ESHAPE;
        }
        (y_vec ? a16 : a4) |= (uintptr_t)op.ys[o];
    }
    if ((a16 & 15) || (a4 & 3)) {
        set_error("w_smm (and y when h'*w' %% 4 == 0) must be 16-byte aligned, x 4-byte aligned");
        return SMMC_ESHAPE;
    }
    if (mode == SMMC_MODE_EXACT && (op.n_out != 1 || op.co_total != g->c_o)) {
        set_error("the fused gather epilogue is implemented for the ffma mode only");
        return SMMC_EUNSUPPORTED;
    }
    const int dev = current_device();
    const int sms = sm_count_for(dev);
    Problem p{};
    p.x = x;
    p.w = w;
    p.y = op.ys[0];
    for (int o = 0; o < op.n_out; ++o) p.ys[o] = op.ys[o];
    p.n_out = op.n_out;
    p.co_total = op.co_total;
    p.co_base = op.co_base;
    p.ws = static_cast<float*>(ws);
    p.ws_floats = ws ? (int64_t)(ws_bytes / sizeof(float)) : 0;
    p.n = g->n;
    p.c = g->c_i;
    p.h = g->h;
    p.w_in = g->w;
    p.co = g->c_o;
    p.kh = g->k_h;
    p.kw = g->k_w;
    p.sh = g->s_h;
    p.sw = g->s_w;
    p.ph = g->p_h;
    p.pw = g->p_w;
    p.oh = oh;
    p.ow = ow;
    p.hw = g->h * g->w;
    p.ohw = oh * ow;
    p.m = g->n * oh * ow;
    p.k = g->c_i * g->k_h * g->k_w;
    p.splits = 1;
    if (mode == SMMC_MODE_EXACT) return cuda_status(launch_exact(p, stream), "conv_exact launch");

    const bool placed = op.n_out != 1 || op.co_total != g->c_o || op.co_base != 0;
    const FfmaPlan pl = placed ? plan_ffma_gather(*g, sms) : plan_ffma(*g, sms);
    p.splits = pl.splits;
    p.kt_total = pl.kt_total;
    p.kt_per_split = pl.kt_per_split;
    p.cvec = pl.cvec;
    p.reduce_mode = pl.reduce_mode;
    p.tiles = pl.tiles;
    p.tiles_n = pl.tiles_n;
    p.sk_iters = pl.sk_iters;
    p.sk_maxseg = pl.sk_maxseg;
    if (pl.ws_bytes > 0) {
        if (!ws || ws_bytes < pl.ws_bytes) {
            set_error("workspace of %zu bytes required (got %zu)", pl.ws_bytes, ws_bytes);
            return SMMC_EWORKSPACE;
        }
        if ((uintptr_t)ws & 255) {
            set_error("workspace must be 256-byte aligned");
            return SMMC_ESHAPE;
        }
    }
    if (pl.ws_bytes > 0) {
        // [counter region (zero at rest)][partial tiles], see kCounterRegion
        p.counters = reinterpret_cast<int*>(static_cast<char*>(ws) + pl.ws_counter_offset);
        p.ws = reinterpret_cast<float*>(static_cast<char*>(ws) + pl.ws_partial_offset);
        p.ws_floats = (int64_t)((ws_bytes - pl.ws_partial_offset) / sizeof(float));
    }
    return cuda_status(launch_ffma(p, pl, stream), "conv_ffma launch");
}

int conv_device(const float* x, const float* w, float* y, const smmc_geom* g, int mode, void* ws,
                size_t ws_bytes, cudaStream_t stream) {
    float* ys[1] = {y};
    const OutPlace op{ys, 1, g ? g->c_o : 0, 0};
    return conv_device_placed(x, w, op, g, mode, ws, ws_bytes, stream);
}

}  // namespace
}  // namespace smmc

using namespace smmc;

extern "C" {

int smmc_abi_version(void) { return SMMC_ABI_VERSION; }

const char* smmc_last_error(void) { return g_last_error.c_str(); }

int smmc_geom_check(const smmc_geom* g, int32_t* out_h, int32_t* out_w) {
    int oh = 0, ow = 0;
    int st = check_geom(g, &oh, &ow);
    if (st) return st;
    if (out_h) *out_h = oh;
    if (out_w) *out_w = ow;
    return SMMC_OK;
}

size_t smmc_workspace_bytes(const smmc_geom* g, int mode) {
    int oh = 0, ow = 0;
    if (check_geom(g, &oh, &ow) || check_mode(mode)) return 0;
    return workspace_for(*g, mode, sm_count_for(current_device()));
}

int smmc_plan_launches(const smmc_geom* g, int mode) {
    int oh = 0, ow = 0;
    if (check_geom(g, &oh, &ow) || check_mode(mode)) return -1;
    if (g->n == 0) return 0;
    if (mode == SMMC_MODE_EXACT) return 1;
    return ffma_launches(plan_ffma(*g, sm_count_for(current_device())));
}

int smmc_tc_plan_describe(const smmc_geom* g, char* buf, size_t len) {
    int oh = 0, ow = 0;
    int st = check_geom(g, &oh, &ow);
    if (st) return st;
    if (!buf || !len) return SMMC_OK;
    smmc_geom gg = *g;
    if (gg.n == 0) gg.n = 1;
    const TcPlan pl = plan_tc(gg);
    if (!pl.supported) {
        snprintf(buf, len, "tc: unsupported (needs stride 1 and c_i %% 8 == 0)");
        return SMMC_OK;
    }
    if (pl.halo)
        snprintf(buf, len,
                 "tc: tcgen05 bf16 M=%d x N=%d x K=64, TMA SW128 halo (%d rows), %s, %lld x %d tiles",
                 128 * (pl.persistent ? pl.mt : 1), pl.bn, pl.halo_rows,
                 pl.persistent ? "persistent warp-specialised, 2 TMEM accumulators, 16 epilogue warps"
                               : "one tile per CTA, 2 CTAs/SM",
                 (long long)((pl.tiles_m + (pl.persistent ? pl.mt : 1) - 1) / (pl.persistent ? pl.mt : 1)),
                 pl.tiles_n);
    if (pl.halo && pl.splits > 1) {
        const size_t used = strlen(buf);
        snprintf(buf + used, len - used, ", split-K %d x %d channel blocks (with workspace)",
                 pl.splits, pl.cb_per_split);
    }
    if (!pl.halo)
        snprintf(buf, len, "tc: tcgen05 bf16 M=128 x N=%d x K=64, TMA SW128 4-D box per tap (%dx%dx%d px), "
                 "%lld x %d tiles", pl.bn, pl.tw, pl.th, pl.nb, (long long)pl.tiles_m, pl.tiles_n);
    return SMMC_OK;
}

int smmc_plan_describe(const smmc_geom* g, int mode, char* buf, size_t len) {
    int oh = 0, ow = 0;
    int st = check_geom(g, &oh, &ow);
    if (st) return st;
    if ((st = check_mode(mode))) return st;
    if (!buf || !len) return SMMC_OK;
    if (mode == SMMC_MODE_EXACT) {
        snprintf(buf, len, "exact: 1 px x 8 c_o per thread, (c,j,k) order, fmul_rn+fadd_rn");
        return SMMC_OK;
    }
    const FfmaPlan pl = plan_ffma(*g, sm_count_for(current_device()));
    if (pl.stem) {
        stem_describe(*g, pl.stem, buf, len);
        return SMMC_OK;
    }
    snprintf(buf, len,
             "ffma: tile %dx%dx%d, %d threads, taps=%d, %s K order, split_k=%d (%d of %d tap blocks "
             "each, reduce=%s), %lld tiles",
             pl.bm, pl.bn, pl.bk, pl.threads, pl.tap_kind, pl.cvec ? "tap-major" : "(c,j,k)",
             pl.splits, pl.kt_per_split, pl.kt_total,
             pl.reduce_mode == 0 ? "none"
             : pl.reduce_mode == 1 ? "last-arriver"
             : pl.reduce_mode == 2 ? "kernel"
             : pl.reduce_mode == 4 ? "cluster DSMEM"
             : pl.reduce_mode == 5 ? "in-kernel, all splits"
                                   : "stream-K",
             (long long)pl.tiles);
    if (pl.groups > 1) {
        const size_t used = strlen(buf);
        snprintf(buf + used, len - used, ", %d warp groups x %d threads", pl.groups, pl.threads);
    }
    if (pl.persist1x1) {
        const size_t used = strlen(buf);
        snprintf(buf + used, len - used, "%s", conv1x1_describe(*g, sm_count_for(current_device())));
    }
    if (pl.reduce_mode == 3) {
        const size_t used = strlen(buf);
        snprintf(buf + used, len - used, ", stream-K %d CTAs x %d tap blocks", pl.sk_ctas,
                 pl.sk_iters);
    }
    return SMMC_OK;
}

uint64_t smmc_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

// Measure the candidate plans of one geometry on the current device and keep
// the fastest for the rest of the process (plan_record).  Scratch operands are
// allocated here (contents irrelevant to the timing: a finite constant), every
// candidate runs `iters` back-to-back launches between CUDA events on a private
// stream after two warm-up launches; a candidate that fails to launch is
// skipped.  The winner replaces the default only when it is > 5 % faster.
int smmc_autotune_f32(const smmc_geom* g, int iters, char* report, size_t report_len) {
    int oh = 0, ow = 0;
    int st = check_geom(g, &oh, &ow);
    if (st) return st;
    if (report && report_len) report[0] = 0;
    if (g->n == 0) return SMMC_OK;
    iters = std::max(1, std::min(iters, 1000));
    const int sms = sm_count_for(current_device());
    plan_record(*g, nullptr);
    plan_force(nullptr);
    PlanChoice cands[64];
    const int nc = plan_candidates(*g, sms, cands, 64);
    size_t ws_bytes = plan_ffma(*g, sms).ws_bytes;
    for (int i = 0; i < nc; ++i) {
        plan_force(&cands[i]);
        ws_bytes = std::max(ws_bytes, plan_ffma(*g, sms).ws_bytes);
    }
    plan_force(nullptr);
    const size_t xb = (size_t)g->n * g->c_i * g->h * g->w * sizeof(float);
    const size_t wb = (size_t)g->c_i * g->k_h * g->k_w * g->c_o * sizeof(float);
    const size_t yb = (size_t)g->n * g->c_o * oh * ow * sizeof(float);
    float *x = nullptr, *w = nullptr, *y = nullptr;
    void* ws = nullptr;
    cudaStream_t s = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    auto cleanup = [&]() {
        plan_force(nullptr);
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
        if (s) cudaStreamDestroy(s);
        cudaFree(x);
        cudaFree(w);
        cudaFree(y);
        cudaFree(ws);
    };
    cudaError_t ce = cudaMalloc(&x, xb);
    if (ce == cudaSuccess) ce = cudaMalloc(&w, wb);
    if (ce == cudaSuccess) ce = cudaMalloc(&y, yb);
    if (ce == cudaSuccess && ws_bytes) ce = cudaMalloc(&ws, ws_bytes);
    if (ce == cudaSuccess) ce = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    if (ce == cudaSuccess) ce = cudaEventCreate(&e0);
    if (ce == cudaSuccess) ce = cudaEventCreate(&e1);
    if (ce == cudaSuccess) ce = cudaMemsetAsync(x, 0x3c, xb, s);   // 0x3c3c3c3c = 0.0115f
    if (ce == cudaSuccess) ce = cudaMemsetAsync(w, 0x3c, wb, s);
    if (ce == cudaSuccess && ws_bytes) ce = cudaMemsetAsync(ws, 0, ws_bytes, s);  // counters zero at rest
    if (ce != cudaSuccess) {
        cleanup();
        return cuda_status(ce, "autotune scratch");
    }
    // one candidate: two warm-up launches, then `iters` launches captured into a
    // CUDA graph (no per-launch host overhead: with stream launches a 5 us kernel
    // is timed at 7-8 us and the cooperative / two-launch plans pay different
    // overheads) replayed once untimed and once between events
    auto time_plan = [&](const PlanChoice* c, float* us) -> bool {
        plan_force(c);
        bool ok = true;
        for (int i = 0; i < 2 && ok; ++i) ok = conv_device(x, w, y, g, SMMC_MODE_FFMA, ws, ws_bytes, s) == SMMC_OK;
        if (ok) ok = cudaStreamSynchronize(s) == cudaSuccess;
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        if (ok) {
            ok = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
            if (ok) {
                for (int i = 0; i < iters && ok; ++i)
                    ok = conv_device(x, w, y, g, SMMC_MODE_FFMA, ws, ws_bytes, s) == SMMC_OK;
                const bool ended = cudaStreamEndCapture(s, &graph) == cudaSuccess && graph;
                ok = ok && ended;
            }
            if (ok) ok = cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
            if (ok) ok = cudaGraphLaunch(exec, s) == cudaSuccess && cudaStreamSynchronize(s) == cudaSuccess;
            if (ok) {
                cudaEventRecord(e0, s);
                ok = cudaGraphLaunch(exec, s) == cudaSuccess;
                cudaEventRecord(e1, s);
                ok = cudaStreamSynchronize(s) == cudaSuccess && ok;
            }
        }
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        plan_force(nullptr);
        if (!ok) {
            cudaGetLastError();  // a refused launch (e.g. cooperative grid too large) is not sticky
            return false;
        }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        *us = ms * 1e3f / (float)iters;
        return true;
    };
    float t_def = 0.f;
    if (!time_plan(nullptr, &t_def)) {
        cleanup();
        set_error("autotune: the default plan failed to run");
        return SMMC_ECUDA;
    }
    int best = -1;
    float t_best = t_def;
    for (int i = 0; i < nc; ++i) {
        float t = 0.f;
        if (time_plan(&cands[i], &t) && t < t_best) {
            t_best = t;
            best = i;
        }
    }
    const bool keep = best >= 0 && t_best < 0.95f * t_def;
    if (keep) plan_record(*g, &cands[best]);
    if (report && report_len) {
        if (keep)
            snprintf(report, report_len, "default %.1f us; kept plan %d,%d,%d,%d%s at %.1f us (%d candidates)",
                     t_def, cands[best].variant, cands[best].splits, cands[best].groups,
                     cands[best].reduce, cands[best].variant < 0 ? " (tiled kernel, cost-model plan)" : "", t_best, nc);
        else
            snprintf(report, report_len, "default %.1f us kept (%d candidates, none > 5 %% faster)", t_def, nc);
    }
    cleanup();
    return SMMC_OK;
}

int smmc_autotune_clear(void) {
    plan_record_clear();
    return SMMC_OK;
}

int smmc_conv2d_fwd_f32(const float* x, const float* w_smm, float* y, const smmc_geom* g, int mode,
                        void* workspace, size_t workspace_bytes, void* stream) {
    return conv_device(x, w_smm, y, g, mode, workspace, workspace_bytes,
                       static_cast<cudaStream_t>(stream));
}

int smmc_conv2d_fwd_f32_gather(const float* x, const float* w_slice, float* const* y_out, int n_out,
                               const smmc_geom* g_local, int co_base, int co_total, void* workspace,
                               size_t workspace_bytes, void* stream) {
    if (!y_out) {
        set_error("y_out must point to n_out device pointers");
        return SMMC_ESHAPE;
    }
    const OutPlace op{y_out, n_out, co_total, co_base};
    return conv_device_placed(x, w_slice, op, g_local, SMMC_MODE_FFMA, workspace, workspace_bytes,
                              static_cast<cudaStream_t>(stream));
}

namespace {
using PFN_memGetAddressRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
PFN_memGetAddressRange address_range_fn() {
    static PFN_memGetAddressRange fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_memGetAddressRange>(ptr);
    });
    return fn;
}
}  // namespace

size_t smmc_gather_workspace_bytes(const smmc_geom* g_local) {
    int oh = 0, ow = 0;
    if (check_geom(g_local, &oh, &ow) || g_local->n == 0) return 0;
    return plan_ffma_gather(*g_local, sm_count_for(current_device())).ws_bytes;
}

int smmc_ipc_handle(const void* dev_ptr, void* handle, size_t* offset) {
    if (!dev_ptr || !handle || !offset) {
        set_error("dev_ptr, handle and offset must be non-NULL");
        return SMMC_ESHAPE;
    }
    static_assert(sizeof(cudaIpcMemHandle_t) <= SMMC_IPC_HANDLE_BYTES, "handle size");
    PFN_memGetAddressRange range = address_range_fn();
    if (!range) {
        set_error("cuMemGetAddressRange unavailable from the driver");
        return SMMC_ECUDA;
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, (CUdeviceptr)(uintptr_t)dev_ptr) != CUDA_SUCCESS) {
        set_error("dev_ptr is not inside a device allocation");
        return SMMC_ESHAPE;
    }
    cudaIpcMemHandle_t h;
    int st = cuda_status(cudaIpcGetMemHandle(&h, (void*)(uintptr_t)base), "cudaIpcGetMemHandle");
    if (st) return st;
    memset(handle, 0, SMMC_IPC_HANDLE_BYTES);
    memcpy(handle, &h, sizeof(h));
    *offset = (size_t)((uintptr_t)dev_ptr - (uintptr_t)base);
    return SMMC_OK;
}

int smmc_ipc_open(const void* handle, size_t offset, void** dev_ptr) {
    if (!handle || !dev_ptr) {
        set_error("handle and dev_ptr must be non-NULL");
        return SMMC_ESHAPE;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    void* base = nullptr;
    int st = cuda_status(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess),
                         "cudaIpcOpenMemHandle");
    if (st) return st;
    *dev_ptr = static_cast<char*>(base) + offset;
    return SMMC_OK;
}

int smmc_ipc_close(void* dev_ptr, size_t offset) {
    if (!dev_ptr) return SMMC_OK;
    return cuda_status(cudaIpcCloseMemHandle(static_cast<char*>(dev_ptr) - offset),
                       "cudaIpcCloseMemHandle");
}

namespace smmc {
namespace {
// The host-buffer pipeline on one staging pool's streams, enqueued only
// (the caller synchronizes hp.s_out).  `w_dev` non-NULL: the weights already
// live on the device (a fitted smmc_layer) and are not uploaded.
int enqueue_host_pipeline(HostPool& hp, const float* x, const float* w_smm, const float* w_dev,
                          float* y, const smmc_geom* g, int mode, int device) {
    int oh = 0, ow = 0;
    int st = check_geom(g, &oh, &ow);
    if (st) return st;
    if ((st = ensure_streams(hp))) return st;
    const size_t xs = (size_t)g->c_i * g->h * g->w;          // floats per input sample
    const size_t ys = (size_t)g->c_o * oh * ow;              // floats per output sample
    const size_t xb = (size_t)g->n * xs * sizeof(float);
    const size_t wb = (size_t)g->c_i * g->k_w * g->k_h * g->c_o * sizeof(float);
    const size_t yb = (size_t)g->n * ys * sizeof(float);
    // Pipeline: the batch is cut into chunks of whole samples; chunk c's H2D
    // (copy stream), conv (compute stream) and D2H (second copy stream) overlap
    // with its neighbours'.  ~4 MB chunks (measured: 4 MB beat 8/16/32 MB on
    // the config-2 step, tools/e2e_probe.py with SMMC_HOST_CHUNK_MB).
    const size_t per_sample = (xs + ys) * sizeof(float);
    int chunks = (int)std::min<size_t>((size_t)kMaxChunks, (size_t)g->n);
    static const size_t chunk_bytes = [] {
        const char* f = getenv("SMMC_HOST_CHUNK_MB");  // tuning hook
        return (size_t)(f && atoi(f) > 0 ? atoi(f) : 16) << 20;
    }();
    chunks = (int)std::min<size_t>((size_t)chunks, std::max<size_t>(1, (per_sample * g->n) / chunk_bytes));
    const int per = (g->n + chunks - 1) / chunks;
    chunks = (g->n + per - 1) / per;
    smmc_geom gc = *g;
    gc.n = per;
    size_t wsb = workspace_for(gc, mode, sm_count_for(device));
    gc.n = g->n - (chunks - 1) * per;
    wsb = std::max(wsb, workspace_for(gc, mode, sm_count_for(device)));
    if ((st = ensure(hp, 0, xb)) || (st = ensure(hp, 1, w_dev ? 16 : wb)) ||
        (st = ensure(hp, 2, yb)) || (st = ensure(hp, 3, wsb)))
        return st;
    float* xd = static_cast<float*>(hp.buf[0]);
    const float* wd = w_dev ? w_dev : static_cast<float*>(hp.buf[1]);
    float* yd = static_cast<float*>(hp.buf[2]);
    if (!w_dev && (st = cuda_status(cudaMemcpyAsync(hp.buf[1], w_smm, wb, cudaMemcpyHostToDevice,
                                                    hp.s_in),
                                    "H2D w_smm")))
        return st;
    // All H2D copies are enqueued first: streams share a few hardware queues,
    // and an H2D queued behind a conv's event wait stalls the copy engine.
    for (int c = 0; c < chunks; ++c) {
        const int n0 = c * per;
        const int nc = std::min(per, g->n - n0);
        const size_t xo = (size_t)n0 * xs;
        if ((st = cuda_status(cudaMemcpyAsync(xd + xo, x + xo, nc * xs * sizeof(float),
                                              cudaMemcpyHostToDevice, hp.s_in),
                              "H2D x")) ||
            (st = cuda_status(cudaEventRecord(hp.ev_in[c], hp.s_in), "cudaEventRecord")))
            return st;
    }
    for (int c = 0; c < chunks; ++c) {
        const int n0 = c * per;
        gc.n = std::min(per, g->n - n0);
        const size_t xo = (size_t)n0 * xs, yo = (size_t)n0 * ys;
        if ((st = cuda_status(cudaStreamWaitEvent(hp.stream, hp.ev_in[c], 0), "cudaStreamWaitEvent")))
            return st;
        if ((st = conv_device(xd + xo, wd, yd + yo, &gc, mode, hp.buf[3], wsb, hp.stream))) return st;
        if ((st = cuda_status(cudaEventRecord(hp.ev_done[c], hp.stream), "cudaEventRecord")) ||
            (st = cuda_status(cudaStreamWaitEvent(hp.s_out, hp.ev_done[c], 0),
                              "cudaStreamWaitEvent")) ||
            (st = cuda_status(cudaMemcpyAsync(y + yo, yd + yo, gc.n * ys * sizeof(float),
                                              cudaMemcpyDeviceToHost, hp.s_out),
                              "D2H y")))
            return st;
    }
    return SMMC_OK;
}

int check_host_args(const float* x, const float* w_smm, const float* w_dev, float* y,
                    const smmc_geom* g, int mode) {
    int oh = 0, ow = 0;
    int st = check_geom(g, &oh, &ow);
    if (st) return st;
    if ((st = check_mode(mode))) return st;
    if (g->n == 0) return SMMC_OK;
    if (!x || !(w_smm || w_dev) || !y) {
        set_error("x, w_smm and y must be non-NULL host pointers");
        return SMMC_ESHAPE;
    }
    return SMMC_OK;
}

// Synchronous host entry: a free staging pool, the pipeline, then wait.
int host_pipeline(const float* x, const float* w_smm, const float* w_dev, float* y,
                  const smmc_geom* g, int mode, int device) {
    int st = check_host_args(x, w_smm, w_dev, y, g, mode);
    if (st || g->n == 0) return st;
    DeviceGuard dg;
    if ((st = select_device(device))) return st;
    HostPool& hp = acquire_pool(device);
    std::lock_guard<std::mutex> lk(hp.mu, std::adopt_lock);
    PoolDrain drain(hp);
    if ((st = enqueue_host_pipeline(hp, x, w_smm, w_dev, y, g, mode, device))) return st;
    return drain.finish(cuda_status(cudaStreamSynchronize(hp.s_out), "conv (host path)"));
}
}  // namespace
}  // namespace smmc

int smmc_conv2d_fwd_f32_host(const float* x, const float* w_smm, float* y, const smmc_geom* g,
                             int mode, int device) {
    if (!w_smm && g && g->n != 0) {
        set_error("x, w_smm and y must be non-NULL host pointers");
        return SMMC_ESHAPE;
    }
    return host_pipeline(x, w_smm, nullptr, y, g, mode, device);
}

// ---- fitted layers: weights uploaded once (Conv2D.fit), forward on host buffers
struct smmc_layer {
    smmc_geom g;     // n unused
    int device;
    float* w = nullptr;
    // asynchronous forward: the layer's own staging buffers and streams
    std::mutex mu;
    smmc::HostPool* pool = nullptr;
    bool pending = false;
};

int smmc_layer_create(const float* w_smm, const smmc_geom* g, int device, smmc_layer** out) {
    if (!out) {
        set_error("out must be non-NULL");
        return SMMC_ESHAPE;
    }
    *out = nullptr;
    int oh = 0, ow = 0;
    smmc_geom gg = g ? *g : smmc_geom{};
    gg.n = 1;
    int st = check_geom(g ? &gg : nullptr, &oh, &ow);
    if (st) return st;
    if (!w_smm) {
        set_error("w_smm must be a non-NULL host pointer");
        return SMMC_ESHAPE;
    }
    DeviceGuard dg;
    if ((st = select_device(device))) return st;
    const size_t wb = (size_t)gg.c_i * gg.k_w * gg.k_h * gg.c_o * sizeof(float);
    smmc_layer* L = new smmc_layer();
    L->g = gg;
    L->device = device;
    if ((st = cuda_status(cudaMalloc(&L->w, wb), "cudaMalloc(weights)")) ||
        (st = cuda_status(cudaMemcpy(L->w, w_smm, wb, cudaMemcpyHostToDevice), "H2D weights"))) {
        if (L->w) cudaFree(L->w);
        delete L;
        return st;
    }
    *out = L;
    return SMMC_OK;
}

int smmc_layer_forward_host(smmc_layer* L, const float* x, float* y, int n, int mode) {
    if (!L) {
        set_error("layer is NULL");
        return SMMC_ESHAPE;
    }
    smmc_geom g = L->g;
    g.n = n;
    return host_pipeline(x, nullptr, L->w, y, &g, mode, L->device);
}

int smmc_layer_forward_host_async(smmc_layer* L, const float* x, float* y, int n, int mode) {
    if (!L) {
        set_error("layer is NULL");
        return SMMC_ESHAPE;
    }
    smmc_geom g = L->g;
    g.n = n;
    int st = check_host_args(x, nullptr, L->w, y, &g, mode);
    if (st || n == 0) return st;
    DeviceGuard dg;
    if ((st = select_device(L->device))) return st;
    std::lock_guard<std::mutex> lk(L->mu);
    if (!L->pool) L->pool = new HostPool();
    if (L->pending) {  // the layer's buffers are still in use by the previous call
        L->pending = false;
        if ((st = cuda_status(cudaStreamSynchronize(L->pool->s_out), "conv (async host path)")))
            return st;
    }
    PoolDrain drain(*L->pool);
    if ((st = enqueue_host_pipeline(*L->pool, x, nullptr, L->w, y, &g, mode, L->device))) return st;
    L->pending = true;
    return drain.finish(SMMC_OK);  // in flight: smmc_layer_wait drains it
}

int smmc_layer_wait(smmc_layer* L) {
    if (!L) {
        set_error("layer is NULL");
        return SMMC_ESHAPE;
    }
    std::lock_guard<std::mutex> lk(L->mu);
    if (!L->pending) return SMMC_OK;
    L->pending = false;
    DeviceGuard dg;
    cudaSetDevice(L->device);
    return cuda_status(cudaStreamSynchronize(L->pool->s_out), "conv (async host path)");
}

int smmc_layer_destroy(smmc_layer* L) {
    if (!L) return SMMC_OK;
    int st = smmc_layer_wait(L);
    DeviceGuard dg;
    cudaSetDevice(L->device);
    if (L->w) {
        const int e = cuda_status(cudaFree(L->w), "cudaFree(weights)");
        if (!st) st = e;
    }
    if (L->pool) {
        destroy_pool(*L->pool);
        delete L->pool;
    }
    delete L;
    return st;
}


// ---- pinned host staging buffers for the *_host entries.  cudaHostAlloc
// memory measured only 29-36 GB/s H2D on the B200 boxes (KVM guest), while
// ordinary pages pinned with cudaHostRegister reach 55 GB/s (the PCIe Gen5
// x16 rate; tools/hostmem_probe.py): allocate 2 MB-aligned anonymous pages
// (transparent-huge-page advised) and register them.
namespace {
std::mutex g_pinned_mu;
std::vector<std::pair<void*, std::pair<void*, size_t>>> g_pinned;  // user ptr -> (map, len)
}  // namespace

int smmc_host_alloc_pinned(size_t bytes, void** ptr) {
    if (!ptr) {
        set_error("ptr must be non-NULL");
        return SMMC_ESHAPE;
    }
    *ptr = nullptr;
    if (bytes == 0) return SMMC_OK;
    constexpr size_t kHuge = 2u << 20;
    const size_t len = (bytes + kHuge - 1) / kHuge * kHuge + kHuge;
    void* map = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (map == MAP_FAILED) {
        set_error("mmap of %zu bytes failed", len);
        return SMMC_ECUDA;
    }
    void* p = reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(map) + kHuge - 1) & ~(uintptr_t)(kHuge - 1));
    const size_t plen = (bytes + kHuge - 1) / kHuge * kHuge;
    madvise(p, plen, MADV_HUGEPAGE);
    int st = cuda_status(cudaHostRegister(p, plen, cudaHostRegisterPortable), "cudaHostRegister");
    if (st) {
        munmap(map, len);
        return st;
    }
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    g_pinned.push_back({p, {map, len}});
    *ptr = p;
    return SMMC_OK;
}

int smmc_host_free_pinned(void* ptr) {
    if (!ptr) return SMMC_OK;
    std::pair<void*, size_t> m{nullptr, 0};
    {
        std::lock_guard<std::mutex> lk(g_pinned_mu);
        for (size_t i = 0; i < g_pinned.size(); ++i)
            if (g_pinned[i].first == ptr) {
                m = g_pinned[i].second;
                g_pinned.erase(g_pinned.begin() + i);
                break;
            }
    }
    if (!m.first) {
        set_error("pointer was not allocated by smmc_host_alloc_pinned");
        return SMMC_ESHAPE;
    }
    const int st = cuda_status(cudaHostUnregister(ptr), "cudaHostUnregister");
    munmap(m.first, m.second);
    return st;
}

size_t smmc_im2col_bytes(const smmc_geom* g) {
    int oh = 0, ow = 0;
    if (check_geom(g, &oh, &ow)) return 0;
    return (size_t)g->n * g->c_i * g->k_h * g->k_w * oh * ow * sizeof(float);
}

int smmc_im2col_pack_f32(const float* x, float* lowered, const smmc_geom* g, void* stream) {
    int oh = 0, ow = 0;
    int st = check_geom(g, &oh, &ow);
    if (st) return st;
    if (g->n == 0) return SMMC_OK;
    if (!x || !lowered) {
        set_error("x and lowered must be non-NULL device pointers");
        return SMMC_ESHAPE;
    }
    return cuda_status(launch_im2col_pack(x, lowered, *g, oh, ow, static_cast<cudaStream_t>(stream)),
                       "im2col_pack launch");
}

int smmc_tc_supported(const smmc_geom* g) {
    int oh = 0, ow = 0;
    if (check_geom(g, &oh, &ow)) return 0;
    smmc_geom gg = *g;
    if (gg.n == 0) gg.n = 1;
    return plan_tc(gg).supported ? 1 : 0;
}

int smmc_pack_input_bf16_nhwc(const float* x, uint16_t* x_nhwc, const smmc_geom* g, void* stream) {
    int oh = 0, ow = 0;
    int st = check_geom(g, &oh, &ow);
    if (st) return st;
    if (g->n == 0) return SMMC_OK;
    if (!x || !x_nhwc) {
        set_error("x and x_nhwc must be non-NULL device pointers");
        return SMMC_ESHAPE;
    }
    if ((g->c_i & 7) || ((uintptr_t)x_nhwc & 15)) {
        set_error("bf16 pack needs c_i %% 8 == 0 and a 16-byte aligned x_nhwc");
        return SMMC_EUNSUPPORTED;
    }
    return cuda_status(launch_pack_input_nhwc(x, x_nhwc, *g, static_cast<cudaStream_t>(stream)),
                       "pack_input_nhwc launch");
}

int smmc_pack_weights_bf16(const float* w_smm, uint16_t* w_tc, const smmc_geom* g, void* stream) {
    int oh = 0, ow = 0;
    int st = check_geom(g, &oh, &ow);
    if (st) return st;
    if (!w_smm || !w_tc) {
        set_error("w_smm and w_tc must be non-NULL device pointers");
        return SMMC_ESHAPE;
    }
    return cuda_status(launch_pack_weights_bf16(w_smm, w_tc, *g, static_cast<cudaStream_t>(stream)),
                       "pack_weights_bf16 launch");
}

int smmc_pack_input_bf16x3_nhwc(const float* x, uint16_t* x3, const smmc_geom* g, void* stream) {
    int oh = 0, ow = 0;
    int st = check_geom(g, &oh, &ow);
    if (st) return st;
    if (g->n == 0) return SMMC_OK;
    if (!x || !x3) {
        set_error("x and x3 must be non-NULL device pointers");
        return SMMC_ESHAPE;
    }
    if ((g->c_i & 7) || ((uintptr_t)x3 & 15)) {
        set_error("bf16x3 pack needs c_i %% 8 == 0 and a 16-byte aligned x3");
        return SMMC_EUNSUPPORTED;
    }
    return cuda_status(launch_pack_input_nhwc(x, x3, *g, static_cast<cudaStream_t>(stream), 3),
                       "pack_input_bf16x3 launch");
}

int smmc_pack_weights_bf16x3(const float* w_smm, uint16_t* w3, const smmc_geom* g, void* stream) {
    int oh = 0, ow = 0;
    int st = check_geom(g, &oh, &ow);
    if (st) return st;
    if (!w_smm || !w3) {
        set_error("w_smm and w3 must be non-NULL device pointers");
        return SMMC_ESHAPE;
    }
    return cuda_status(launch_pack_weights_bf16(w_smm, w3, *g, static_cast<cudaStream_t>(stream), 3),
                       "pack_weights_bf16x3 launch");
}

int smmc_conv2d_fwd_bf16x3_tc(const uint16_t* x3, const uint16_t* w3, float* y, const smmc_geom* g,
                              void* ws, size_t ws_bytes, void* stream) {
    int oh = 0, ow = 0;
    int st = check_geom(g, &oh, &ow);
    if (st) return st;
    if (g->c_i > INT32_MAX / 3) {
        set_error("c_i too large for the split-bf16 path");
        return SMMC_EUNSUPPORTED;
    }
    smmc_geom g3 = *g;  // the bf16 conv over the 3*c_i split channels
    g3.c_i *= 3;
    return smmc_conv2d_fwd_bf16_tc_ws(x3, w3, y, &g3, ws, ws_bytes, stream);
}

size_t smmc_tc_workspace_bytes(const smmc_geom* g, int split3) {
    int oh = 0, ow = 0;
    if (!g || check_geom(g, &oh, &ow) || g->n == 0) return 0;
    smmc_geom gg = *g;
    if (split3) {
        if (gg.c_i > INT32_MAX / 3) return 0;
        gg.c_i *= 3;
    }
    return tc_workspace_bytes(gg);
}

int smmc_conv2d_fwd_bf16_tc(const uint16_t* x_nhwc, const uint16_t* w_tc, float* y,
                            const smmc_geom* g, void* stream) {
    return smmc_conv2d_fwd_bf16_tc_ws(x_nhwc, w_tc, y, g, nullptr, 0, stream);
}

int smmc_conv2d_fwd_bf16_tc_ws(const uint16_t* x_nhwc, const uint16_t* w_tc, float* y,
                               const smmc_geom* g, void* ws, size_t ws_bytes, void* stream) {
    int oh = 0, ow = 0;
    int st = check_geom(g, &oh, &ow);
    if (st) return st;
    if (g->n == 0) return SMMC_OK;
    if (!x_nhwc || !w_tc || !y) {
        set_error("x_nhwc, w_tc and y must be non-NULL device pointers");
        return SMMC_ESHAPE;
    }
    if (((uintptr_t)x_nhwc | (uintptr_t)w_tc) & 15) {
        set_error("x_nhwc and w_tc must be 16-byte aligned (TMA)");
        return SMMC_ESHAPE;
    }
    const char* why = "";
    if (ws && ((uintptr_t)ws & 15)) {
        set_error("workspace must be 16-byte aligned");
        return SMMC_ESHAPE;
    }
    cudaError_t e = launch_tc_bf16(x_nhwc, w_tc, y, *g, static_cast<cudaStream_t>(stream), &why,
                                   static_cast<float*>(ws), ws_bytes);
    if (e == cudaErrorNotSupported) {
        set_error("%s", why);
        return SMMC_EUNSUPPORTED;
    }
    if (e != cudaSuccess && why[0]) {
        set_error("%s (%s)", why, cudaGetErrorString(e));
        return SMMC_ECUDA;
    }
    return cuda_status(e, "conv_tc_bf16 launch");
}

int smmc_extract_slice_f32(const float* x, const smmc_geom* g, int32_t c, int32_t j, float* buf,
                           void* stream) {
    int oh = 0, ow = 0;
    int st = check_geom(g, &oh, &ow);
    if (st) return st;
    if (c < 0 || c >= g->c_i) {
        set_error("channel %d out of range [0, %d)", c, g->c_i);
        return SMMC_EINDEX;
    }
    if (j < 0 || j >= g->k_w) {
        set_error("kernel column %d out of range [0, %d)", j, g->k_w);
        return SMMC_EINDEX;
    }
    if (!x || !buf) {
        set_error("x and buf must be non-NULL");
        return SMMC_ESHAPE;
    }
    return cuda_status(launch_extract_slice(x, *g, c, j, buf, static_cast<cudaStream_t>(stream)),
                       "extract_slice launch");
}

int smmc_scalar_matrix_fma_f32(float alpha, const float* src, int64_t src_row_stride, float* dst,
                               int64_t dst_row_stride, int32_t rows, int32_t cols, void* stream) {
    if (rows < 0 || cols < 0) {
        set_error("rows/cols must be >= 0");
        return SMMC_ESHAPE;
    }
    if ((rows && cols) && (!src || !dst)) {
        set_error("src and dst must be non-NULL");
        return SMMC_ESHAPE;
    }
    return cuda_status(launch_scalar_matrix_fma(alpha, src, src_row_stride, dst, dst_row_stride,
                                                rows, cols, static_cast<cudaStream_t>(stream)),
                       "scalar_matrix_fma launch");
}

int smmc_extract_slice_f32_host(const float* x, const smmc_geom* g, int32_t c, int32_t j,
                                float* buf, int device) {
    int oh = 0, ow = 0;
    int st = check_geom(g, &oh, &ow);
    if (st) return st;
    if (c < 0 || c >= g->c_i || j < 0 || j >= g->k_w) {
        set_error("slice index (c=%d, j=%d) out of range", c, j);
        return SMMC_EINDEX;
    }
    DeviceGuard dg;
    if ((st = select_device(device))) return st;
    HostPool& hp = acquire_pool(device);
    std::lock_guard<std::mutex> lk(hp.mu, std::adopt_lock);
    PoolDrain drain(hp);
    if ((st = ensure_streams(hp))) return st;
    const size_t xb = (size_t)g->c_i * g->h * g->w * sizeof(float);
    const size_t bb = (size_t)(g->h + 2 * g->p_h) * ow * sizeof(float);
    if ((st = ensure(hp, 0, xb)) || (st = ensure(hp, 2, bb))) return st;
    cudaStream_t s = hp.stream;
    if ((st = cuda_status(cudaMemcpyAsync(hp.buf[0], x, xb, cudaMemcpyHostToDevice, s), "H2D x")))
        return st;
    if ((st = smmc_extract_slice_f32(static_cast<float*>(hp.buf[0]), g, c, j,
                                     static_cast<float*>(hp.buf[2]), s)))
        return st;
    if ((st = cuda_status(cudaMemcpyAsync(buf, hp.buf[2], bb, cudaMemcpyDeviceToHost, s), "D2H")))
        return st;
    return drain.finish(cuda_status(cudaStreamSynchronize(s), "extract_slice (host path)"));
}

int smmc_scalar_matrix_fma_f32_host(float alpha, const float* src, int64_t src_row_stride,
                                    float* dst, int64_t dst_row_stride, int32_t rows, int32_t cols,
                                    int device) {
    if (rows < 0 || cols < 0 || src_row_stride < cols || dst_row_stride < cols) {
        set_error("invalid fma view (rows=%d cols=%d strides %lld/%lld)", rows, cols,
                  (long long)src_row_stride, (long long)dst_row_stride);
        return SMMC_ESHAPE;
    }
    if (!rows || !cols) return SMMC_OK;
    DeviceGuard dg;
    int st = select_device(device);
    if (st) return st;
    HostPool& hp = acquire_pool(device);
    std::lock_guard<std::mutex> lk(hp.mu, std::adopt_lock);
    PoolDrain drain(hp);
    if ((st = ensure_streams(hp))) return st;
    const size_t sb = ((size_t)(rows - 1) * src_row_stride + cols) * sizeof(float);
    const size_t db = ((size_t)(rows - 1) * dst_row_stride + cols) * sizeof(float);
    if ((st = ensure(hp, 0, sb)) || (st = ensure(hp, 2, db))) return st;
    cudaStream_t s = hp.stream;
    if ((st = cuda_status(cudaMemcpyAsync(hp.buf[0], src, sb, cudaMemcpyHostToDevice, s), "H2D")))
        return st;
    if ((st = cuda_status(cudaMemcpyAsync(hp.buf[2], dst, db, cudaMemcpyHostToDevice, s), "H2D")))
        return st;
    if ((st = smmc_scalar_matrix_fma_f32(alpha, static_cast<float*>(hp.buf[0]), src_row_stride,
                                         static_cast<float*>(hp.buf[2]), dst_row_stride, rows, cols,
                                         s)))
        return st;
    if ((st = cuda_status(cudaMemcpyAsync(dst, hp.buf[2], db, cudaMemcpyDeviceToHost, s), "D2H")))
        return st;
    return drain.finish(cuda_status(cudaStreamSynchronize(s), "scalar_matrix_fma (host path)"));
}

}  // extern "C"
