// smmc_internal.cuh — shared device/host plumbing for the sm_100a SMM-Conv kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <atomic>
#include <string>

#include "../../include/smmc.h"

// ---- SMMC_CHECKED builds (tools/checked_build.sh -> lib/checked/libsmmc.so,
// selected with SMMC_LIB): device-side bounds asserts on the global and
// shared-memory accesses of every kernel family; a violation prints the
// site and traps.  compute-sanitizer is closed on the GPU pool, so this is
// the out-of-bounds check.  Compiled out of the product library.
#ifdef SMMC_CHECKED
#include <cstdio>
#define SMMC_ASSERT(cond)                                                                    \
    do {                                                                                     \
        if (!(cond)) {                                                                       \
            printf("SMMC_CHECKED %s:%d: %s (block %d,%d,%d thread %d)\n", __FILE__, __LINE__, \
                   #cond, (int)blockIdx.x, (int)blockIdx.y, (int)blockIdx.z, (int)threadIdx.x);     \
            __trap();                                                                        \
        }                                                                                    \
    } while (0)
__device__ __forceinline__ uint32_t smmc_dyn_smem_bytes() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
    return r;
}
// [addr, addr + bytes) inside the dynamic shared memory starting at base (u32 addresses)
#define SMMC_CHECK_SMEM(base, addr, bytes)                                 \
    SMMC_ASSERT((uint32_t)(addr) >= (uint32_t)(base) &&                    \
                (uint32_t)(addr) - (uint32_t)(base) + (uint32_t)(bytes) <= \
                    smmc_dyn_smem_bytes())
// [off, off + count) inside [0, total)
#define SMMC_CHECK_RANGE(off, count, total) \
    SMMC_ASSERT((int64_t)(off) >= 0 && (int64_t)(off) + (int64_t)(count) <= (int64_t)(total))
#else
#define SMMC_ASSERT(cond) \
    do {                  \
    } while (0)
#define SMMC_CHECK_SMEM(base, addr, bytes) \
    do {                                   \
    } while (0)
#define SMMC_CHECK_RANGE(off, count, total) \
    do {                                    \
    } while (0)
#endif

namespace smmc {

// ----------------------------------------------------------------- problem
// Resolved problem description passed by value to every kernel.
constexpr int kMaxOut = 8;  // output replicas of the fused c_o-shard gather

struct Problem {
    const float* x;      // (n, c_i, h, w)
    const float* w;      // (c_i, k_w, k_h, c_o) == row-major [K][c_o], K = c_i*k_w*k_h
    float* y;            // (n, c_o, oh, ow)
    float* ws;           // split-K partial tiles [tiles][splits][BM*BN] (or null)
    int64_t ws_floats;   // capacity of ws in floats (bounds of the checked build)
    int* counters;       // split-K arrival counters [tiles] (zero at rest)
    int n, c, h, w_in, co, kh, kw, sh, sw, ph, pw, oh, ow;
    int hw;              // h*w
    int ohw;             // oh*ow
    int m;               // GEMM rows: n*oh*ow output pixels
    int k;               // GEMM depth: c_i*k_w*k_h taps (SMM (c, j, k) order)
    int kt_total;        // BK-wide tap blocks along K
    int kt_per_split;    // tap blocks per split
    int splits;
    int cvec;            // 1: tap-major K order (c_i % BK == 0)
    int reduce_mode;     // 0 none, 1 split-K last-arriver, 2 split-K reduce kernel, 3 stream-K,
                         // 4 split-K reduced in a thread-block cluster (DSMEM),
                         // 5 split-K reduced in-kernel by all S CTAs of a tile (co-resident grid)
    int64_t tiles;       // pixel tiles x channel tiles
    int tiles_n;         // channel tiles
    int sk_iters;        // stream-K: tap blocks per CTA
    int sk_maxseg;       // stream-K: partial-tile slots per tile in the workspace
    // Output placement.  Normally n_out = 1, ys[0] = y, co_total = co,
    // co_base = 0.  The fused c_o-shard all-gather (smmc_conv2d_fwd_f32_gather)
    // writes this rank's channels [co_base, co_base + co) of a
    // (n, co_total, oh, ow) tensor into every replica ys[0..n_out) — local and
    // NVLink peer memory — straight from the epilogue.
    float* ys[kMaxOut];
    int n_out;
    int co_total;
    int co_base;
};

// Last-error / launch bookkeeping (defined in smmc_api.cu).
void set_error(const char* fmt, ...);
void count_launches(int n);

// Opt `fn` in to `bytes` of dynamic shared memory on the CURRENT device.  The
// attribute lives in the device's context, so it is cached per (kernel,
// device); failures are not cached (defined in smmc_api.cu).
cudaError_t smem_optin(const void* fn, int bytes);
template <typename F>
inline cudaError_t smem_optin(F* fn, int bytes) {
    return smem_optin(reinterpret_cast<const void*>(fn), bytes);
}

// Launch a ONE-WAVE kernel with programmatic stream serialization: the kernel
// releases its dependents at entry (`pdl_entry()`), so the next grid's launch
// latency overlaps this grid, and waits for the previous grid before its first
// global access.  Only for grids that are fully resident at once -- early
// dependents would take CTA slots from later waves.  SMMC_NO_PDL: A/B hook.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = getenv("SMMC_NO_PDL") ? 0 : 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_entry() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}
#endif

// Kernel launchers (defined in the kernel translation units).  They return
// a cudaError_t from cudaGetLastError() after the launch.
cudaError_t launch_exact(const Problem& p, cudaStream_t s);
struct FfmaPlan {
    int variant;       // index into the tile table
    int bm, bn, bk;    // CTA tile
    int threads;
    int splits;        // split-K factor (1 = no workspace)
    int kt_total;      // BK-wide tap blocks
    int kt_per_split;
    int tap_kind;      // 0 generic, 1: 3x3s1, 2: 1x1s1, 3: 7x7s2, 4: 11x11s4, 5: 5x5s1
    int cvec;          // tap-major K order
    int reduce_mode;   // 0 none, 1 last-arriver, 2 reduce kernel, 3 stream-K, 4 cluster DSMEM
    int groups;        // warp groups per CTA splitting the CTA's tap blocks (1 = off)
    int persist1x1;    // 1x1 layers: persistent block-stream kernel (conv_1x1.cu), BN = 64/128
    int stem;          // c_i <= kStemMaxCi layers: direct register-window kernel (conv_stem.cu) kind
    int64_t tiles;     // pixel tiles x channel tiles
    int tiles_n;
    int sk_ctas;       // stream-K grid
    int sk_iters;      // stream-K tap blocks per CTA
    int sk_maxseg;
    size_t ws_bytes;   // counter region + partial tiles
    size_t ws_counter_offset;   // counters (modes 1, 3, 5): always 0
    size_t ws_partial_offset;   // partial tiles: after the counter region
    int zero_counters;          // counters do not fit the resident region: zero per call
};
// Workspace layout of every split plan: [counter region][partial tiles].  The
// counter region (kCounterRegion bytes) is zero at rest: it must be zero-filled
// once when the workspace is allocated, and every kernel that uses counters
// re-arms them before it exits, so no per-call zeroing launch is needed.  Plans
// of other reduce modes never touch it, so one workspace may serve any
// sequence of layers.
constexpr size_t kCounterRegion = 64 * 1024;
// A plan choice outside the cost model: tile variant, splits (0 = stream-K),
// warp groups, reduce (5 = in-kernel), no_stem (tiled kernel for a stem layer).
// plan_force() pins one for the calling thread (the autotuner's candidate
// runs); plan_record() stores the measured winner of a geometry for the
// process, consulted by plan_ffma before the static tuning table.
struct PlanChoice {
    int variant, splits, groups, reduce, no_stem;
};
void plan_force(const PlanChoice* c);  // nullptr clears
void plan_record(const smmc_geom& g, const PlanChoice* c);  // nullptr forgets g
void plan_record_clear();
bool plan_recorded(const smmc_geom& g, PlanChoice* out);
// Candidate plans worth measuring for g (never the default plan itself).
int plan_candidates(const smmc_geom& g, int sm_count, PlanChoice* out, int max_out);
FfmaPlan plan_ffma(const smmc_geom& g, int sm_count);
FfmaPlan plan_ffma_gather(const smmc_geom& g, int sm_count);
cudaError_t launch_ffma(const Problem& p, const FfmaPlan& plan, cudaStream_t s);
bool conv1x1_eligible(const smmc_geom& g);
const char* conv1x1_describe(const smmc_geom& g, int sm_count);
constexpr int kStemMaxCi = 4;
constexpr size_t kStemMaxSmem = 200 * 1024;
int stem_kind(const smmc_geom& g, int sm_count = 148);
int stem_bn(const smmc_geom& g, int kind);
cudaError_t launch_stem(const Problem& p, int kind, cudaStream_t s);
int stem_describe(const smmc_geom& g, int kind, char* buf, size_t len);
cudaError_t launch_conv1x1(const Problem& p, int bn, int sm_count, cudaStream_t s);
int ffma_launches(const FfmaPlan& plan);
// bf16 tensor-core variant (conv_tc.cu)
struct TcPlan {
    int supported;
    int halo;          // flattened padded-pixel tiles, one halo box per channel block
    int halo_rows;
    int tw, th, nb;    // box kernel pixel tile
    int bn;            // output channels per tile (128, or 256 for the halo kernel)
    int persistent;    // halo: persistent warp-specialised kernel (always for bn = 256)
    int mt;            // persistent: 128-pixel M sub-tiles per tile sharing one B stage
    int64_t tiles_m;
    int tiles_n;
    int splits;        // persistent kernel split-K over channel blocks (few-tile layers)
    int cb_per_split;
};
TcPlan plan_tc(const smmc_geom& g);
size_t tc_workspace_bytes(const smmc_geom& g);
cudaError_t launch_tc_bf16(const uint16_t* x_nhwc, const uint16_t* w_tc, float* y, const smmc_geom& g,
                           cudaStream_t s, const char** why, float* ws = nullptr,
                           size_t ws_bytes = 0);
// split = 1: plain bf16; split = 3: [hi | lo | hi] input / [hi | hi | lo]
// weight channels of the fp32-accurate bf16x3 path (run as a 3*c_i bf16 conv)
cudaError_t launch_pack_input_nhwc(const float* x, uint16_t* out, const smmc_geom& g, cudaStream_t s,
                                   int split = 1);
cudaError_t launch_pack_weights_bf16(const float* w, uint16_t* out, const smmc_geom& g,
                                     cudaStream_t s, int split = 1);
cudaError_t launch_im2col_pack(const float* x, float* low, const smmc_geom& g, int oh, int ow,
                               cudaStream_t s);
cudaError_t launch_extract_slice(const float* x, const smmc_geom& g, int c, int j,
                                 float* buf, cudaStream_t s);
cudaError_t launch_scalar_matrix_fma(float alpha, const float* src, int64_t ss,
                                     float* dst, int64_t ds, int rows, int cols,
                                     cudaStream_t s);

// ----------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 4-byte cp.async with zero-fill: copies `src` when `valid`, else writes 0.
// This is the "zero packing" of the reference's slice extraction
// (smm.py:56-73) done by the copy engine path instead of a buffer pass.
__device__ __forceinline__ void cp_async4_zfill(uint32_t dst, const void* src, bool valid) {
    const int n = valid ? 4 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src), "r"(n));
}

// 16-byte cp.async (L2 only) with zero-fill of the tail past `bytes`.
__device__ __forceinline__ void cp_async16_zfill(uint32_t dst, const void* src, int bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(bytes));
}

// Blackwell packed FP32 FMA (SASS FFMA2): d = a*b + c on two lanes, each an
// IEEE round-to-nearest fma.  The scalar `a` is broadcast to both lanes;
// ptxas folds the {a, a} pair into FFMA2's .F32 scalar-operand form.
__device__ __forceinline__ uint64_t ffma2_bcast(float a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("{\n\t.reg .b64 t;\n\tmov.b64 t, {%1, %1};\n\tfma.rn.f32x2 %0, t, %2, %3;\n\t}"
        : "=l"(d)
        : "f"(a), "l"(b), "l"(c));
    return d;
}

__device__ __forceinline__ uint64_t pack2(float lo, float hi) {
    uint64_t d;
    asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
    return d;
}

__device__ __forceinline__ float2 unpack2(uint64_t v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

}  // namespace smmc
