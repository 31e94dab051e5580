/*
 * smmc.h — C ABI of the B200 (sm_100a) SMM-Conv forward-convolution path.
 *
 * This is the drop-in boundary for the one hot path of arxiv 2411.15659 as
 * packaged by the reference (`smmconv`, /root/reference/pkg): channels-first
 * (NCHW) fp32 forward convolution by scalar-matrix accumulation with zero
 * packing.  The reference has no C ABI of its own — its entry points are the
 * Python functions cited beside each symbol below — so these are the symbols a
 * ctypes / cffi binding of that interface binds.
 *
 * Conventions
 *  - Plain pointers and sizes only; no framework types.
 *  - Device entry points take caller-owned DEVICE pointers, allocate nothing,
 *    and are asynchronous on the caller's stream (`stream` is a cudaStream_t;
 *    NULL = the legacy default stream).
 *  - `*_host` entry points take HOST pointers, do H2D + kernel(s) + D2H on an
 *    internal per-device stream and return after the result is in `y`
 *    (the reference's numpy semantics: a freshly computed output).
 *  - Every function returns an int status (SMMC_OK == 0); on failure
 *    smmc_last_error() returns a thread-local message.  No CPU fallback exists:
 *    without a usable GPU the status is SMMC_ENODEVICE.
 *  - Re-entrant: no global mutable state except the per-device host-staging
 *    pool (mutex-protected) and an atomic launch counter.
 *
 * Tensor layouts (all C-contiguous)
 *  x      : float32 (n, c_i, h, w)                       — NCHW input
 *  w_smm  : float32 (c_i, k_w, k_h, c_o)                 — the reference's repacked
 *           "SMM access order" (smm.py:164-167); c_o innermost
 *  y      : float32 (n, c_o, out_h, out_w)                — NCHW output
 *  out_h  = (h + 2*p_h - k_h) / s_h + 1, out_w likewise   (geometry.py:60-66)
 */
#ifndef SMMC_H_
#define SMMC_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SMMC_API __attribute__((visibility("default")))
#else
#define SMMC_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define SMMC_ABI_VERSION 1

/* Status codes; the Python layer maps them to the reference's exception types. */
enum smmc_status {
    SMMC_OK = 0,
    SMMC_EGEOM = 1,        /* -> GeometryError          (geometry.py:32-50)   */
    SMMC_ESHAPE = 2,       /* -> ShapeMismatchError     (validation.py:25-34) */
    SMMC_EUNSUPPORTED = 3, /* -> BackendUnsupportedError (errors.py)          */
    SMMC_EWORKSPACE = 4,   /* -> ValueError: caller workspace too small       */
    SMMC_ECUDA = 5,        /* -> DeviceError (RuntimeError)                    */
    SMMC_ENODEVICE = 6,    /* -> DeviceError: no CUDA device / driver          */
    SMMC_EINDEX = 7        /* -> IndexError             (smm.py:196-199, 211)  */
};

/* Kernel variants. */
enum smmc_mode {
    SMMC_MODE_FFMA = 0,  /* product: register-tiled fp32 FFMA, any order; ~1e-6 rel */
    SMMC_MODE_EXACT = 1  /* bitwise-equal to smm_conv_single: (c, j, k) order,
                            separately rounded mul then add (smm.py:84-114)      */
};

/* One convolution problem: the reference's ConvGeometry (geometry.py:19-30)
 * plus a batch size n (the Conv2D.transform batch, estimator.py:112-125). */
typedef struct smmc_geom {
    int32_t n;    /* samples                  */
    int32_t c_i;  /* in_channels              */
    int32_t h;    /* in_h                     */
    int32_t w;    /* in_w                     */
    int32_t c_o;  /* out_channels             */
    int32_t k_h;  /* kernel rows              */
    int32_t k_w;  /* kernel columns           */
    int32_t s_h;  /* stride_h                 */
    int32_t s_w;  /* stride_w                 */
    int32_t p_h;  /* pad_h                    */
    int32_t p_w;  /* pad_w                    */
} smmc_geom;

/* ABI version (SMMC_ABI_VERSION). */
SMMC_API int smmc_abi_version(void);

/* Thread-local message for the last non-OK status on this thread. */
SMMC_API const char* smmc_last_error(void);

/* Validate a geometry (ConvGeometry.__post_init__, geometry.py:32-50) and
 * return the output size.  SMMC_EGEOM on any rejection. */
SMMC_API int smmc_geom_check(const smmc_geom* g, int32_t* out_h, int32_t* out_w);

/* Device scratch (bytes) smmc_conv2d_fwd_f32 needs for this problem/mode:
 * 0 for the fused kernels, the split-K partial planes otherwise.
 * GPU analogue of smm_workspace_elements (smm.py:176-180). */
SMMC_API size_t smmc_workspace_bytes(const smmc_geom* g, int mode);

/* Forward convolution, device pointers, async on `stream`.
 * Replaces the compute of smm_conv_single (smm.py:226-251),
 * smm_conv_parallel (smm.py:254-306) and the per-sample loop of
 * Conv2D.transform (estimator.py:112-125) with one batched launch.
 * `workspace` must hold smmc_workspace_bytes(g, mode) bytes (may be NULL if 0),
 * 256-byte aligned, and be ZERO-FILLED before its first use: its leading
 * 64 KB counter region is zero at rest (every launch that uses split-K
 * counters re-arms them before it exits), so one workspace serves any
 * sequence of layers on one stream without a per-call memset.  Alignment: w_smm 16 bytes; y 16 bytes when h'*w' % 4 == 0
 * (float4 stores), else 4; x 4 bytes (any sample or channel offset works). */
SMMC_API int smmc_conv2d_fwd_f32(const float* x, const float* w_smm, float* y,
                        const smmc_geom* g, int mode, void* workspace,
                        size_t workspace_bytes, void* stream);

/* Same, HOST pointers: H2D(x, w_smm) + conv + D2H(y), synchronous.
 * The numpy drop-in for smm_conv_single / smm_conv_parallel. */
SMMC_API int smmc_conv2d_fwd_f32_host(const float* x, const float* w_smm, float* y,
                             const smmc_geom* g, int mode, int device);

/* Zero-packing slice (smm.py:56-73 / extract_slice smm.py:190-203), device:
 * buf[r, t] = x[c, r - p_h, j + t*s_w - p_w] (0 outside), buf is
 * (h + 2*p_h) x out_w.  Uses sample 0 of x; g->n is ignored. */
SMMC_API int smmc_extract_slice_f32(const float* x, const smmc_geom* g, int32_t c,
                           int32_t j, float* buf, void* stream);

/* dst[r, t] += alpha * src[r, t] with one rounded multiply then one rounded
 * add (scalar_matrix_fma, smm.py:76-81, 217-223); row strides in elements. */
SMMC_API int smmc_scalar_matrix_fma_f32(float alpha, const float* src,
                               int64_t src_row_stride, float* dst,
                               int64_t dst_row_stride, int32_t rows,
                               int32_t cols, void* stream);

/* Host-pointer versions of the two helpers above (synchronous). */
SMMC_API int smmc_extract_slice_f32_host(const float* x, const smmc_geom* g, int32_t c,
                                int32_t j, float* buf, int device);
SMMC_API int smmc_scalar_matrix_fma_f32_host(float alpha, const float* src,
                                    int64_t src_row_stride, float* dst,
                                    int64_t dst_row_stride, int32_t rows,
                                    int32_t cols, int device);

/* ---------------------------------------------------------------------------
 * Separately labelled tensor-core variant (BASELINE config 5): bf16 inputs,
 * fp32 accumulation in TMEM (tcgen05), fp32 NCHW output.  Parity bar
 * 2e-2 * max|ref| against the fp32 oracle.  Stride 1, c_i % 8 == 0.
 * Replaces the same compute as smmc_conv2d_fwd_f32 (smm.py:226-306), with the
 * input in channels-last bf16 and the weights packed per tap.
 * ------------------------------------------------------------------------- */

/* 1 if smmc_conv2d_fwd_bf16_tc supports this geometry, else 0. */
SMMC_API int smmc_tc_supported(const smmc_geom* g);

/* x fp32 NCHW (n, c_i, h, w) -> x_nhwc bf16 ZERO-PADDED channels-last
 * (n, h + 2*p_h, w + 2*p_w, c_i): the reference's zero-packed slice buffer
 * (smm.py:56-73) materialised for all channels.  Device, async. */
SMMC_API int smmc_pack_input_bf16_nhwc(const float* x, uint16_t* x_nhwc, const smmc_geom* g,
                                       void* stream);

/* w_smm fp32 (c_i, k_w, k_h, c_o) -> w_tc bf16 (k_w*k_h, c_o, c_i), tap = j*k_h + k
 * (the tensor-core analogue of repack_weights, smm.py:164-167). */
SMMC_API int smmc_pack_weights_bf16(const float* w_smm, uint16_t* w_tc, const smmc_geom* g,
                                    void* stream);

/* y fp32 NCHW = conv(x_nhwc, w_tc), x_nhwc as written by
 * smmc_pack_input_bf16_nhwc (zero-padded): tcgen05 implicit GEMM over the
 * k_h*k_w shifted windows (each a constant row offset of one TMA halo tile).
 * Device pointers, async. */
SMMC_API int smmc_conv2d_fwd_bf16_tc(const uint16_t* x_nhwc, const uint16_t* w_tc, float* y,
                                     const smmc_geom* g, void* stream);

/* Device scratch (bytes) of the tensor-core kernels' split-K (layers with
 * fewer tiles than SMs split their channel blocks across CTAs and sum fp32
 * partial planes in split order); 0 when the plan does not split.  split3 = 1
 * for the bf16x3 path below (its 3*c_i channels). */
SMMC_API size_t smmc_tc_workspace_bytes(const smmc_geom* g, int split3);

/* smmc_conv2d_fwd_bf16_tc with a caller workspace (enables split-K; with
 * ws = NULL or too small the kernel runs unsplit). */
SMMC_API int smmc_conv2d_fwd_bf16_tc_ws(const uint16_t* x_nhwc, const uint16_t* w_tc, float* y,
                                        const smmc_geom* g, void* ws, size_t ws_bytes,
                                        void* stream);

/* ---------------------------------------------------------------------------
 * fp32-accurate tensor-core path ("bf16x3", split bf16): x = x_hi + x_lo and
 * w = w_hi + w_lo with hi = bf16(v), lo = bf16(v - hi); y = x_hi*w_hi +
 * x_lo*w_hi + x_hi*w_lo accumulated in fp32 TMEM — the bf16 tcgen05 conv
 * above run over 3*c_i channels ([hi|lo|hi] input, [hi|hi|lo] weights).
 * Parity bar: the fp32 one, 1e-4 * max|ref| (dropped x_lo*w_lo ~ 2^-16).
 * Same geometry support as smmc_tc_supported.  Device pointers, async.
 * ------------------------------------------------------------------------- */

/* x fp32 NCHW -> x3 bf16 zero-padded NHWC (n, h + 2*p_h, w + 2*p_w, 3*c_i). */
SMMC_API int smmc_pack_input_bf16x3_nhwc(const float* x, uint16_t* x3, const smmc_geom* g,
                                         void* stream);

/* w_smm fp32 (c_i, k_w, k_h, c_o) -> w3 bf16 (k_w*k_h, c_o, 3*c_i). */
SMMC_API int smmc_pack_weights_bf16x3(const float* w_smm, uint16_t* w3, const smmc_geom* g,
                                      void* stream);

/* y fp32 NCHW = conv(x, w) from the split operands above; workspace as
 * smmc_tc_workspace_bytes(g, 1) (NULL: unsplit). */
SMMC_API int smmc_conv2d_fwd_bf16x3_tc(const uint16_t* x3, const uint16_t* w3, float* y,
                                       const smmc_geom* g, void* ws, size_t ws_bytes,
                                       void* stream);

/* GPU im2col comparator (the paper's baseline): the explicit
 * lowered matrix of im2col_pack (im2col.py:22-71), per sample
 * [c_i*k_h*k_w][out_h*out_w], row (c*k_h + k)*k_w + j, zero-filled padding.
 * `lowered` holds n*c_i*k_h*k_w*out_h*out_w floats — the scratch SMM avoids. */
SMMC_API size_t smmc_im2col_bytes(const smmc_geom* g);
SMMC_API int smmc_im2col_pack_f32(const float* x, float* lowered, const smmc_geom* g, void* stream);

/* Number of kernels smmc_conv2d_fwd_f32 launches for this problem/mode. */
SMMC_API int smmc_plan_launches(const smmc_geom* g, int mode);

/* Per-shape autotuning (no counterpart in the reference: its numba kernel has
 * one schedule, smm.py:254-306).  smmc_autotune_f32 times the candidate kernel
 * plans of geometry g (its n included) on the current device -- in-kernel-split
 * grids sized to the SM count, stream-K, the tiled kernel for stem / 1x1 layers
 * -- with scratch operands it allocates itself, `iters` launches per candidate,
 * and keeps the fastest for the rest of the process when it beats the default
 * plan by more than 5 %: later smmc_conv2d_fwd_f32 / smmc_workspace_bytes /
 * smmc_plan_describe calls for the same geometry use it (call it BEFORE sizing a
 * workspace or creating a layer).  Every candidate is one of the parity-tested
 * plan kinds; results stay within the fp32 bar and deterministic for a fixed
 * choice.  `report` (optional) receives a one-line summary.
 * smmc_autotune_clear forgets every recorded choice. */
SMMC_API int smmc_autotune_f32(const smmc_geom* g, int iters, char* report, size_t report_len);
SMMC_API int smmc_autotune_clear(void);

/* Short human-readable description of the kernel plan (tile, split-K). */
SMMC_API int smmc_plan_describe(const smmc_geom* g, int mode, char* buf, size_t len);

/* Same for the bf16 tensor-core variant (tile shape, halo/box, persistence). */
SMMC_API int smmc_tc_plan_describe(const smmc_geom* g, char* buf, size_t len);

/* ---- Fitted layers (the GPU form of Conv2D.fit / transform,
 * estimator.py:71-125): the repacked weights are uploaded once at fit time
 * and stay in HBM; each forward moves only the input batch up and the output
 * down (the same chunked H2D / conv / D2H pipeline as the _host entry).
 * Synchronous, re-entrant per device (staging pool mutex). */
typedef struct smmc_layer smmc_layer;
SMMC_API int smmc_layer_create(const float* w_smm, const smmc_geom* g, int device,
                               smmc_layer** out);
SMMC_API int smmc_layer_forward_host(smmc_layer* layer, const float* x, float* y, int n,
                                     int mode);
/* Asynchronous forward of a fitted layer on host buffers: enqueues the
 * H2D / conv / D2H pipeline on the layer's OWN staging buffers and streams
 * (created on first use) and returns at once, so calls on different layers
 * overlap (one layer's output copy-back with the next layer's upload and
 * conv).  x and y must stay valid (and y unread) until smmc_layer_wait;
 * page-locked buffers make the copies truly asynchronous.  A second async
 * call on the same layer first waits for the previous one. */
SMMC_API int smmc_layer_forward_host_async(smmc_layer* layer, const float* x, float* y, int n,
                                           int mode);
SMMC_API int smmc_layer_wait(smmc_layer* layer);
SMMC_API int smmc_layer_destroy(smmc_layer* layer);

/* ---- Fused output-channel-shard all-gather.
 * Rank r of P holds the full input and W_smm[..., co_base:co_base+c_o] as a
 * compact (c_i, k_w, k_h, c_o) slice (g_local->c_o = its channel count).  The
 * conv epilogue stores its channels straight into every replica
 * y_out[0..n_out) of the full (N, co_total, h', w') output — this rank's own
 * buffer and the peers' buffers mapped over NVLink with smmc_ipc_open — so no
 * gather buffer, collective payload or permute copy exists.  The caller orders
 * completion (a stream-ordered barrier after the call, e.g. a 1-element NCCL
 * all-reduce) before peers read.  Replaces the reference's Algorithm-2 channel
 * partition + join (smm.py:273-306) lifted to devices.  ffma mode. */
#define SMMC_MAX_OUT 8
#define SMMC_IPC_HANDLE_BYTES 64
SMMC_API int smmc_conv2d_fwd_f32_gather(const float* x, const float* w_slice, float* const* y_out,
                                        int n_out, const smmc_geom* g_local, int co_base,
                                        int co_total, void* workspace, size_t workspace_bytes,
                                        void* stream);

/* Page-locked host memory for the *_host entries' buffers: 2 MB-aligned
 * anonymous pages registered with cudaHostRegister (measured 55 GB/s H2D on
 * B200 vs 29-36 GB/s for cudaHostAlloc memory on the same host). */
SMMC_API int smmc_host_alloc_pinned(size_t bytes, void** ptr);
SMMC_API int smmc_host_free_pinned(void* ptr);

/* Workspace the gather needs (its plan always places through the reduce pass). */
SMMC_API size_t smmc_gather_workspace_bytes(const smmc_geom* g_local);

/* CUDA IPC for the gather: handle (SMMC_IPC_HANDLE_BYTES) + byte offset of an
 * interior device pointer, and open/close of a peer's pointer in this process. */
SMMC_API int smmc_ipc_handle(const void* dev_ptr, void* handle, size_t* offset);
SMMC_API int smmc_ipc_open(const void* handle, size_t offset, void** dev_ptr);
SMMC_API int smmc_ipc_close(void* dev_ptr, size_t offset);

/* Total kernels this library has launched in this process (atomic). */
SMMC_API uint64_t smmc_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* SMMC_H_ */
