/*
 * imconv.h -- C ABI of the B200 (sm_100a) blocked implicit-im2col convolution.
 *
 * This is the drop-in boundary for the reference's kernel plug-in surface
 * (/root/reference/pkg/src/sasim/_kernels/__init__.py).  Every entry point
 * takes plain pointers and sizes; device pointers are CUDA global-memory
 * addresses, `stream` is a cudaStream_t (NULL = legacy default stream).
 * All calls are stream-ordered, re-entrant and keep no global mutable state
 * other than a mutex-guarded, read-mostly cache of the driver entry point.
 *
 * Return codes: 0 on success, negative IMCONV_E* on argument errors,
 * positive values are cudaError_t / CUresult codes from the runtime/driver.
 * There is no CPU fallback: a missing GPU is an error (IMCONV_ENODEV).
 */
#ifndef IMCONV_H_
#define IMCONV_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IMCONV_ABI_VERSION 4

#if defined(__GNUC__)
#define IMCONV_API __attribute__((visibility("default")))
#else
#define IMCONV_API
#endif

/* error codes (negative) */
#define IMCONV_OK 0
#define IMCONV_EINVAL -1     /* invalid spec / null pointer / bad extent          */
#define IMCONV_EDTYPE -2     /* unsupported (in, out) dtype combination           */
#define IMCONV_EALIGN -3     /* pointer not 16-byte aligned                       */
#define IMCONV_ECHAN -4      /* C*elem or K*elem not a multiple of 16 bytes        */
#define IMCONV_ETMAP -5      /* cuTensorMapEncode* rejected the operand            */
#define IMCONV_ENODEV -6     /* no CUDA device / driver entry point unavailable    */
#define IMCONV_ERANGE -7     /* extent exceeds a TMA limit (corner/offset/dim)     */

/* element types */
#define IMCONV_BF16 0
#define IMCONV_F16 1
#define IMCONV_I8 2
#define IMCONV_F32 3
#define IMCONV_I32 4

/* scheduler order of the k-subtiles inside one output block
 * (blocksched.py:25-30, :83-99) */
#define IMCONV_ORDER_REUSE_AWARE 0  /* channel chunk outer, filter tap inner (default) */
#define IMCONV_ORDER_FILTER_MAJOR 1 /* filter tap outer, channel chunk inner          */

/* imconv_conv_args.flags */
#define IMCONV_FLAG_SINGLE_CTA 1  /* never use CTA pairs (cta_group::2)        */
#define IMCONV_FLAG_CTA_PAIR 2    /* use CTA pairs whenever the shape allows   */
#define IMCONV_FLAG_KSUB1 4       /* one k-subtile per pipeline stage (N<=128 default is 2) */
#define IMCONV_FLAG_MT1 8         /* one 128-pixel m-tile per CTA (N<=128 default is two)  */
#define IMCONV_FLAG_GATHER16 16   /* 16-byte pixels: generic kernel with cp.async tap gathers
                                     instead of the row-band (stride-phase plane) kernel     */
#define IMCONV_FLAG_NO_HALO 32    /* 128-byte pixels, stride 1, resident filter: generic
                                     per-tap kernel instead of the halo-tile kernel          */
#define IMCONV_FLAG_CHANNEL_LAST 64 /* channel-last BASELINE (bf16/fp16): reduction order
                                     k = (c, r, s), A gathered element by element -- the
                                     paper's CL lowering, for the stride contrast only        */
#define IMCONV_FLAG_STATIC_FILTER 128 /* the caller guarantees the filter is not written by any
                                     kernel still in flight on the stream (weights uploaded or
                                     converted before the step): the kernel's filter loads then
                                     start before its programmatic-launch wait, overlapping the
                                     previous conv's tail.  Inputs are always ordered.         */
#define IMCONV_FLAG_INDEPENDENT 256   /* the caller guarantees that no kernel still in flight on the
                                     stream writes this launch's input or filter, or reads or
                                     writes its output (independent convolutions, e.g. a sweep of
                                     layers over their own buffers): the kernel then never waits
                                     for the preceding grid -- its CTAs start computing on the SMs
                                     the previous conv's tail leaves idle.  Implies
                                     IMCONV_FLAG_STATIC_FILTER.  Stream order is otherwise kept:
                                     a later launch without the flag still waits for this one.  */
#define IMCONV_FLAG_BARRIER 512       /* every preceding grid completes before this launch lets the
                                     launches queued after it start (it waits, then triggers its
                                     dependents): the first launch of a batch of
                                     IMCONV_FLAG_INDEPENDENT launches, so that none of them can
                                     run ahead of the work queued before the batch.  Takes
                                     precedence over IMCONV_FLAG_INDEPENDENT / _STATIC_FILTER. */

/*
 * Forward convolution, NHWC input x HWCN filter -> NHWC output, stride,
 * zero padding (virtual) and dilation per axis.
 *
 * Replaces: sasim._kernels.conv2d_nhwc(x, w, sh, sw, ph, pw, dh, dw)
 *           (/root/reference/pkg/src/sasim/_kernels/__init__.py:37-46,
 *            _native.pyx:20-47, _fallback.py:17-42),
 *           and therefore core.direct_conv (core.py:194-208).
 * Semantics: y[n,p,q,k] = sum_{r,s,c} x[n, p*sh + r*dh - ph, q*sw + s*dw - pw, c]
 *                                   * w[r, s, c, k], out-of-range reads are 0.
 * The lowered (n*p*q, r*s*c) matrix is never materialised: operands are
 * produced by TMA im2col tensor maps straight into shared memory and
 * contracted by tcgen05.mma with the accumulator in tensor memory.
 *
 * Layout: x (n,h,w,c) contiguous, w (r,s,c,k) contiguous, y (n,p,q,k)
 * contiguous, caller-allocated (p, q from imconv_out_extent).
 * dtypes: in = BF16/F16 -> out = BF16/F16/F32 (fp32 accumulation);
 *         in = I8 -> out = I32 (int32 accumulation, bit-exact).
 * Requires c*elem % 16 == 0 and k*elem % 16 == 0 (the Python shim pads).
 * tile_n: 0 = auto, else 64/128/256 (output channels per CTA tile).
 * num_ctas: 0 = one persistent CTA per SM, else the grid size.  Above the SM
 *   count the grid is no longer co-resident, so the split-K tail (whose splits
 *   wait for each other) is turned off for such grids.
 * Stream capture: every call may be captured into a CUDA graph and the graph
 *   replayed any number of times (split-K counters are monotonic tickets, the
 *   partial-sum workspace is a stream-ordered allocation, i.e. a graph memory
 *   node).  A captured graph must not run concurrently with another replay of
 *   a graph captured from the same call.
 */
typedef struct imconv_conv_args {
    const void *x;
    const void *w;
    void *y;
    int32_t in_dtype;
    int32_t out_dtype;
    int64_t n, h, w_, c;   /* input extents (w_ = width) */
    int64_t k, r, s;       /* output channels, filter rows, filter cols */
    int32_t stride_h, stride_w;
    int32_t pad_h, pad_w;
    int32_t dil_h, dil_w;
    int32_t tile_n;
    int32_t num_ctas;
    int32_t order;         /* IMCONV_ORDER_* */
    int32_t flags;         /* IMCONV_FLAG_*: block-shape overrides (0 = automatic) */
} imconv_conv_args;

IMCONV_API int imconv_conv2d_nhwc(const imconv_conv_args *args, void *stream);

/* Output extent, core.py:89-95: (size + 2*pad - dil*(f-1) - 1)/stride + 1
 * (returns <= 0 when the effective filter exceeds the padded input). */
IMCONV_API int64_t imconv_out_extent(int64_t size, int64_t f, int64_t stride, int64_t pad, int64_t dil);

/*
 * C = A @ B, row-major A (m, kd) and B (kd, n), through the same tcgen05
 * kernel (a 1x1 stride-1 convolution over an (1, 1, m, kd) "image").
 * Replaces: core.gemm (core.py:211-218) on the explicit-lowering path
 * (simulator.py:527-532, lowering.py:98-122).
 */
IMCONV_API int imconv_gemm(const void *a, const void *b, void *c, int32_t in_dtype, int32_t out_dtype,
                int64_t m, int64_t kd, int64_t n, void *stream);

/*
 * One decomposed 1x1 tile's gather, (n*ho*wo, c) row-major, zero rows at
 * padding.  Replaces _kernels.tile_gather_nhwc (__init__.py:49-50,
 * _native.pyx:50-69) used by TileDescriptor.gather_matrix (lowering.py:88-95).
 * elem_bytes in {1,2,4,8}.
 */
IMCONV_API int imconv_tile_gather_nhwc(const void *x, void *out, int32_t elem_bytes,
                            int64_t n, int64_t h, int64_t w_, int64_t c,
                            int32_t r, int32_t s, int32_t stride_h, int32_t stride_w,
                            int32_t pad_h, int32_t pad_w, int32_t dil_h, int32_t dil_w,
                            int64_t ho, int64_t wo, void *stream);

/*
 * Explicit im2col, (n*ho*wo, hf*wf*c) row-major; column order channel-first
 * (r*wf + s)*c + ch or channel-last (ch*hf + r)*wf + s.
 * Replaces _kernels.im2col_nhwc (__init__.py:53-54, _native.pyx:72-99) and
 * lowering.im2col_explicit (lowering.py:98-110).  This is the K3 kernel of
 * the explicit-overhead measurement; it writes the lowered matrix to HBM.
 */
IMCONV_API int imconv_im2col_nhwc(const void *x, void *out, int32_t elem_bytes,
                       int64_t n, int64_t h, int64_t w_, int64_t c,
                       int32_t hf, int32_t wf, int32_t stride_h, int32_t stride_w,
                       int32_t pad_h, int32_t pad_w, int32_t dil_h, int32_t dil_w,
                       int32_t channel_first, void *stream);

/*
 * Zero-padding copy (outer, c, d) -> (outer, c_pad, d_pad), elem_bytes in
 * {1,2,4}; used by the Python shim to meet the 16-byte channel alignment
 * (exact: padded channels/filters are zero).  Device pointers.
 */
IMCONV_API int imconv_pad_copy(const void *src, void *dst, int32_t elem_bytes, int64_t outer,
                    int64_t c, int64_t d, int64_t c_pad, int64_t d_pad, void *stream);

/*
 * Fully-associative LRU replay of an int64 key stream (host memory, host
 * code).  Replaces _kernels.lru_simulate (__init__.py:57-59,
 * _native.pyx:102-149) behind blocksched.reuse_traffic (blocksched.py:131-151).
 */
IMCONV_API int imconv_lru_simulate(const int64_t *keys, int64_t count, int64_t capacity,
                        int64_t *hits, int64_t *misses);

/*
 * DRAM-traffic prediction for the generic kernel's actual B200 raster (host
 * code, no GPU needed).  Replays the schedule
 * imconv_conv2d_nhwc would run -- the same block shape, persistent round-robin
 * over `sms` CTAs (all CTAs advanced stage by stage in lockstep), the
 * k-subtile order of a->order, B-stationary and split-K decisions -- as a
 * stream of 128-byte line accesses (NHWC activations with batch-aware
 * addresses, HWCN filter, NHWC output), through a fully-associative
 * write-back LRU of l2_bytes.  Reads that miss are DRAM reads; dirty output
 * lines evicted during the kernel are DRAM writes; dirty lines still resident
 * at the end are reported separately (an ncu launch list with a flushed L2
 * counts them only when they are evicted later).  Extends the reference's
 * reuse_traffic model (blocksched.py:102-151, keys without the batch) to the
 * GPU schedule.  x/w/y pointers are ignored.
 */
typedef struct imconv_traffic {
    int64_t dram_read_bytes;       /* predicted DRAM reads */
    int64_t dram_write_bytes;      /* dirty lines evicted during the kernel */
    int64_t resident_dirty_bytes;  /* output bytes still in L2 at the end */
    int64_t line_requests;         /* 128-byte line accesses (A + B + y) */
    int64_t compulsory_read_bytes; /* distinct A and B lines touched x 128 */
    int64_t tiles;                 /* output blocks */
    int32_t bn, mt, grid, k_subtiles;
    int32_t kernel;                /* kernel imconv_conv2d_nhwc picks: 0 generic, 1 row-band, 2 halo,
                                      3 halo with a streamed filter
                                      (the replay always models the generic raster) */
} imconv_traffic;
IMCONV_API int imconv_predict_traffic(const imconv_conv_args *args, int64_t l2_bytes, int32_t sms,
                                      imconv_traffic *out);

/*
 * The launch imconv_conv2d_nhwc would issue for these arguments on a device
 * with `sms` SMs (host code, no GPU, pointers ignored): which kernel, and for
 * the generic kernel the planner's block shape, grid, CTA pairs, B-stationary
 * and split-K decisions.  Introspection for tests and tools (the branches the
 * benchmarked batch sizes select); same return codes as imconv_conv2d_nhwc's
 * argument checks.
 */
typedef struct imconv_plan_info {
    int32_t kernel;      /* 0 generic, 1 row-band, 2 halo, 3 halo with a streamed filter */
    int32_t grid;        /* generic kernel: CTAs launched */
    int32_t bn;          /* output channels per block */
    int32_t mt;          /* 128-row m-tiles per CTA block */
    int32_t ksub;        /* k-subtiles per pipeline stage */
    int32_t cta_pair;    /* 1: cta_group::2 CTA pairs (256-row blocks) */
    int32_t b_resident;  /* 1: each CTA loads its filter slice once */
    int32_t sk_split;    /* split-K ways of the tail tiles (1 = no split) */
    int64_t tiles;       /* output blocks */
    int64_t sk_tail;     /* tail blocks whose k-loop is split (sk_mode 1) or streamed (sk_mode 2) */
    int32_t sk_mode;     /* 0 whole blocks, 1 split-K tail, 2 stream-K over the last two waves */
} imconv_plan_info;
IMCONV_API int imconv_plan(const imconv_conv_args *args, int32_t sms, imconv_plan_info *out);

/* Device / build introspection (no compute). */
IMCONV_API int imconv_abi_version(void);
IMCONV_API int imconv_device_sm_count(int32_t *sm_count);
IMCONV_API const char *imconv_strerror(int code);

/* Number of kernel launches issued by this library on the calling thread
 * since the last reset (instrumentation for bench.py's gpu_launches). */
IMCONV_API int64_t imconv_launch_count(void);
IMCONV_API void imconv_reset_launch_count(void);

/* Instrumentation: when set (device buffer of >= 8 * num_ctas int64), the
 * next launches record per-CTA role cycles and blocking-wait cycles into it.
 * NULL (the default) disables recording. */
IMCONV_API void imconv_debug_set_buffer(void *dev_buf);
/* Instrumentation only: bit flags that switch off pipeline roles of the
 * specialised kernels (results are then WRONG); 0 = normal operation. */
IMCONV_API void imconv_debug_set_flags(int flags);

#ifdef __cplusplus
}
#endif

#endif /* IMCONV_H_ */
