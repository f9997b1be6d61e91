// imconv_api.cu -- C ABI (include/imconv.h) over the sm_100a kernels.
//
// Host-side responsibilities: validate the spec (the reference validates in
// ConvSpec.__post_init__, core.py:72-87, and _as_nhwc/_as_filter_hwcn,
// core.py:178-191), encode the TMA tensor maps (im2col map for the NHWC
// activations, tiled map for the HWCN filter), choose the block shape, and
// launch the persistent kernel on the caller's stream.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <mutex>
#include <type_traits>

#include "../../include/imconv.h"
#include "aux_kernels.cuh"
#include "conv_kernel.cuh"
#include "conv_halo.cuh"
#include "conv_halo_stream.cuh"
#include "conv_rowband.cuh"
#include "lru.h"

namespace imconv {
namespace {

thread_local int64_t g_launches = 0;
long long *g_debug_buf = nullptr;  // instrumentation target (imconv_debug_set_buffer)
int g_debug_flags = 0;
// imconv_debug_set_flags layout: bits 0-7 kernel instrumentation switches (instrumented
// build), bits 8-15 row-band rows-per-stage override, bits 16+ host-side A/B switches
constexpr int kDbgNoTiledA = 1 << 16;     // 1x1 stride-1 layers keep the im2col A map
constexpr int kDbgNoBResident = 1 << 17;  // never load the filter slice once per CTA
constexpr int kDbgNoPdl = 1 << 18;        // launch without programmatic stream serialization
constexpr int kDbgNoSplitK = 1 << 19;     // never split the tail wave's k-loops
constexpr int kDbgPlanePitch128 = 1 << 20;  // row-band planes at a 128-byte-multiple pitch (A/B)
constexpr int kDbgNoAutoPair = 1 << 21;   // never pick CTA pairs automatically
constexpr int kDbgNoRowPairs = 1 << 22;   // row-band kernel: no N = 128 MMAs over two output rows
constexpr int kDbgNoStemSpec = 1 << 23;   // row-band kernel: no compile-time stem instantiation
constexpr int kDbgThrNoPair = 1 << 24;    // throughput mode: sub-wave layers keep single CTAs
constexpr int kDbgNoHaloStack = 1 << 25;  // halo kernel: one sub-block per block (no shared N = 128 taps)
constexpr int kDbgNoHaloStream = 1 << 26; // multi-chunk stride-1 layers keep the generic kernel
constexpr int kDbgNo1x1Stream = 1 << 27;  // output-heavy 1x1 layers keep the B-stationary layout
constexpr int kDbgNoPairSplit = 1 << 28;  // CTA pairs never split the tail wave's k-loops
constexpr int kDbgStreamK = 1 << 29;      // stream-K the last two waves (measured slower: opt-in, see plan_generic_bn)
constexpr int kDbgHaloStreamSingle = 1 << 30;  // halo and halo-stream kernels keep single CTAs (A/B of the pairs)

// Split-K ticket counters (conv_kernel.cuh sk_arrive): one per tail tile, never
// cleared (they only grow, in steps that leave a multiple of kSkRound between
// launches).  Each launch takes one of kSkSlices slices round-robin, so launches
// in flight at the same time on different streams do not share a counter.  The
// counters are allocated and zeroed on first use of a device; that first use may
// happen while the caller's stream is being captured into a CUDA graph, so the
// allocation runs in relaxed capture mode and the zeroing on a private stream
// that is not part of any capture.
std::mutex g_sk_mutex;
unsigned long long *g_sk_counters[64] = {};
std::atomic<unsigned long long> g_sk_slice{0};
constexpr int kSkSlices = 256, kSkSliceLen = 256;

unsigned long long *sk_counters(int dev) {
    std::lock_guard<std::mutex> lock(g_sk_mutex);
    if (dev < 0 || dev >= 64) return nullptr;
    if (!g_sk_counters[dev]) {
        cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
        cudaThreadExchangeStreamCaptureMode(&mode);
        void *ptr = nullptr;
        cudaStream_t zs = nullptr;
        const size_t bytes = sizeof(unsigned long long) * kSkSlices * kSkSliceLen;
        bool ok = cudaMalloc(&ptr, bytes) == cudaSuccess &&
                  cudaStreamCreateWithFlags(&zs, cudaStreamNonBlocking) == cudaSuccess &&
                  cudaMemsetAsync(ptr, 0, bytes, zs) == cudaSuccess && cudaStreamSynchronize(zs) == cudaSuccess;
        if (zs) cudaStreamDestroy(zs);
        if (!ok && ptr) cudaFree(ptr);
        cudaThreadExchangeStreamCaptureMode(&mode);  // restore the caller's mode
        if (!ok) {
            cudaGetLastError();
            return nullptr;
        }
        g_sk_counters[dev] = static_cast<unsigned long long *>(ptr);
    }
    return g_sk_counters[dev];
}

// cudaFuncSetAttribute is per device: each kernel instantiation keeps a bitmask of
// the devices it has been configured on (a process may drive several GPUs).
template <typename Kern>
cudaError_t ensure_attrs(std::atomic<unsigned long long> &done, Kern kern, int smem, bool cluster) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess && cluster) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

std::mutex g_mu;
PFN_cuTensorMapEncodeIm2col_v12000 g_encode_im2col = nullptr;
PFN_cuTensorMapEncodeTiled_v12000 g_encode_tiled = nullptr;
int g_driver_version = 0;
int g_sm_count[64] = {0};

int load_driver_entry_points() {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_encode_im2col && g_encode_tiled) return 0;
    cudaDriverEntryPointQueryResult q1, q2;
    void *f1 = nullptr, *f2 = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f1, cudaEnableDefault, &q1) != cudaSuccess ||
        q1 != cudaDriverEntryPointSuccess || f1 == nullptr)
        return IMCONV_ENODEV;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f2, cudaEnableDefault, &q2) != cudaSuccess ||
        q2 != cudaDriverEntryPointSuccess || f2 == nullptr)
        return IMCONV_ENODEV;
    cudaDriverGetVersion(&g_driver_version);
    g_encode_im2col = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(f1);
    g_encode_tiled = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f2);
    return 0;
}

int sm_count_for_current_device(int *out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return IMCONV_ENODEV;
    if (dev >= 0 && dev < 64 && g_sm_count[dev] > 0) {
        *out = g_sm_count[dev];
        return 0;
    }
    int n = 0;
    e = cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess || n <= 0) return IMCONV_ENODEV;
    if (dev >= 0 && dev < 64) g_sm_count[dev] = n;
    *out = n;
    return 0;
}

inline int64_t out_extent(int64_t size, int64_t f, int64_t stride, int64_t pad, int64_t dil) {
    return (size + 2 * pad - dil * (f - 1) - 1) / stride + 1;
}

inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

CUtensorMapDataType tmap_dtype(int in_dtype) {
    switch (in_dtype) {
        case IMCONV_BF16: return CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
        case IMCONV_F16: return CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
        default: return CU_TENSOR_MAP_DATA_TYPE_UINT8;  // int8 bytes; zero fill is 0 either way
    }
}

int elem_bytes(int in_dtype) { return in_dtype == IMCONV_I8 ? 1 : 2; }

// Programmatic-launch wait mode of the kernels' b_early parameter: 0 every role waits for the
// preceding grid, 1 the filter loads start before the wait (IMCONV_FLAG_STATIC_FILTER), 2 no role
// waits (IMCONV_FLAG_INDEPENDENT: nothing in flight touches this launch's buffers), 3 the kernel
// waits before it triggers its dependents (IMCONV_FLAG_BARRIER: head of an independent batch).
int early_mode(int flags) {
    if (flags & IMCONV_FLAG_BARRIER) return 3;  // wait for every preceding grid, then trigger
    if (flags & IMCONV_FLAG_INDEPENDENT) return 2;
    return (flags & IMCONV_FLAG_STATIC_FILTER) ? 1 : 0;
}

// Conv kernels are launched with programmatic stream serialization (PDL): the
// next kernel's CTAs may start their setup (barrier init, TMEM allocation,
// tensor-map prefetch) on SMs this kernel has released, and block in
// griddepcontrol.wait before touching global memory.  Debug flag kDbgNoPdl turns
// it off (A/B measurements).
template <typename Kern, typename... Args>
cudaError_t launch_pdl(Kern kern, int grid, int block, int smem, cudaStream_t st, int cluster, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(static_cast<unsigned>(block));
    cfg.dynamicSmemBytes = static_cast<size_t>(smem);
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (!(g_debug_flags & kDbgNoPdl)) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (cluster > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = static_cast<unsigned>(cluster);
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = static_cast<unsigned>(na);
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <int ELEM, int OUT, int BN, int STAGES, int KSUB, int MT, int CG = 1>
int launch_conv(const CUtensorMap &ta, const CUtensorMap &tb, const CUtensorMap &ty, const ConvParams &p, int grid,
                cudaStream_t st) {
    using Cfg = ConvCfg<ELEM, OUT, BN, STAGES, KSUB, MT, CG>;
    auto kern = conv_fwd_kernel<ELEM, OUT, BN, STAGES, KSUB, MT, CG>;
    static std::atomic<unsigned long long> attr_done{0};
    const cudaError_t attr_err = ensure_attrs(attr_done, kern, Cfg::kSmemBytes, CG == 2);
    if (attr_err != cudaSuccess) return static_cast<int>(attr_err);
    const int g = CG == 1 ? grid : (grid & ~1);
    cudaError_t le = launch_pdl(kern, g, kThreadsGeneric, Cfg::kSmemBytes, st, CG, ta, tb, ty, p);
    if (le != cudaSuccess) return static_cast<int>(le);
    ++g_launches;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : static_cast<int>(e);
}

// CTA pairs (cta_group::2): one m-tile, one k-subtile per stage, half of B per CTA.
template <int ELEM, int OUT>
int dispatch_bn_pair(int bn, const CUtensorMap &ta, const CUtensorMap &tb, const CUtensorMap &ty,
                     const ConvParams &p, int grid, cudaStream_t st) {
    if constexpr (ELEM == ELEM_I8) {
        if (bn == 256) return launch_conv<ELEM, OUT, 256, 6, 1, 1, 2>(ta, tb, ty, p, grid, st);
    } else {
        if (bn == 128) return launch_conv<ELEM, OUT, 128, 8, 1, 1, 2>(ta, tb, ty, p, grid, st);
        if (bn == 256) return launch_conv<ELEM, OUT, 256, 6, 1, 1, 2>(ta, tb, ty, p, grid, st);
    }
    return IMCONV_EINVAL;
}

// Block shape -> pipeline depth that fits the shared memory:
//   variant 0 (default N <= 128): MT = 2 m-tiles per CTA, 1 k-subtile per stage
//   variant 1 (IMCONV_FLAG_MT1):  MT = 1, KSUB = 2
//   variant 2 (IMCONV_FLAG_KSUB1): MT = 1, KSUB = 1
// N = 256 always runs MT = 1, KSUB = 1 (4 x 128-cycle MMAs per stage).
template <int ELEM, int OUT>
int dispatch_bn(int bn, int variant, const CUtensorMap &ta, const CUtensorMap &tb, const CUtensorMap &ty,
                const ConvParams &p, int grid, cudaStream_t st) {
    if constexpr (ELEM == ELEM_I8) {
        if (bn == 128) {
            if (variant == 0) return launch_conv<ELEM, OUT, 128, 4, 1, 2>(ta, tb, ty, p, grid, st);
            if (variant == 1) return launch_conv<ELEM, OUT, 128, 3, 2, 1>(ta, tb, ty, p, grid, st);
            return launch_conv<ELEM, OUT, 128, 6, 1, 1>(ta, tb, ty, p, grid, st);
        }
        if (bn == 256) return launch_conv<ELEM, OUT, 256, 4, 1, 1>(ta, tb, ty, p, grid, st);
    } else {
        if (bn == 64) {
            if (variant == 0) return launch_conv<ELEM, OUT, 64, 4, 1, 2>(ta, tb, ty, p, grid, st);
            if (variant == 1) return launch_conv<ELEM, OUT, 64, 4, 2, 1>(ta, tb, ty, p, grid, st);
            return launch_conv<ELEM, OUT, 64, 8, 1, 1>(ta, tb, ty, p, grid, st);
        }
        if (bn == 128) {
            if (variant == 0) return launch_conv<ELEM, OUT, 128, 4, 1, 2>(ta, tb, ty, p, grid, st);
            if (variant == 1) return launch_conv<ELEM, OUT, 128, 3, 2, 1>(ta, tb, ty, p, grid, st);
            return launch_conv<ELEM, OUT, 128, 6, 1, 1>(ta, tb, ty, p, grid, st);
        }
        if (bn == 256) return launch_conv<ELEM, OUT, 256, 4, 1, 1>(ta, tb, ty, p, grid, st);
    }
    return IMCONV_EINVAL;
}

int pick_bn(int in_dtype, int64_t k, int requested) {
    const int nc = in_dtype == IMCONV_I8 ? 128 : 64;
    if (requested != 0) {
        if (requested % nc != 0 || requested > 256 || requested < nc) return -1;
        return requested;
    }
    int64_t bn = ((k + nc - 1) / nc) * nc;
    if (bn > 256) bn = 256;
    return static_cast<int>(bn);
}

constexpr int kMaxDynSmem = 227 * 1024;

inline int floordiv(int a, int b) { return (a >= 0) ? a / b : -((-a + b - 1) / b); }

template <int ELEM, int OUT, int BN, int TP, int NP, int STEM = 0>
int launch_rowband(const CUtensorMap &tw, const CUtensorMap &ty, const RowbandParams &p, int smem, int grid,
                   cudaStream_t st) {
    auto kern = conv_rowband_kernel<ELEM, OUT, BN, TP, NP, STEM>;
    static std::atomic<unsigned long long> attr_done{0};
    const cudaError_t attr_err = ensure_attrs(attr_done, kern, kMaxDynSmem, false);
    if (attr_err != cudaSuccess) return static_cast<int>(attr_err);
    cudaError_t le = launch_pdl(kern, grid, kThreadsRowband, smem, st, 1, tw, ty, p);
    if (le != cudaSuccess) return static_cast<int>(le);
    ++g_launches;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : static_cast<int>(e);
}

constexpr int kNotApplicable = -1000;  // internal: layer does not qualify for a specialised path

template <int ELEM, int OUT, int BN, int HB = 1, int CG = 1>
int launch_halo(const CUtensorMap &ta, const CUtensorMap &tb, const CUtensorMap &ty, const CUtensorMap &tb64,
                const HaloParams &p, int smem, int grid, cudaStream_t st) {
    auto kern = conv_halo_kernel<ELEM, OUT, BN, HB, CG>;
    static std::atomic<unsigned long long> attr_done{0};
    const cudaError_t attr_err = ensure_attrs(attr_done, kern, kMaxDynSmem, CG == 2);
    if (attr_err != cudaSuccess) return static_cast<int>(attr_err);
    cudaError_t le = launch_pdl(kern, grid, kThreadsGeneric, smem, st, CG, ta, tb, ty, tb64, p);
    if (le != cudaSuccess) return static_cast<int>(le);
    ++g_launches;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : static_cast<int>(e);
}

// Halo-tile path (conv_halo.cuh): stride 1, one 128-byte swizzle row per pixel
// (bf16/fp16 C = 64, int8 C = 128), K = BN in {64,128,256} with the whole
// filter resident in shared memory.  Returns kNotApplicable otherwise.
int try_halo(const imconv_conv_args *a, int64_t P, int64_t Q, int sms, cudaStream_t st, bool dry = false) {
    const int E = elem_bytes(a->in_dtype);
    if (a->c * E != 128 || a->stride_h != 1 || a->stride_w != 1) return kNotApplicable;
    if (a->tile_n != 0 || a->order == IMCONV_ORDER_FILTER_MAJOR) return kNotApplicable;
    const int K = static_cast<int>(a->k), R = static_cast<int>(a->r), S = static_cast<int>(a->s);
    const int nc = 128 / E;
    // 1x1 filters have no tap reuse to gain, and the padded row pitch costs M utilisation
    if (R * S == 1) return kNotApplicable;
    if (K % nc != 0 || !(K == 64 || K == 128 || K == 256) || (E == 1 && K < 128)) return kNotApplicable;
    HaloParams p{};
    p.b_early = early_mode(a->flags);
    p.n = static_cast<int>(a->n);
    p.h = static_cast<int>(a->h);
    p.w = static_cast<int>(a->w_);
    p.k = K;
    p.r = R;
    p.s = S;
    p.ph = a->pad_h;
    p.pw = a->pad_w;
    p.dh = a->dil_h;
    p.dw = a->dil_w;
    p.p = static_cast<int>(P);
    p.q = static_cast<int>(Q);
    p.qp = static_cast<int>(Q) + (S - 1) * p.dw;
    if (p.qp > 128 || p.qp > 256) return kNotApplicable;
    p.tpr = 128 / p.qp;
    // two stacked sub-blocks per block (BN = 64, 16-bit): taps shared across them run as N = 128 MMAs
    const int hb = (K == 64 && E == 2 && !(g_debug_flags & kDbgNoHaloStack)) ? 2 : 1;
    p.tr = hb * p.tpr + (R - 1) * p.dh;
    if (p.tr > 256) return kNotApplicable;
    p.p_tiles = static_cast<int>((P + hb * p.tpr - 1) / (hb * p.tpr));
    p.n_tiles = 1;
    p.tiles = static_cast<long long>(p.n) * p.p_tiles;
    p.a_box_bytes = p.tr * p.qp * 128;
    // the last taps read up to 128 + (R-1)*dh*QP + (S-1)*dw rows (rows past the box feed only discarded accumulator rows)
    const int rows_read = std::max(p.tr * p.qp, (hb - 1) * p.tpr * p.qp + 128 + (R - 1) * p.dh * p.qp + (S - 1) * p.dw);
    p.a_stage_bytes = (rows_read * 128 + 1023) / 1024 * 1024;
    p.b_bytes = R * S * K * 128;
    // stacked bf16/fp16 BN = 64 blocks run on CTA pairs once there is a wave of blocks: each CTA
    // holds the shared taps' filter rows for one sub-block and 32 of the 64 columns of every tap
    // (conv_halo.cuh, CG = 2)
    const int dr_pair = (hb == 2 && p.tpr % p.dh == 0 && p.tpr / p.dh < R) ? p.tpr / p.dh : 0;
    const int cg = (hb == 2 && E == 2 && p.tiles >= sms && !(a->flags & IMCONV_FLAG_SINGLE_CTA) &&
                    !(g_debug_flags & kDbgHaloStreamSingle) && (a->num_ctas <= 0 || a->num_ctas % 2 == 0))
                       ? 2
                       : 1;
    if (cg == 2) {
        p.pair_dr = dr_pair;
        // shared-tap atoms first (8 KB each, so the SW64 region stays aligned); none without shared taps
        p.b_single_off = dr_pair > 0 ? (R - dr_pair) * S * K * 128 : 0;
        p.b_bytes = p.b_single_off + R * S * K * 64;
    }
    const int kOutTiles = 2 * kBM * 128;
    const int fixed = p.b_bytes + kOutTiles + 1024 /*align*/ + 1024 /*barriers*/;
    if (p.b_bytes > 120 * 1024) return kNotApplicable;
    p.n_stages = std::min(8, (kMaxDynSmem - fixed) / p.a_stage_bytes);
    if (p.n_stages < 2) return kNotApplicable;
    const int smem = fixed + p.n_stages * p.a_stage_bytes;

    if (dry) return 0;  // imconv_plan: applicable, nothing encoded or launched
    CUtensorMap ta, tb, ty, tb64;
    std::memset(&ta, 0, sizeof(ta));
    std::memset(&tb, 0, sizeof(tb));
    std::memset(&ty, 0, sizeof(ty));
    std::memset(&tb64, 0, sizeof(tb64));
    const int64_t N = a->n, H = a->h, W = a->w_, C = a->c;
    if (cg == 2) {  // half-column (32 x 64 rows, SW64) boxes of the filter for the pair's single taps
        cuuint64_t gdim[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(R * S * C)};
        cuuint64_t gstride[1] = {static_cast<cuuint64_t>(K * E)};
        cuuint32_t box[2] = {static_cast<cuuint32_t>(K / 2), static_cast<cuuint32_t>(nc)};
        cuuint32_t es[2] = {1, 1};
        if (g_encode_tiled(&tb64, tmap_dtype(a->in_dtype), 2, const_cast<void *>(a->w), gdim, gstride, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return IMCONV_ETMAP;
    }
    {
        cuuint64_t gdim[4] = {static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H),
                              static_cast<cuuint64_t>(N)};
        cuuint64_t gstride[3] = {static_cast<cuuint64_t>(C * E), static_cast<cuuint64_t>(W * C * E),
                                 static_cast<cuuint64_t>(H * W * C * E)};
        cuuint32_t box[4] = {static_cast<cuuint32_t>(nc), static_cast<cuuint32_t>(p.qp),
                             static_cast<cuuint32_t>(p.tr), 1};
        cuuint32_t es[4] = {1, 1, 1, 1};
        if (g_encode_tiled(&ta, tmap_dtype(a->in_dtype), 4, const_cast<void *>(a->x), gdim, gstride, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return IMCONV_ETMAP;
    }
    {
        cuuint64_t gdim[3] = {static_cast<cuuint64_t>(nc), static_cast<cuuint64_t>(R * S * C),
                              static_cast<cuuint64_t>(K / nc)};
        cuuint64_t gstride[2] = {static_cast<cuuint64_t>(K * E), static_cast<cuuint64_t>(nc * E)};
        cuuint32_t box[3] = {static_cast<cuuint32_t>(nc), static_cast<cuuint32_t>(nc),
                             static_cast<cuuint32_t>(K / nc)};
        cuuint32_t es[3] = {1, 1, 1};
        if (g_encode_tiled(&tb, tmap_dtype(a->in_dtype), 3, const_cast<void *>(a->w), gdim, gstride, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return IMCONV_ETMAP;
    }
    const int eo = (a->out_dtype == IMCONV_F32 || a->out_dtype == IMCONV_I32) ? 4 : 2;
    {
        CUtensorMapDataType dt = a->out_dtype == IMCONV_F32   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : a->out_dtype == IMCONV_I32 ? CU_TENSOR_MAP_DATA_TYPE_INT32
                                 : a->out_dtype == IMCONV_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                              : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
        cuuint64_t gdim[4] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(Q), static_cast<cuuint64_t>(P),
                              static_cast<cuuint64_t>(N)};
        cuuint64_t gstride[3] = {static_cast<cuuint64_t>(K * eo), static_cast<cuuint64_t>(Q * K * eo),
                                 static_cast<cuuint64_t>(P * Q * K * eo)};
        cuuint32_t box[4] = {static_cast<cuuint32_t>(128 / eo), static_cast<cuuint32_t>(Q),
                             static_cast<cuuint32_t>(p.tpr), 1};
        cuuint32_t es[4] = {1, 1, 1, 1};
        if (g_encode_tiled(&ty, dt, 4, a->y, gdim, gstride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return IMCONV_ETMAP;
    }
    int grid = a->num_ctas > 0 ? a->num_ctas : sms;
    if (cg == 2) {  // one pair per two blocks, whole clusters
        grid = static_cast<int>(std::min<long long>(grid, 2 * ((p.tiles + 1) / 2))) & ~1;
    } else if (grid > p.tiles) {
        grid = static_cast<int>(p.tiles);
    }
#define IMCONV_HALO(EL, OUTK)                                                                           \
    switch (K) {                                                                                        \
        case 64:                                                                                        \
            if (cg == 2) return launch_halo<EL, OUTK, 64, 2, 2>(ta, tb, ty, tb64, p, smem, grid, st);    \
            if (hb == 2) return launch_halo<EL, OUTK, 64, 2>(ta, tb, ty, tb64, p, smem, grid, st);       \
            return launch_halo<EL, OUTK, 64>(ta, tb, ty, tb64, p, smem, grid, st);                      \
        case 128: return launch_halo<EL, OUTK, 128>(ta, tb, ty, tb64, p, smem, grid, st);               \
        default: return launch_halo<EL, OUTK, 256>(ta, tb, ty, tb64, p, smem, grid, st);                \
    }
    const bool f32 = a->out_dtype == IMCONV_F32;
    switch (a->in_dtype) {
        case IMCONV_BF16:
            if (f32) { IMCONV_HALO(ELEM_BF16, OUT_F32) } else { IMCONV_HALO(ELEM_BF16, OUT_BF16) }
        case IMCONV_F16:
            if (f32) { IMCONV_HALO(ELEM_F16, OUT_F32) } else { IMCONV_HALO(ELEM_F16, OUT_F16) }
        case IMCONV_I8:
            if (K == 128) return launch_halo<ELEM_I8, OUT_I32, 128>(ta, tb, ty, tb64, p, smem, grid, st);
            return launch_halo<ELEM_I8, OUT_I32, 256>(ta, tb, ty, tb64, p, smem, grid, st);
        default: return kNotApplicable;
    }
#undef IMCONV_HALO
}

template <int ELEM, int OUT, int BN, int CG = 1>
int launch_halo_stream(const CUtensorMap &ta, const CUtensorMap &tb, const CUtensorMap &ty, const HaloStreamParams &p,
                       int smem, int grid, cudaStream_t st) {
    auto kern = conv_halo_stream_kernel<ELEM, OUT, BN, 2, CG>;
    static std::atomic<unsigned long long> attr_done{0};
    const cudaError_t attr_err = ensure_attrs(attr_done, kern, kMaxDynSmem, CG == 2);
    if (attr_err != cudaSuccess) return static_cast<int>(attr_err);
    cudaError_t le = launch_pdl(kern, grid, kThreadsGeneric, smem, st, CG, ta, tb, ty, p);
    if (le != cudaSuccess) return static_cast<int>(le);
    ++g_launches;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : static_cast<int>(e);
}

// Halo tiles with a streamed filter (conv_halo_stream.cuh): stride 1, 16-bit pixels of
// several 128-byte chunks (C = 128, 192, ...), K in {64, 128} (one or two 128-byte column
// atoms; two stacked sub-blocks per block).  Each input pixel crosses L2 -> SM once per
// block and chunk instead of R*S times.  Returns kNotApplicable otherwise.
// Wave quantisation against the generic kernel's 256-pixel blocks (K <= 128: one
// column block): a halo-stream wave costs ~0.81 of a generic wave (s3 3x3, N = 128 / 256:
// 7.2 vs 8.9 us per wave), so it is taken while ceil(halo tiles / SMs) <= 1.23 x
// ceil(generic tiles / SMs).  Measured (tools/shape_sweep.py): N = 128 halo 4 waves
// 29.5 us vs generic 3 waves 26.6 us; N = 256 halo 7 waves 50.0 vs generic 6 waves 52.6.
// blocks of the halo-stream kernel: per image, output-row groups of two sub-blocks of
// tpr = 128 / QP rows each (QP = Q + (S-1)*dw, the padded pitch)
inline long long halo_stream_tiles(int64_t N, int64_t P, int64_t Q, int64_t S, int dw) {
    const int64_t rows = 2 * (128 / (Q + (S - 1) * dw));
    return N * ((P + rows - 1) / rows);
}

inline bool halo_stream_wave_ok(long long halo_tiles, int64_t M, int sms) {
    const long long gen_tiles = (M + 2 * kBM - 1) / (2 * kBM);
    const long long wh = (halo_tiles + sms - 1) / sms, wg = (gen_tiles + sms - 1) / sms;
    return 100 * wh <= 123 * wg;
}

int try_halo_stream(const imconv_conv_args *a, int64_t P, int64_t Q, int sms, cudaStream_t st, bool dry = false) {
    const int E = elem_bytes(a->in_dtype);
    if (E != 2 || a->stride_h != 1 || a->stride_w != 1) return kNotApplicable;
    if (a->c * E <= 128 || (a->c * E) % 128 != 0) return kNotApplicable;
    if (a->tile_n != 0 || a->order == IMCONV_ORDER_FILTER_MAJOR) return kNotApplicable;
    if (a->flags & (IMCONV_FLAG_NO_HALO | IMCONV_FLAG_CHANNEL_LAST)) return kNotApplicable;
    if (g_debug_flags & kDbgNoHaloStream) return kNotApplicable;
    const int K = static_cast<int>(a->k), R = static_cast<int>(a->r), S = static_cast<int>(a->s);
    if (R * S == 1 || !(K == 64 || K == 128)) return kNotApplicable;
    constexpr int HB = 2;
    HaloStreamParams p{};
    p.b_early = early_mode(a->flags);
    p.n = static_cast<int>(a->n);
    p.h = static_cast<int>(a->h);
    p.w = static_cast<int>(a->w_);
    p.c = static_cast<int>(a->c);
    p.k = K;
    p.r = R;
    p.s = S;
    p.ph = a->pad_h;
    p.pw = a->pad_w;
    p.dh = a->dil_h;
    p.dw = a->dil_w;
    p.p = static_cast<int>(P);
    p.q = static_cast<int>(Q);
    p.qp = static_cast<int>(Q) + (S - 1) * p.dw;
    if (p.qp > 128) return kNotApplicable;
    p.tpr = 128 / p.qp;
    p.tr = HB * p.tpr + (R - 1) * p.dh;
    if (p.tr > 256) return kNotApplicable;
    p.p_tiles = static_cast<int>((P + HB * p.tpr - 1) / (HB * p.tpr));
    p.tiles = static_cast<long long>(p.n) * p.p_tiles;
    if (a->num_ctas <= 0 && !halo_stream_wave_ok(p.tiles, a->n * P * Q, sms)) return kNotApplicable;
    p.chunks = static_cast<int>(a->c * E / 128);
    // K = 128: a CTA pair runs two blocks with M = 256 MMAs, each CTA holding half of every filter
    // slice (one 64-column atom): 6 instead of 8 KB of operands per SM per 16-deep MMA
    // (below one wave of blocks the single-CTA kernel wins: s3 3x3 at N = 32 9.9 vs 10.4 us)
    const int cg = (K == 128 && !(a->flags & IMCONV_FLAG_SINGLE_CTA) && !(g_debug_flags & kDbgHaloStreamSingle) &&
                    (a->num_ctas <= 0 || a->num_ctas % 2 == 0) && p.tiles >= sms)
                       ? 2
                       : 1;
    p.a_box_bytes = p.tr * p.qp * 128;
    const int rows_read =
        std::max(p.tr * p.qp, (HB - 1) * p.tpr * p.qp + 128 + (R - 1) * p.dh * p.qp + (S - 1) * p.dw);
    p.a_slot_bytes = (rows_read * 128 + 1023) / 1024 * 1024;
    const int b_stage = K * 128 / cg;
    const int fixed = 2 * kBM * 128 + 1024 /*align*/ + 1024 /*barriers*/;
    p.na = 2;  // (3 input slots with the pair's 8 KB filter stages: 47.1 -> 47.4 us, not kept)
    p.nb = std::min(cg == 2 ? 12 : 8, (kMaxDynSmem - fixed - p.na * p.a_slot_bytes) / b_stage);
    if (p.nb < 3) return kNotApplicable;
    const int smem = fixed + p.na * p.a_slot_bytes + p.nb * b_stage;

    if (dry) return 0;  // imconv_plan: applicable, nothing encoded or launched
    CUtensorMap ta, tb, ty;
    std::memset(&ta, 0, sizeof(ta));
    std::memset(&tb, 0, sizeof(tb));
    std::memset(&ty, 0, sizeof(ty));
    const int64_t N = a->n, H = a->h, W = a->w_, C = a->c;
    const int nc = 128 / E;
    {
        cuuint64_t gdim[4] = {static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H),
                              static_cast<cuuint64_t>(N)};
        cuuint64_t gstride[3] = {static_cast<cuuint64_t>(C * E), static_cast<cuuint64_t>(W * C * E),
                                 static_cast<cuuint64_t>(H * W * C * E)};
        cuuint32_t box[4] = {static_cast<cuuint32_t>(nc), static_cast<cuuint32_t>(p.qp),
                             static_cast<cuuint32_t>(p.tr), 1};
        cuuint32_t es[4] = {1, 1, 1, 1};
        if (g_encode_tiled(&ta, tmap_dtype(a->in_dtype), 4, const_cast<void *>(a->x), gdim, gstride, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return IMCONV_ETMAP;
    }
    {
        cuuint64_t gdim[3] = {static_cast<cuuint64_t>(nc), static_cast<cuuint64_t>(R * S * C),
                              static_cast<cuuint64_t>(K / nc)};
        cuuint64_t gstride[2] = {static_cast<cuuint64_t>(K * E), static_cast<cuuint64_t>(nc * E)};
        cuuint32_t box[3] = {static_cast<cuuint32_t>(nc), static_cast<cuuint32_t>(nc),
                             static_cast<cuuint32_t>(K / nc / cg)};
        cuuint32_t es[3] = {1, 1, 1};
        if (g_encode_tiled(&tb, tmap_dtype(a->in_dtype), 3, const_cast<void *>(a->w), gdim, gstride, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return IMCONV_ETMAP;
    }
    const int eo = a->out_dtype == IMCONV_F32 ? 4 : 2;
    {
        CUtensorMapDataType dt = a->out_dtype == IMCONV_F32   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : a->out_dtype == IMCONV_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                              : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
        cuuint64_t gdim[4] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(Q), static_cast<cuuint64_t>(P),
                              static_cast<cuuint64_t>(N)};
        cuuint64_t gstride[3] = {static_cast<cuuint64_t>(K * eo), static_cast<cuuint64_t>(Q * K * eo),
                                 static_cast<cuuint64_t>(P * Q * K * eo)};
        cuuint32_t box[4] = {static_cast<cuuint32_t>(128 / eo), static_cast<cuuint32_t>(Q),
                             static_cast<cuuint32_t>(p.tpr), 1};
        cuuint32_t es[4] = {1, 1, 1, 1};
        if (g_encode_tiled(&ty, dt, 4, a->y, gdim, gstride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return IMCONV_ETMAP;
    }
    int grid = a->num_ctas > 0 ? a->num_ctas : sms;
    if (cg == 2) {  // one pair per two blocks, whole clusters
        grid = static_cast<int>(std::min<long long>(grid, 2 * ((p.tiles + 1) / 2))) & ~1;
    } else if (grid > p.tiles) {
        grid = static_cast<int>(p.tiles);
    }
    const bool f32 = a->out_dtype == IMCONV_F32;
#define IMCONV_HS(EL, OUTK)                                                                   \
    return K == 64    ? launch_halo_stream<EL, OUTK, 64>(ta, tb, ty, p, smem, grid, st)        \
           : cg == 2  ? launch_halo_stream<EL, OUTK, 128, 2>(ta, tb, ty, p, smem, grid, st)    \
                      : launch_halo_stream<EL, OUTK, 128>(ta, tb, ty, p, smem, grid, st);
    if (a->in_dtype == IMCONV_BF16) {
        if (f32) { IMCONV_HS(ELEM_BF16, OUT_F32) } else { IMCONV_HS(ELEM_BF16, OUT_BF16) }
    } else {
        if (f32) { IMCONV_HS(ELEM_F16, OUT_F32) } else { IMCONV_HS(ELEM_F16, OUT_F16) }
    }
#undef IMCONV_HS
}

// Row-band path for 16-byte pixels (bf16/fp16, C = 8).  Returns kNotApplicable
// when the layer does not qualify (the caller then uses the generic kernel).
int try_rowband(const imconv_conv_args *a, int64_t P, int64_t Q, int sms, cudaStream_t st, bool dry = false) {
    if (!(a->in_dtype == IMCONV_BF16 || a->in_dtype == IMCONV_F16) || a->c != 8) return kNotApplicable;
    if (a->tile_n != 0 || a->k > 256 || a->s > 2 * kMaxPairs || a->stride_w > 8) return kNotApplicable;
    const int K = static_cast<int>(a->k), R = static_cast<int>(a->r), S = static_cast<int>(a->s);
    const int BN = K <= 64 ? 64 : (K <= 128 ? 128 : 256);
    const int TP = 256 / BN;
    RowbandParams p{};
    p.b_early = early_mode(a->flags);
    p.n = static_cast<int>(a->n);
    p.h = static_cast<int>(a->h);
    p.w = static_cast<int>(a->w_);
    p.k = K;
    p.r = R;
    p.s = S;
    p.sh = a->stride_h;
    p.sw = a->stride_w;
    p.ph = a->pad_h;
    p.pw = a->pad_w;
    p.dh = a->dil_h;
    p.dw = a->dil_w;
    p.p = static_cast<int>(P);
    p.q = static_cast<int>(Q);
    p.p_groups = static_cast<int>((P + TP - 1) / TP);
    p.q_blocks = static_cast<int>((Q + 127) / 128);
    p.tiles = static_cast<long long>(p.n) * p.p_groups * p.q_blocks;
    int t_s[2 * kMaxPairs], e_s[2 * kMaxPairs];
    int t_min = 1 << 30, t_max = -(1 << 30);
    for (int s = 0; s < S; ++s) {
        const int off = s * p.dw - p.pw;
        t_s[s] = floordiv(off, p.sw);
        e_s[s] = off - p.sw * t_s[s];
        t_min = std::min(t_min, t_s[s]);
        t_max = std::max(t_max, t_s[s]);
    }
    p.t_min = t_min;
    // +1: a pair's zero half reads the run one pixel past its first tap
    p.needed = static_cast<int>(std::min<int64_t>(Q, 128)) + t_max - t_min + 1;
    const int plane_pix = 129 + t_max - t_min;
    p.x = static_cast<const uint8_t *>(a->x);
    p.dbg = g_debug_buf;
    p.dbg_flags = g_debug_flags;
    // plane pitch: 128 / sw bytes past a multiple of 128, so the sw planes' slots written by one
    // 8-lane copy phase fall on disjoint banks (a 128-byte multiple made every phase 2-way
    // conflicted: 2.9 M excess wavefronts per stem launch); descriptors need 16-byte alignment only
    p.plane_bytes = ((plane_pix * 16 + 127) / 128) * 128 +
                    ((p.sw > 1 && 8 % p.sw == 0 && !(g_debug_flags & kDbgPlanePitch128)) ? 128 / p.sw : 0);
    p.row_bytes_planes = p.sw * p.plane_bytes;
    const int rows_needed = (TP - 1) * p.sh + (R - 1) * p.dh + 1;
    p.npairs = (S + 1) / 2;
    p.b_chunk_bytes = R * p.npairs * 2 * 1024;
    p.b_bytes = (BN / 64) * p.b_chunk_bytes;
    const int kStaging = 2 * kBM * 128;  // two 128-pixel x 128-byte epilogue staging tiles
    const int fixed = p.b_bytes + kStaging + 1024 /*align*/ + 1024 /*barriers + tables*/;
    const int room = kMaxDynSmem - fixed;
    // input rows per pipeline stage: every stage costs the MMA issuer a fixed
    // handshake (wait, fences, commit), so stages are made as large as the
    // ring allows while keeping >= kMinStages of them in flight
    constexpr int kMinStages = 4;
    p.rps = 1;
    for (int spb = 1; spb <= rows_needed; ++spb) {  // fewest stages per block, then fewest padding rows
        const int rps = (rows_needed + spb - 1) / spb;
        if (room / (rps * p.row_bytes_planes) >= kMinStages) {
            p.rps = rps;
            break;
        }
    }
    if ((g_debug_flags >> 8) & 0xff) p.rps = std::min(rows_needed, (g_debug_flags >> 8) & 0xff);  // experiment override
    p.a_stage_bytes = p.rps * p.row_bytes_planes;
    p.in_rows = (rows_needed + p.rps - 1) / p.rps * p.rps;
    // taps ordered by their run address inside a stage, paired neighbour-wise
    int order[2 * kMaxPairs], addr[2 * kMaxPairs];
    for (int s = 0; s < S; ++s) {
        order[s] = s;
        addr[s] = e_s[s] * p.plane_bytes + (t_s[s] - t_min) * 16;
    }
    std::sort(order, order + S, [&](int x, int y) { return addr[x] < addr[y]; });
    for (int pr = 0; pr < p.npairs; ++pr) {
        const int s0 = order[2 * pr];
        const int s1 = 2 * pr + 1 < S ? order[2 * pr + 1] : -1;
        p.pair_s0[pr] = s0;
        p.pair_s1[pr] = s1;
        p.pair_a_off[pr] = addr[s0];
        p.pair_lbo[pr] = s1 >= 0 ? addr[s1] - addr[s0] : 16;  // zero tap: any finite run
    }
    p.n_stages = std::min(24, room / p.a_stage_bytes);
    // adjacent output rows share N = 128 MMAs (BN = 64, no dilation: filter rows sh apart)
    p.row_pair_lbo = (BN == 64 && TP >= 2 && p.dh == 1 && !(g_debug_flags & kDbgNoRowPairs))
                         ? p.sh * p.npairs * 2048 : 0;
    if (p.row_pair_lbo >= (1 << 18)) p.row_pair_lbo = 0;  // (14-bit LBO field, 16-byte units)

    if (p.b_bytes > 128 * 1024 || p.n_stages < 3 || p.in_rows * TP > 256 || 2 * p.n_stages * 8 + 64 > 512 ||
        p.sw * p.needed > kProducers * kMaxEntPerThread)
        return kNotApplicable;
    const int smem = fixed + p.n_stages * p.a_stage_bytes;

    if (dry) return 0;  // imconv_plan: applicable, nothing encoded or launched
    CUtensorMap tw, ty;
    std::memset(&tw, 0, sizeof(tw));
    std::memset(&ty, 0, sizeof(ty));
    const int64_t N = a->n, C = 8;
    {
        cuuint64_t gdim[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(R * S * C)};
        cuuint64_t gstride[1] = {static_cast<cuuint64_t>(K * 2)};
        cuuint32_t box[2] = {64, 8};
        cuuint32_t es[2] = {1, 1};
        if (g_encode_tiled(&tw, tmap_dtype(a->in_dtype), 2, const_cast<void *>(a->w), gdim, gstride, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return IMCONV_ETMAP;
    }
    {
        const int eo = a->out_dtype == IMCONV_F32 ? 4 : 2;
        CUtensorMapDataType dt = a->out_dtype == IMCONV_F32   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : a->out_dtype == IMCONV_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                              : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
        cuuint64_t gdim[4] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(Q), static_cast<cuuint64_t>(P),
                              static_cast<cuuint64_t>(N)};
        cuuint64_t gstride[3] = {static_cast<cuuint64_t>(K * eo), static_cast<cuuint64_t>(Q * K * eo),
                                 static_cast<cuuint64_t>(P * Q * K * eo)};
        cuuint32_t box[4] = {static_cast<cuuint32_t>(128 / eo), 128, 1, 1};  // one 128-byte chunk x 128 pixels
        cuuint32_t es[4] = {1, 1, 1, 1};
        if (g_encode_tiled(&ty, dt, 4, a->y, gdim, gstride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return IMCONV_ETMAP;
    }
    int grid = a->num_ctas > 0 ? a->num_ctas : sms;
    if (grid > p.tiles) grid = static_cast<int>(p.tiles);
    const bool f32 = a->out_dtype == IMCONV_F32;
    // the ResNet stem geometry runs an instantiation whose MMA issue is fully compile-time
    const bool stem = BN == 64 && R == kStemR && S == 7 && p.sh == kStemSh && p.dh == 1 && p.rps == kStemRps &&
                      p.in_rows == kStemInRows && p.npairs == 4 && p.row_pair_lbo > 0 && !(g_debug_flags & kDbgNoStemSpec);
#define IMCONV_RB(EL, OUTK)                                                                               \
    if (stem) return launch_rowband<EL, OUTK, 64, 4, 4, 1>(tw, ty, p, smem, grid, st);                    \
    if (p.npairs <= 4) {                                                                                   \
        switch (BN) {                                                                                      \
            case 64: return launch_rowband<EL, OUTK, 64, 4, 4>(tw, ty, p, smem, grid, st);                 \
            case 128: return launch_rowband<EL, OUTK, 128, 2, 4>(tw, ty, p, smem, grid, st);               \
            default: return launch_rowband<EL, OUTK, 256, 1, 4>(tw, ty, p, smem, grid, st);                \
        }                                                                                                  \
    } else {                                                                                               \
        switch (BN) {                                                                                      \
            case 64: return launch_rowband<EL, OUTK, 64, 4, 8>(tw, ty, p, smem, grid, st);                 \
            case 128: return launch_rowband<EL, OUTK, 128, 2, 8>(tw, ty, p, smem, grid, st);               \
            default: return launch_rowband<EL, OUTK, 256, 1, 8>(tw, ty, p, smem, grid, st);                \
        }                                                                                                  \
    }
    if (a->in_dtype == IMCONV_BF16) {
        if (f32) { IMCONV_RB(ELEM_BF16, OUT_F32) } else { IMCONV_RB(ELEM_BF16, OUT_BF16) }
    } else {
        if (f32) { IMCONV_RB(ELEM_F16, OUT_F32) } else { IMCONV_RB(ELEM_F16, OUT_F16) }
    }
#undef IMCONV_RB
}

}  // namespace
}  // namespace imconv

using namespace imconv;

int predict_traffic_impl(const imconv_conv_args *a, int64_t l2_bytes, int sms, imconv_traffic *out);

static int grid_for(long long work) {
    long long g = (work + 255) / 256;
    if (g > 148LL * 16) g = 148LL * 16;
    if (g < 1) g = 1;
    return static_cast<int>(g);
}

extern "C" {

int imconv_abi_version(void) { return IMCONV_ABI_VERSION; }

int imconv_predict_traffic(const imconv_conv_args *args, int64_t l2_bytes, int32_t sms, imconv_traffic *out) {
    if (!args || !out) return IMCONV_EINVAL;
    try {
        return predict_traffic_impl(args, l2_bytes, sms, out);
    } catch (...) {
        return IMCONV_EINVAL;  // (allocation failure of the replay's bookkeeping)
    }
}

int64_t imconv_out_extent(int64_t size, int64_t f, int64_t stride, int64_t pad, int64_t dil) {
    if (stride < 1 || dil < 1 || f < 1 || pad < 0) return 0;
    const int64_t ext = dil * (f - 1) + 1;
    if (ext > size + 2 * pad) return 0;
    return out_extent(size, f, stride, pad, dil);
}

const char *imconv_strerror(int code) {
    switch (code) {
        case IMCONV_OK: return "ok";
        case IMCONV_EINVAL: return "invalid argument (spec, extent or null pointer)";
        case IMCONV_EDTYPE: return "unsupported dtype combination";
        case IMCONV_EALIGN: return "pointer is not 16-byte aligned";
        case IMCONV_ECHAN: return "channel count times element size must be a multiple of 16 bytes";
        case IMCONV_ETMAP: return "TMA tensor-map encoding rejected the operand";
        case IMCONV_ENODEV: return "no CUDA device or driver entry point";
        case IMCONV_ERANGE: return "extent exceeds a TMA im2col limit";
        default: break;
    }
    if (code > 0) return cudaGetErrorString(static_cast<cudaError_t>(code));
    return "unknown error";
}

int imconv_device_sm_count(int32_t *sm_count) {
    if (!sm_count) return IMCONV_EINVAL;
    int n = 0;
    int rc = sm_count_for_current_device(&n);
    if (rc) return rc;
    *sm_count = n;
    return 0;
}

int64_t imconv_launch_count(void) { return g_launches; }
void imconv_debug_set_buffer(void *dev_buf) { g_debug_buf = static_cast<long long *>(dev_buf); }
void imconv_debug_set_flags(int flags) { g_debug_flags = flags; }
void imconv_reset_launch_count(void) { g_launches = 0; }

}  // extern "C" (the planner below is internal C++)

// Block-shape / raster decisions of the generic kernel, shared by the launcher
// and the DRAM-traffic predictor (imconv_predict_traffic) so the model replays
// exactly the schedule that runs.
struct GenericPlan {
    int bn, variant, mt, ksub;
    bool use_pair;
    int row_bytes, tps, c_chunks, k_subs;  // k_subs: k-subtiles per block
    long long m_tiles, n_tiles, tiles;
    int grid;
    bool b_resident;
    int sk_split;        // 1 = off
    long long sk_tail;   // sk_mode 1: tail tiles split S ways; sk_mode 2: tiles of the stream-K region
    int sk_mode;         // 0 whole tiles, 1 split-K tail, 2 stream-K (conv_kernel.cuh UnitWalk)
};

// One candidate block shape: bn output channels, variant_force >= 0 overrides
// the m-tile / k-subtile variant (see dispatch_bn).
// split-K: cycles one split tail pays for the partials' L2 round trip (fitted, see plan_generic)
constexpr int kSkCyclesPerSplit = 15000;
constexpr int kSkStreamMinStages = 8;  // stream-K: shortest k-loop (stages) worth cutting

int plan_generic_bn(const imconv_conv_args *a, int64_t P, int64_t Q, int sms, int bn_req, int variant_force,
                    GenericPlan *g, bool pair_force = false) {
    const int64_t K = a->k, R = a->r, S = a->s, C = a->c;
    const int E = elem_bytes(a->in_dtype);
    const int64_t M = a->n * P * Q;
    g->bn = pick_bn(a->in_dtype, K, bn_req);
    if (g->bn < 0) return IMCONV_EINVAL;
    const int bn = g->bn;
    // (A wave-quantisation chooser over {256x128, 128x256, 128x128, ...} blocks
    // was measured worse on the stage-5 layers: smaller blocks lose more
    // per-block efficiency than they gain in wave fill, so BN is fixed by K.)
    // 1x1 layers with N = 128: one m-tile per CTA and two k-subtiles per stage measured
    // faster than two m-tiles (s3 1x1a: 102.5 -> 94.0 us, 44.8 -> 43.7 us); 3x3 and N = 64 lose.
    const bool no_override = !(a->flags & (IMCONV_FLAG_KSUB1 | IMCONV_FLAG_MT1));
    const int auto_variant = (no_override && R * S == 1 && bn == 128) ? 1 : -1;
    // ---- block shape: single CTA or CTA pair (cta_group::2, B split across the pair) ----
    // pairs need whole swizzle-atom columns per CTA (BN >= 128 bf16 / 256 int8)
    // and enough 256-row blocks to fill the clusters.
    const int64_t m_tiles_ = (M + kBM - 1) / kBM;
    const int64_t n_tiles_ = (K + bn - 1) / bn;
    const long long pair_tiles = ((m_tiles_ + 1) / 2) * n_tiles_;
    const bool pair_ok = (a->in_dtype == IMCONV_I8) ? bn == 256 : bn >= 128;
    // Measured (tools/run_layer.py --flags 1/2): once the producers issue one
    // TMA per operand per stage, single CTAs match or beat pairs on the
    // ResNet-50 shapes, so pairs are opt-in for now.
    g->use_pair = pair_ok && !(a->flags & IMCONV_FLAG_SINGLE_CTA) &&
                  ((a->flags & IMCONV_FLAG_CTA_PAIR) || pair_force) && pair_tiles >= 1;
    // single-CTA block shape (see dispatch_bn): N <= 128 -> 2 m-tiles per CTA
    g->variant = variant_force >= 0 ? variant_force
                 : auto_variant >= 0 ? auto_variant
                 : (a->flags & IMCONV_FLAG_KSUB1) ? 2 : (a->flags & IMCONV_FLAG_MT1) ? 1 : 0;
    g->mt = (!g->use_pair && bn <= 128 && g->variant == 0) ? 2 : 1;
    g->ksub = (!g->use_pair && g->variant == 1) ? 2 : 1;
    const int64_t cbytes = C * E;
    g->row_bytes = cbytes >= 128 ? 128 : static_cast<int>(cbytes);  // 16, 32, 64 or 128
    if (g->row_bytes != 128 && g->row_bytes != 64 && g->row_bytes != 32 && g->row_bytes != 16) return IMCONV_ECHAN;
    g->tps = kRowBytes / g->row_bytes;
    g->c_chunks = g->tps == 1 ? static_cast<int>((cbytes + kRowBytes - 1) / kRowBytes) : 1;
    g->k_subs = g->tps == 1 ? g->c_chunks * static_cast<int>(R * S) : static_cast<int>((R * S + g->tps - 1) / g->tps);
    const bool cl = (a->flags & IMCONV_FLAG_CHANNEL_LAST) != 0;
    if (cl) {  // channel-last baseline: one m-tile, one k-subtile per stage, k = (c, r, s) in 128-byte subtiles
        g->use_pair = false;
        g->variant = 2;
        g->mt = 1;
        g->ksub = 1;
        g->row_bytes = 128;
        g->tps = 1;
        g->c_chunks = 1;
        g->k_subs = static_cast<int>((R * S * C * E + kRowBytes - 1) / kRowBytes);
    }
    const int rows = kBM * g->mt * (g->use_pair ? 2 : 1);
    g->m_tiles = (M + rows - 1) / rows;
    g->n_tiles = (K + bn - 1) / bn;
    g->tiles = g->m_tiles * g->n_tiles;
    const bool a_gather = !cl && g->row_bytes == 16 && E == 2 && !g->use_pair && g->variant != 1;
    int grid = a->num_ctas > 0 ? a->num_ctas : sms;
    // B-stationary (1x1 layers with C*e <= 512 B): every k-subtile of a block fits the
    // 4-deep B ring, so a CTA that always works on the same output-channel block loads
    // its filter slice once.  Needs grid % n_tiles == 0 (persistent round-robin over
    // n-fastest tiles then keeps each CTA on one n-block); allowed to drop <= 4% of SMs.
    g->b_resident = false;
    if (!cl && !g->use_pair && g->variant != 1 && !a_gather && g->k_subs <= 4 && !(g_debug_flags & kDbgNoBResident)) {
        int gg = static_cast<int>(std::min<long long>(grid, g->tiles));
        gg = static_cast<int>(gg / g->n_tiles * g->n_tiles);
        if (gg >= g->n_tiles && gg * 100 >= 96 * std::min<long long>(grid, g->tiles)) {
            grid = gg;
            g->b_resident = true;
        }
    }
    // Split-K: when the blocks do not fill one wave (small per-GPU batches), or the
    // last wave would be at most half full, each tail tile's k-loop is split S ways
    // across otherwise-idle CTAs (S*tail <= grid).  Every split writes its 32-bit
    // partial sums to a workspace, waits for its peers, and reduces + stores the
    // output blocks it owns (the reduction is spread over the S splits, with one
    // bulk copy per peer block).  Full waves stay data-parallel.  (Not with
    // B-stationary: split units change a CTA's output-channel block.)  Each split
    // keeps >= 4 pipeline stages; S <= 5 so S peer blocks fit the idle operand ring.
    g->sk_split = 1;
    g->sk_tail = 0;
    g->sk_mode = 0;
    // Splits of one tile spin-wait for each other, so every CTA of the grid must be
    // resident at once: never with a caller grid above one CTA per SM.
    // CTA pairs split pair tiles over clusters (g0 = grid / 2 pairs; a pair's two CTAs exchange
    // their own 128-row halves with the same-rank CTAs of the other splits).
    if (!cl && !a_gather && !g->b_resident && grid <= sms && !(g_debug_flags & kDbgNoSplitK) &&
        !(g->use_pair && (g_debug_flags & kDbgNoPairSplit))) {
        const int k_st = (g->k_subs + g->ksub - 1) / g->ksub;
        const long long g0 = g->use_pair ? grid / 2 : grid;
        const long long tail = g->tiles >= g0 ? g->tiles % g0 : g->tiles;
        // Measured (tools/small_n_probe.py): the partials' L2 round trip (write 4 B per
        // output, fence, peer wait, read back) costs ~5-7k cycles per split.  Below one wave
        // it is exposed, so only long k-loops gain (3x3 with C >= 256: 36+ stages).  Behind
        // full waves the split units run first and the exchange hides behind the CTA's next
        // whole tile (UnitWalk): k-loops of >= 24 stages gain (tools/ab_layers.py: s5 3x3 at
        // N = 256 49.6 -> 41.1 us, s5 1x1a (32 stages) 26.0 -> 23.9; 16-stage 1x1 layers lose ~8%).
        constexpr int kSkMaxSplit = 5, kSkMinStages = 36, kSkMinStagesHidden = 24;
        // Throughput mode (IMCONV_FLAG_INDEPENDENT): a layer's idle SMs -- below one wave or in its
        // last wave -- run the next launch, so splitting only adds the partials' round trip
        // (measured: 2-GPU shard of the cfg4 sweep 1598 -> 1679 TFLOP/s without split tails).
        const bool thr = (a->flags & IMCONV_FLAG_INDEPENDENT) != 0;
        const bool sub_wave = g->tiles < g0 && k_st >= kSkMinStages && !thr;
        const bool short_tail = g->tiles >= g0 && tail > 0 && 2 * tail <= g0 && k_st >= kSkMinStagesHidden && !thr;
        if (sub_wave || short_tail) {
            const int Sk = static_cast<int>(std::min<long long>(
                {g0 / tail, static_cast<long long>(k_st / 4), kSkMaxSplit}));
            // sub-wave: only when the stages saved (k_st * (1 - 1/S) at ~600 cycles) beat the
            // ~15k-cycle exposed round trip (a 3-way split of a 36-stage k-loop loses: s4 3x3
            // at N = 128, 31.6 us split vs 29.3 us with CTA pairs)
            const bool pays = short_tail || static_cast<long long>(k_st) * (Sk - 1) >
                                                static_cast<long long>(kSkCyclesPerSplit / 600) * Sk;
            if (Sk >= 2 && tail * (g->use_pair ? 2 : 1) <= kSkSliceLen && pays) {
                g->sk_split = Sk;
                g->sk_tail = tail;
                g->sk_mode = 1;
                if (g->tiles < g0) grid = static_cast<int>(tail * Sk * (g->use_pair ? 2 : 1));
            }
        }
        // Stream-K (opt-in, kDbgStreamK): a last wave more than half full cannot be split S >= 2
        // ways, so the last partial wave and one full wave are streamed as equal k-ranges over all
        // CTAs (a tile is cut at most once; the writer/finisher exchange runs in the epilogue).
        // Measured slower on every candidate (tools/ab_layers.py, N = 256: s4 3x3 41.1 -> 43.6 us,
        // s4 1x1a 27.4 -> 39.1; N = 128 s5 1x1b 15.3 -> 26.6): every cut tile moves a 128 KB fp32
        // partial per CTA through L2 twice, and the epilogue's global-store throughput (~32 GB/s
        // per SM, the same limit as the output stream) makes that cost more than the wave saved.
        const long long n_sk = tail + g0;
        if (g->sk_mode == 0 && g->tiles >= g0 && 2 * tail > g0 && tail < g0 && k_st >= kSkStreamMinStages &&
            n_sk * (g->use_pair ? 2 : 1) <= kSkSliceLen && (g_debug_flags & kDbgStreamK)) {
            g->sk_mode = 2;
            g->sk_tail = n_sk;
        }
    }
    if (g->use_pair) {
        if (g->sk_split == 1 && grid > 2 * g->tiles) grid = static_cast<int>(2 * g->tiles);
        if (grid < 2) grid = 2;
    } else if (g->sk_split == 1 && grid > g->tiles) {
        grid = static_cast<int>(g->tiles);
    }
    g->grid = grid;
    return 0;
}

// Block-shape choice.  BN follows K (<= 256); but when the 128 x 256 blocks do
// not fill one wave (small per-GPU batches: the stage-4/5 layers at N = 32),
// 128 x 128 blocks with two k-subtiles per stage (twice the blocks, half the
// tensor work per stage) are compared against 128 x 256 (+ split-K) with a
// per-CTA latency model: ceil(units / grid) * (stages per unit * cycles per
// stage + split-K partial round trip).  Measured (tools/small_n_probe.py,
// N = 32): s4 1x1a 9.7 -> 8.0 us, s5 1x1a 14.5 -> 12.1, s4 3x3 16.3 -> 13.2;
// s5 3x3 keeps 128 x 256 with a 5-way split (18.0 vs 19.4).
inline bool R_S_is_1x1(const imconv_conv_args *a) { return a->r == 1 && a->s == 1; }

int plan_generic(const imconv_conv_args *a, int64_t P, int64_t Q, int sms, GenericPlan *g) {
    int rc = plan_generic_bn(a, P, Q, sms, a->tile_n, -1, g);
    if (rc || a->tile_n != 0 || g->bn != 256 || g->use_pair || (a->flags & (IMCONV_FLAG_CHANNEL_LAST |
                                                                             IMCONV_FLAG_KSUB1 | IMCONV_FLAG_MT1)))
        return rc;
    if (R_S_is_1x1(a) && g->b_resident && g->tiles >= 16LL * sms && !(g_debug_flags & kDbgNo1x1Stream)) {
        // Output-heavy 1x1 layers with a 1-2 k-subtile filter slice and many blocks (>= 16 waves):
        // the streamed filter beats the B-stationary layout (measured: s2 1x1b / projection
        // 90.5 -> 85.4 us with 128 x 128 blocks; s3 1x1b 47.2 -> 45.0 us with 128 x 256 blocks).
        GenericPlan h;
        if (g->k_subs == 1 && a->k >= 256 && plan_generic_bn(a, P, Q, sms, 128, 1, &h) == 0 && !h.use_pair) {
            *g = h;
            return 0;
        }
        if (g->k_subs == 2 && g->bn == 256 && plan_generic_bn(a, P, Q, sms, 256, 1, &h) == 0 && !h.use_pair) {
            *g = h;
            return 0;
        }
    }
    if (g->tiles >= sms) {
        // At least one wave of 128 x 256 blocks with the filter streamed (not B-stationary,
        // no split-K tail): CTA pairs (cta_group::2, 256 x 256 per pair, each CTA loads
        // half of B) cut the per-SM operand bytes per stage by a third and run a 6-deep
        // ring.  Measured N = 256: s4 1x1a 29.4 -> 26.6 us, s4 proj 51.7 -> 46.3,
        // s5 1x1b 25.7 -> 23.9, s4 3x3 42.2 -> 40.7; B-stationary and split-K layers lose.
        // With >= 2 waves the pair's per-stage saving outweighs a single-CTA split tail (s5
        // 1x1a / proj at N = 256: pair 43.3 / 40.4 us, 128 x 256 + split tail 48.1 / 44.8).
        // A pair plan may carry its own split tail (pair tiles over grid / 2 clusters).
        if (!g->b_resident && !(a->flags & IMCONV_FLAG_SINGLE_CTA) && !(g_debug_flags & kDbgNoAutoPair)) {
            GenericPlan h;
            if (plan_generic_bn(a, P, Q, sms, 256, -1, &h, true) == 0 && h.use_pair) *g = h;
        }
        return 0;
    }
    if (a->flags & IMCONV_FLAG_INDEPENDENT) {
        // Throughput mode (sub-wave, independent launch): the SMs this layer leaves idle run the
        // next launch, so the block shape minimises SM time (CTAs x per-CTA time), not this
        // layer's latency: the largest blocks, CTA pairs when a pair block exists, no split.
        GenericPlan h;
        if (!(g_debug_flags & kDbgThrNoPair) && !(a->flags & IMCONV_FLAG_SINGLE_CTA) &&
            plan_generic_bn(a, P, Q, sms, 256, -1, &h, true) == 0 && h.use_pair)
            *g = h;
        return 0;
    }
    GenericPlan h;
    if (plan_generic_bn(a, P, Q, sms, 128, 1, &h) != 0 || h.use_pair) return 0;
    // Full waves run k_st stages per block; a split-K tail runs k_st / S stages plus the
    // partials' round trip.  Cycles per stage in this latency-bound regime, fitted to
    // tools/shape_sweep.py at N = 32 / 128: ~600 for a 128 x 256 x 64 stage (48 KB of
    // operands), ~900 for a 2-k-subtile 128 x 128 stage (64 KB, same tensor work);
    // ~15k cycles per split-K tail (s5 3x3 at N = 128: 128 x 256 blocks 29.0 us vs
    // 128 x 128 blocks + split tail 36.7 us; s4 3x3 at N = 32: 128 x 128 13.2 vs
    // 128 x 256 + 3-way split 16.3).
    auto cost = [&](const GenericPlan &q, double cyc_stage) {
        const double k_st = static_cast<double>((q.k_subs + q.ksub - 1) / q.ksub);
        const long long full = q.tiles - (q.sk_mode == 1 ? q.sk_tail : 0);
        const long long full_waves = (full + q.grid - 1) / q.grid;
        const long long tail_waves = q.sk_mode == 1 ? (q.sk_tail * q.sk_split + q.grid - 1) / q.grid : 0;
        return static_cast<double>(full_waves) * k_st * cyc_stage +
               static_cast<double>(tail_waves) * (k_st / q.sk_split * cyc_stage + kSkCyclesPerSplit);
    };
    if (cost(h, 900.0) < cost(*g, 600.0)) *g = h;
    return 0;
}

// ---- DRAM-traffic predictor (imconv_predict_traffic) ----
// Line keys: x, w and y live in disjoint 128-byte-line ranges; an activation
// line is (((n*H + h)*W + w)*C*e + byte) >> 7 -- batch-aware, unlike the
// reference's (h, w, c) element keys that count every image's identical
// stream again.
int predict_traffic_impl(const imconv_conv_args *a, int64_t l2_bytes, int sms, imconv_traffic *out) {
    const int64_t N = a->n, H = a->h, W = a->w_, C = a->c, K = a->k, R = a->r, S = a->s;
    if (N < 1 || H < 1 || W < 1 || C < 1 || K < 1 || R < 1 || S < 1 || sms < 1 || l2_bytes < 0) return IMCONV_EINVAL;
    if (a->stride_h < 1 || a->stride_w < 1 || a->dil_h < 1 || a->dil_w < 1 || a->pad_h < 0 || a->pad_w < 0)
        return IMCONV_EINVAL;
    const bool f16in = a->in_dtype == IMCONV_BF16 || a->in_dtype == IMCONV_F16;
    if (!f16in && a->in_dtype != IMCONV_I8) return IMCONV_EDTYPE;
    const int E = elem_bytes(a->in_dtype);
    const int EO = (a->out_dtype == IMCONV_F32 || a->out_dtype == IMCONV_I32) ? 4 : 2;
    if ((C * E) % 16 != 0 || (K * E) % 16 != 0) return IMCONV_ECHAN;
    const int64_t P = imconv_out_extent(H, R, a->stride_h, a->pad_h, a->dil_h);
    const int64_t Q = imconv_out_extent(W, S, a->stride_w, a->pad_w, a->dil_w);
    if (P < 1 || Q < 1) return IMCONV_EINVAL;
    const int64_t M = N * P * Q;
    GenericPlan g;
    const int rc = plan_generic(a, P, Q, sms, &g);
    if (rc) return rc;
    std::memset(out, 0, sizeof(*out));
    out->bn = g.bn;
    out->mt = g.mt;
    out->grid = g.grid;
    out->k_subtiles = g.k_subs;
    out->tiles = g.tiles;
    out->kernel = (C * E == 16 && f16in && !(a->flags & IMCONV_FLAG_GATHER16)) ? 1
                  : (C * E == 128 && a->stride_h == 1 && a->stride_w == 1 && R * S > 1 &&
                     !(a->flags & IMCONV_FLAG_NO_HALO) && (K == 64 || K == 128 || K == 256) &&
                     R * S * K * 128 <= 120 * 1024)
                      ? 2
                  : (E == 2 && C * E > 128 && (C * E) % 128 == 0 && a->stride_h == 1 && a->stride_w == 1 &&
                     R * S > 1 && (K == 64 || K == 128) && Q + (S - 1) * a->dil_w <= 128 &&
                     !(a->flags & IMCONV_FLAG_NO_HALO) &&
                     (a->num_ctas > 0 || halo_stream_wave_ok(halo_stream_tiles(N, P, Q, S, a->dil_w), M, sms)))
                      ? 3
                      : 0;
    const int64_t x_lines = (N * H * W * C * E + 127) / 128;
    const int64_t w_lines = (R * S * C * K * E + 127) / 128;
    const int64_t w_base = x_lines, y_base = x_lines + w_lines;
    const int64_t cap = l2_bytes / 128;
    imconv::LineLRU lru(std::max<int64_t>(cap, 1));
    std::vector<uint8_t> seen(static_cast<size_t>(x_lines + w_lines), 0);
    int64_t reads = 0, requests = 0, compulsory = 0;
    auto touch_read = [&](int64_t line) {
        ++requests;
        if (!seen[static_cast<size_t>(line)]) {
            seen[static_cast<size_t>(line)] = 1;
            ++compulsory;
        }
        if (cap <= 0 || !lru.access(line, false)) ++reads;
    };
    // a CTA pair is one 256-row unit: each CTA loads its 128 rows of A and half of B
    const int rows_per_tile = kBM * g.mt * (g.use_pair ? 2 : 1);
    const int kbke = kRowBytes / E;  // k-rows (reduction elements) per k-subtile
    const int rs = static_cast<int>(R * S);
    // A lines of k-subtile ks of m-tile mt_idx (im2col of rows_per_tile output pixels)
    auto a_lines = [&](long long m_tile, int ks) {
        const int64_t m0 = m_tile * rows_per_tile;
        for (int64_t m = m0; m < std::min<int64_t>(m0 + rows_per_tile, M); ++m) {
            const int64_t n = m / (P * Q), pq = m - n * P * Q, p = pq / Q, q = pq - p * Q;
            const int taps = g.tps == 1 ? 1 : g.tps;
            for (int t = 0; t < taps; ++t) {
                int tap, chunk;
                if (g.tps == 1) {
                    if (a->order == IMCONV_ORDER_FILTER_MAJOR) {
                        tap = ks / g.c_chunks;
                        chunk = ks - tap * g.c_chunks;
                    } else {
                        chunk = ks / rs;
                        tap = ks - chunk * rs;
                    }
                } else {
                    tap = ks * g.tps + t;
                    chunk = 0;
                    if (tap >= rs) break;
                }
                const int64_t r = tap / S, s = tap - r * S;
                const int64_t h = p * a->stride_h - a->pad_h + r * a->dil_h;
                const int64_t w = q * a->stride_w - a->pad_w + s * a->dil_w;
                if (h < 0 || h >= H || w < 0 || w >= W) continue;  // zero fill: no memory access
                const int64_t byte = ((n * H + h) * W + w) * C * E + static_cast<int64_t>(chunk) * 128;
                const int64_t bytes = std::min<int64_t>(g.tps == 1 ? 128 : C * E, C * E - chunk * 128);
                for (int64_t l = byte >> 7; l <= (byte + bytes - 1) >> 7; ++l) touch_read(l);
            }
        }
    };
    auto b_lines = [&](int n_tile, int ks) {
        int64_t row0;
        if (g.tps == 1) {
            int tap, chunk;
            if (a->order == IMCONV_ORDER_FILTER_MAJOR) {
                tap = ks / g.c_chunks;
                chunk = ks - tap * g.c_chunks;
            } else {
                chunk = ks / rs;
                tap = ks - chunk * rs;
            }
            row0 = static_cast<int64_t>(tap) * C + static_cast<int64_t>(chunk) * kbke;
        } else {
            row0 = static_cast<int64_t>(ks) * g.tps * C;
        }
        const int64_t col0 = static_cast<int64_t>(n_tile) * g.bn;
        const int64_t cols = std::min<int64_t>(g.bn, K - col0);
        for (int64_t row = row0; row < std::min<int64_t>(row0 + kbke, R * S * C); ++row) {
            const int64_t byte = (row * K + col0) * E;
            for (int64_t l = byte >> 7; l <= (byte + cols * E - 1) >> 7; ++l) touch_read(w_base + l);
        }
    };
    auto y_lines = [&](long long m_tile, int n_tile) {
        const int64_t m0 = m_tile * rows_per_tile, col0 = static_cast<int64_t>(n_tile) * g.bn;
        const int64_t cols = std::min<int64_t>(g.bn, K - col0);
        for (int64_t m = m0; m < std::min<int64_t>(m0 + rows_per_tile, M); ++m) {
            const int64_t byte = (m * K + col0) * EO;
            for (int64_t l = byte >> 7; l <= (byte + cols * EO - 1) >> 7; ++l) {
                ++requests;
                if (cap > 0) lru.access(y_base + l, true);
            }
        }
    };
    // persistent schedule: the kernel's own unit walk (conv_kernel.cuh UnitWalk)
    const long long G = g.use_pair ? g.grid / 2 : g.grid;
    const long long sk_first = g.sk_mode ? g.tiles - g.sk_tail : g.tiles;
    const int k_stages = (g.k_subs + g.ksub - 1) / g.ksub;
    struct U { long long tile; int kb0, kb1; bool stores; };
    // round r of CTA b = its r-th unit (rounds advance together in the replay)
    auto unit = [&](long long b, long long round, U &u) {
        const UnitWalk wk(b, G, g.tiles, g.sk_mode, g.sk_split, sk_first, k_stages);
        Unit w;
        if (!wk.get(round, w)) return false;
        // the output lines are written by the split that stores them (the last split, as an
        // approximation of the owner spread) or by a stream-K finisher / whole tile
        const bool stores = g.sk_mode == 1 ? (w.split < 0 || w.split == g.sk_split - 1) : w.sk != 1;
        u = {w.tile, w.kb0, w.kb1, stores};
        return true;
    };
    std::vector<uint8_t> b_loaded(static_cast<size_t>(G), 0);
    for (long long round = 0;; ++round) {
        bool any = false;
        for (int kb = 0; kb < k_stages; ++kb) {
            for (long long b = 0; b < G; ++b) {
                U u;
                if (!unit(b, round, u) || kb < u.kb0 || kb >= u.kb1) continue;
                any = true;
                const long long m_tile = u.tile / g.n_tiles;
                const int n_tile = static_cast<int>(u.tile - m_tile * g.n_tiles);
                for (int sub = 0; sub < g.ksub; ++sub) {
                    const int ks = kb * g.ksub + sub;
                    if (ks >= g.k_subs) break;
                    a_lines(m_tile, ks);
                    if (!g.b_resident || !b_loaded[static_cast<size_t>(b)]) b_lines(n_tile, ks);
                }
                if (kb == u.kb1 - 1) {
                    if (g.b_resident) b_loaded[static_cast<size_t>(b)] = 1;
                    if (u.stores) y_lines(m_tile, n_tile);
                }
            }
        }
        if (!any) break;
    }
    out->dram_read_bytes = reads * 128;
    out->dram_write_bytes = lru.dirty_evictions() * 128;
    out->resident_dirty_bytes = cap > 0 ? lru.dirty_resident() * 128 : 0;
    if (cap <= 0) out->dram_write_bytes = (M * K * EO + 127) / 128 * 128;
    out->line_requests = requests;
    out->compulsory_read_bytes = compulsory * 128;
    return 0;
}

// Argument checks shared by imconv_conv2d_nhwc and imconv_plan (the reference
// validates in ConvSpec.__post_init__, core.py:72-87; the kernel level adds the
// dtype, 16-byte and TMA im2col limits).
static int validate_conv_args(const imconv_conv_args *a, int64_t *P_out, int64_t *Q_out, bool need_ptrs) {
    if (!a) return IMCONV_EINVAL;
    if (need_ptrs && (!a->x || !a->w || !a->y)) return IMCONV_EINVAL;
    const int64_t N = a->n, H = a->h, W = a->w_, C = a->c, K = a->k, R = a->r, S = a->s;
    if (N < 1 || H < 1 || W < 1 || C < 1 || K < 1 || R < 1 || S < 1) return IMCONV_EINVAL;
    if (a->stride_h < 1 || a->stride_w < 1 || a->dil_h < 1 || a->dil_w < 1 || a->pad_h < 0 || a->pad_w < 0)
        return IMCONV_EINVAL;
    const int64_t P = imconv_out_extent(H, R, a->stride_h, a->pad_h, a->dil_h);
    const int64_t Q = imconv_out_extent(W, S, a->stride_w, a->pad_w, a->dil_w);
    if (P < 1 || Q < 1) return IMCONV_EINVAL;
    const bool f16in = a->in_dtype == IMCONV_BF16 || a->in_dtype == IMCONV_F16;
    if (!(f16in && (a->out_dtype == a->in_dtype || a->out_dtype == IMCONV_F32)) &&
        !(a->in_dtype == IMCONV_I8 && a->out_dtype == IMCONV_I32))
        return IMCONV_EDTYPE;
    if ((a->flags & IMCONV_FLAG_CHANNEL_LAST) && !f16in) return IMCONV_EDTYPE;
    const int E = elem_bytes(a->in_dtype);
    if ((C * E) % 16 != 0 || (K * E) % 16 != 0) return IMCONV_ECHAN;
    if (need_ptrs && (!aligned16(a->x) || !aligned16(a->w) || !aligned16(a->y))) return IMCONV_EALIGN;
    // TMA im2col limits for a 4-D tensor: corners in [-128,127], tap offsets
    // in [0,255], traversal stride <= 8, dims < 2^32.
    const int64_t lo_w = -a->pad_w, lo_h = -a->pad_h;
    const int64_t up_w = a->pad_w - static_cast<int64_t>(a->dil_w) * (S - 1);
    const int64_t up_h = a->pad_h - static_cast<int64_t>(a->dil_h) * (R - 1);
    if (lo_w < -128 || lo_h < -128 || up_w < -128 || up_h < -128 || up_w > 127 || up_h > 127) return IMCONV_ERANGE;
    if (static_cast<int64_t>(a->dil_w) * (S - 1) > 255 || static_cast<int64_t>(a->dil_h) * (R - 1) > 255)
        return IMCONV_ERANGE;
    if (a->stride_h > 8 || a->stride_w > 8) return IMCONV_ERANGE;
    const int64_t M = N * P * Q;
    if (M >= (1ll << 31) || R * S * C >= (1ll << 31) || H * W >= (1ll << 31)) return IMCONV_ERANGE;
    *P_out = P;
    *Q_out = Q;
    return 0;
}

// The specialised kernels, in the order imconv_conv2d_nhwc tries them (shared with
// imconv_plan, which asks the same questions with dry = true):
//   16-byte pixels -> the row-band kernel (unless the generic kernel's cp.async tap
//   gathers are requested; measured 0.47 vs 0.94 ms on the ResNet stem);
//   128-byte pixels, stride 1, filter resident in smem -> halo tiles (each input
//   pixel enters shared memory once per block, taps are descriptor offsets);
//   multi-chunk 16-bit pixels, stride 1, K <= 128 -> halo tiles with a streamed filter.
// Returns kNotApplicable when the generic kernel runs; *kernel = 1/2/3 otherwise.
static int route_special(const imconv_conv_args *a, int64_t P, int64_t Q, int sms, cudaStream_t st, bool dry,
                         int *kernel) {
    const bool cl = (a->flags & IMCONV_FLAG_CHANNEL_LAST) != 0;
    *kernel = 0;
    if (!cl && !(a->flags & IMCONV_FLAG_GATHER16) && a->order != IMCONV_ORDER_FILTER_MAJOR) {
        const int rb = try_rowband(a, P, Q, sms, st, dry);
        if (rb != kNotApplicable) {
            *kernel = 1;
            return rb;
        }
    }
    if (!cl && !(a->flags & IMCONV_FLAG_NO_HALO)) {
        const int hr = try_halo(a, P, Q, sms, st, dry);
        if (hr != kNotApplicable) {
            *kernel = 2;
            return hr;
        }
        const int hs = try_halo_stream(a, P, Q, sms, st, dry);
        if (hs != kNotApplicable) {
            *kernel = 3;
            return hs;
        }
    }
    return kNotApplicable;
}

extern "C" int imconv_plan(const imconv_conv_args *a, int32_t sms, imconv_plan_info *out) {
    if (!a || !out || sms < 1) return IMCONV_EINVAL;
    int64_t P = 0, Q = 0;
    int rc = validate_conv_args(a, &P, &Q, false);
    if (rc) return rc;
    std::memset(out, 0, sizeof(*out));
    int kernel = 0;
    if (route_special(a, P, Q, sms, nullptr, true, &kernel) != kNotApplicable) {
        out->kernel = kernel;
        out->sk_split = 1;
        return 0;
    }
    GenericPlan g;
    rc = plan_generic(a, P, Q, sms, &g);
    if (rc) return rc;
    out->kernel = 0;
    out->grid = g.grid;
    out->bn = g.bn;
    out->mt = g.mt;
    out->ksub = g.ksub;
    out->cta_pair = g.use_pair ? 1 : 0;
    out->b_resident = g.b_resident ? 1 : 0;
    out->sk_split = g.sk_split;
    out->tiles = g.tiles;
    out->sk_tail = g.sk_tail;
    out->sk_mode = g.sk_mode;
    return 0;
}

extern "C" {

int imconv_conv2d_nhwc(const imconv_conv_args *a, void *stream) {
    int64_t P = 0, Q = 0;
    int rc = validate_conv_args(a, &P, &Q, true);
    if (rc) return rc;
    const int64_t N = a->n, H = a->h, W = a->w_, C = a->c, K = a->k, R = a->r, S = a->s;
    const int E = elem_bytes(a->in_dtype);
    const int64_t lo_w = -a->pad_w, lo_h = -a->pad_h;
    const int64_t up_w = a->pad_w - static_cast<int64_t>(a->dil_w) * (S - 1);
    const int64_t up_h = a->pad_h - static_cast<int64_t>(a->dil_h) * (R - 1);
    const int64_t M = N * P * Q;

    rc = load_driver_entry_points();
    if (rc) return rc;
    int sms = 0;
    rc = sm_count_for_current_device(&sms);
    if (rc) return rc;

    const bool cl = (a->flags & IMCONV_FLAG_CHANNEL_LAST) != 0;  // (2-byte elements only: validated)
    int kernel = 0;
    const int sp = route_special(a, P, Q, sms, reinterpret_cast<cudaStream_t>(stream), false, &kernel);
    if (sp != kNotApplicable) return sp;

    GenericPlan plan;
    rc = plan_generic(a, P, Q, sms, &plan);
    if (rc) return rc;
#if IMCONV_DEBUG
    // debug builds: the planner's schedule invariants (what the kernels' waits rely on)
    {
        const long long G = plan.use_pair ? plan.grid / 2 : plan.grid;
        const char *bad = nullptr;
        if (plan.grid > sms) bad = "grid above one CTA per SM";
        else if (plan.use_pair && (plan.grid & 1)) bad = "odd grid for CTA pairs";
        else if (plan.sk_mode == 1 && (plan.sk_split < 2 || plan.sk_tail * plan.sk_split > G))
            bad = "split-K units exceed the co-resident CTAs";
        else if (plan.sk_mode == 2 && (plan.sk_tail < G || plan.sk_tail > plan.tiles))
            bad = "stream-K region shorter than one tile per CTA";
        else if (plan.sk_mode && plan.sk_tail * (plan.use_pair ? 2 : 1) > kSkSliceLen)
            bad = "split-K counters exceed one slice";
        if (bad) {
            std::fprintf(stderr, "imconv debug: planner invariant violated: %s (grid %d, tiles %lld, mode %d, S %d, tail %lld)\n",
                         bad, plan.grid, plan.tiles, plan.sk_mode, plan.sk_split, plan.sk_tail);
            return IMCONV_EINVAL;
        }
    }
#endif
    const int bn = plan.bn, variant = plan.variant, mt = plan.mt;
    const bool use_pair = plan.use_pair;

    // ---- A operand: im2col tensor map over NHWC ----
    const int64_t cbytes = C * E;
    const int row_bytes = (cl || cbytes >= 128) ? 128 : static_cast<int>(cbytes);  // 16, 32, 64 or 128
    int a_layout;
    CUtensorMapSwizzle a_swz;
    switch (row_bytes) {
        case 128: a_layout = A_SW128; a_swz = CU_TENSOR_MAP_SWIZZLE_128B; break;
        case 64: a_layout = A_SW64; a_swz = CU_TENSOR_MAP_SWIZZLE_64B; break;
        case 32: a_layout = A_SW32; a_swz = CU_TENSOR_MAP_SWIZZLE_32B; break;
        case 16: a_layout = A_NONE; a_swz = CU_TENSOR_MAP_SWIZZLE_NONE; break;
        default: return IMCONV_ECHAN;  // 48, 80, 96, 112 bytes: pad to the next power of two
    }
    const int tps = kRowBytes / row_bytes;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);

    CUtensorMap ta, tb;
    std::memset(&ta, 0, sizeof(ta));
    std::memset(&tb, 0, sizeof(tb));
    // 1x1, stride 1, no padding: the implicit im2col is the identity, so A is
    // the (N*H*W, C) activation matrix itself -- a tiled map (one TMA box of
    // 128 B of channels x 128*mt rows per k-subtile) replaces the im2col map.
    const bool a_tiled = !cl && R == 1 && S == 1 && a->stride_h == 1 && a->stride_w == 1 && a->pad_h == 0 &&
                         a->pad_w == 0 && row_bytes == 128 && !(g_debug_flags & kDbgNoTiledA);
    if (cl) {
        // channel-last baseline: A is gathered by threads (no A tensor map)
    } else if (a_tiled) {
        cuuint64_t gdim[2] = {static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(N * H * W)};
        cuuint64_t gstride[1] = {static_cast<cuuint64_t>(C * E)};
        cuuint32_t box[2] = {static_cast<cuuint32_t>(row_bytes / E), static_cast<cuuint32_t>(kBM * mt)};
        cuuint32_t estride[2] = {1, 1};
        if (g_encode_tiled(&ta, tmap_dtype(a->in_dtype), 2, const_cast<void *>(a->x), gdim, gstride, box, estride,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, a_swz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return IMCONV_ETMAP;
    } else {
        cuuint64_t gdim[4] = {static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H),
                              static_cast<cuuint64_t>(N)};
        cuuint64_t gstride[3] = {static_cast<cuuint64_t>(C * E), static_cast<cuuint64_t>(W * C * E),
                                 static_cast<cuuint64_t>(H * W * C * E)};
        int lower[2] = {static_cast<int>(lo_w), static_cast<int>(lo_h)};  // {W, H}
        int upper[2] = {static_cast<int>(up_w), static_cast<int>(up_h)};
        cuuint32_t estride[4] = {1, static_cast<cuuint32_t>(a->stride_w), static_cast<cuuint32_t>(a->stride_h), 1};
        CUresult cr = g_encode_im2col(&ta, tmap_dtype(a->in_dtype), 4, const_cast<void *>(a->x), gdim, gstride,
                                      lower, upper, static_cast<cuuint32_t>(row_bytes / E),
                                      static_cast<cuuint32_t>(kBM * mt), estride,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, a_swz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (cr != CUDA_SUCCESS) return IMCONV_ETMAP;
        // Same driver quirk CUTLASS works around for im2col maps over small
        // tensors on drivers <= 13.1 (copy_traits_sm90_im2col.hpp).
        if (g_driver_version <= 13010 && N * H * W * C * E < 131072)
            reinterpret_cast<uint64_t *>(&ta)[1] &= ~(1ull << 21);
    }
    // channel-last baseline: the filter permuted to the (c, r, s) reduction order
    void *w_cl = nullptr;
    const void *w_src = a->w;
    if (cl) {
        const size_t wbytes = static_cast<size_t>(R * S * C * K) * E;
        if (cudaMallocAsync(&w_cl, wbytes, st) != cudaSuccess) return static_cast<int>(cudaGetLastError());
        const long long work = R * S * C * K;
        permute_filter_cl_kernel<uint16_t><<<grid_for(work), 256, 0, st>>>(
            reinterpret_cast<const uint16_t *>(a->w), reinterpret_cast<uint16_t *>(w_cl), static_cast<int>(R * S),
            static_cast<int>(C), static_cast<int>(K));
        ++g_launches;
        w_src = w_cl;
    }
    // ---- B operand: the HWCN filter as (R*S*C rows, K cols).  When K is a whole
    // number of 128-byte column chunks it is viewed 3-D {chunk cols, rows, chunks}
    // so ONE TMA instruction fetches all of a stage's B chunks. ----
    const int nc = kRowBytes / E;
    const bool b_3d = (K % nc) == 0;
    {
        const int chunks_per_load = (use_pair ? bn / 2 : bn) / nc;
        CUresult cr;
        if (b_3d) {
            cuuint64_t gdim[3] = {static_cast<cuuint64_t>(nc), static_cast<cuuint64_t>(R * S * C),
                                  static_cast<cuuint64_t>(K / nc)};
            cuuint64_t gstride[2] = {static_cast<cuuint64_t>(K * E), static_cast<cuuint64_t>(nc * E)};
            cuuint32_t box[3] = {static_cast<cuuint32_t>(nc), static_cast<cuuint32_t>(kRowBytes / E),
                                 static_cast<cuuint32_t>(chunks_per_load)};
            cuuint32_t estride[3] = {1, 1, 1};
            cr = g_encode_tiled(&tb, tmap_dtype(a->in_dtype), 3, const_cast<void *>(w_src), gdim, gstride, box,
                                estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
            cuuint64_t gdim[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(R * S * C)};
            cuuint64_t gstride[1] = {static_cast<cuuint64_t>(K * E)};
            cuuint32_t box[2] = {static_cast<cuuint32_t>(nc), static_cast<cuuint32_t>(kRowBytes / E)};
            cuuint32_t estride[2] = {1, 1};
            cr = g_encode_tiled(&tb, tmap_dtype(a->in_dtype), 2, const_cast<void *>(w_src), gdim, gstride, box,
                                estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        if (cr != CUDA_SUCCESS) return IMCONV_ETMAP;
    }

    // ---- output: tiled map over y viewed as (M, K): one 128-row x 128-byte box per store ----
    CUtensorMap ty;
    std::memset(&ty, 0, sizeof(ty));
    {
        const int eo = (a->out_dtype == IMCONV_F32 || a->out_dtype == IMCONV_I32) ? 4 : 2;
        CUtensorMapDataType dt = a->out_dtype == IMCONV_F32   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : a->out_dtype == IMCONV_I32 ? CU_TENSOR_MAP_DATA_TYPE_INT32
                                 : a->out_dtype == IMCONV_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                              : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
        cuuint64_t gdim[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(M)};
        cuuint64_t gstride[1] = {static_cast<cuuint64_t>(K * eo)};
        cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / eo), 128u};
        cuuint32_t estride[2] = {1, 1};
        CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B;
        CUresult cr = g_encode_tiled(&ty, dt, 2, a->y, gdim, gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                     swz, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (cr != CUDA_SUCCESS) return IMCONV_ETMAP;
    }

    ConvParams p{};
    p.n = static_cast<int>(N);
    p.h = static_cast<int>(H);
    p.w = static_cast<int>(W);
    p.c = static_cast<int>(C);
    p.k = static_cast<int>(K);
    p.r = static_cast<int>(R);
    p.s = static_cast<int>(S);
    p.sh = a->stride_h;
    p.sw = a->stride_w;
    p.ph = a->pad_h;
    p.pw = a->pad_w;
    p.dh = a->dil_h;
    p.dw = a->dil_w;
    p.p = static_cast<int>(P);
    p.q = static_cast<int>(Q);
    p.m = M;
    p.m_tiles = static_cast<int>((M + kBM * mt * (use_pair ? 2 : 1) - 1) / (kBM * mt * (use_pair ? 2 : 1)));
    p.n_tiles = static_cast<int>((K + bn - 1) / bn);
    p.rs = static_cast<int>(R * S);
    p.tps = tps;
    p.c_chunks = tps == 1 ? static_cast<int>((cbytes + kRowBytes - 1) / kRowBytes) : 1;
    p.k_stages = tps == 1 ? p.c_chunks * p.rs : (p.rs + tps - 1) / tps;
    p.a_layout = a_layout;
    p.order = a->order == IMCONV_ORDER_FILTER_MAJOR ? 1 : 0;
    p.y = a->y;
    p.ldy = K;
    p.dbg = g_debug_buf;
    p.b_3d = b_3d ? 1 : 0;
    // bf16/fp16 C = 8 with KSUB = 1 and >= 4 stages (variants 0 and 2)
    p.a_gather = (row_bytes == 16 && E == 2 && !use_pair && variant != 1) ? 1 : 0;
    p.x = static_cast<const uint8_t *>(a->x);
    p.a_tiled = a_tiled ? 1 : 0;
    if (cl) {
        p.a_cl = 1;
        p.a_gather = 0;
        p.tps = 1;
        p.c_chunks = 1;
        p.k_stages = plan.k_subs;
    }
    p.dbg_flags = g_debug_flags & 0xff;
    p.b_early = cl ? 0 : early_mode(a->flags);

    const long long tiles = static_cast<long long>(p.m_tiles) * p.n_tiles;
    int grid = plan.grid;
    p.b_resident = plan.b_resident ? 1 : 0;

    // split-K tail (plan_generic): stream-ordered partial-sum workspace + ticket counters
    void *sk_ws = nullptr;
    p.sk_split = 1;
    p.sk_mode = 0;
    if (plan.sk_mode) {
        int dev = 0;
        cudaGetDevice(&dev);
        unsigned long long *cnt = sk_counters(dev);
        const int cg = use_pair ? 2 : 1;
        // mode 1: S partials per tail tile; mode 2: one (the writer's) per streamed tile
        const size_t ws_bytes = static_cast<size_t>(plan.sk_tail) * (plan.sk_mode == 1 ? plan.sk_split : 1) * cg *
                                (kBM * mt) * bn * 4;
        if (plan.sk_tail * cg > kSkSliceLen) return IMCONV_EINVAL;  // (planner guarantees it)
        if (cnt && cudaMallocAsync(&sk_ws, ws_bytes, st) == cudaSuccess) {
            const unsigned long long slice = g_sk_slice.fetch_add(1) % kSkSlices;
            p.sk_mode = plan.sk_mode;
            p.sk_split = plan.sk_split;
            p.sk_first = tiles - plan.sk_tail;
            p.sk_ws = static_cast<float *>(sk_ws);
            p.sk_cnt = cnt + slice * kSkSliceLen;
        } else {
            sk_ws = nullptr;
            cudaGetLastError();  // (allocation failure: run without splitting)
            grid = static_cast<int>(std::min<long long>(grid, tiles * cg));
        }
    }
    if (use_pair) {
        const int g2 = grid;
        int rc_pair;
        switch (a->in_dtype) {
            case IMCONV_BF16:
                rc_pair = a->out_dtype == IMCONV_F32 ? dispatch_bn_pair<ELEM_BF16, OUT_F32>(bn, ta, tb, ty, p, g2, st)
                                                     : dispatch_bn_pair<ELEM_BF16, OUT_BF16>(bn, ta, tb, ty, p, g2, st);
                break;
            case IMCONV_F16:
                rc_pair = a->out_dtype == IMCONV_F32 ? dispatch_bn_pair<ELEM_F16, OUT_F32>(bn, ta, tb, ty, p, g2, st)
                                                     : dispatch_bn_pair<ELEM_F16, OUT_F16>(bn, ta, tb, ty, p, g2, st);
                break;
            case IMCONV_I8: rc_pair = dispatch_bn_pair<ELEM_I8, OUT_I32>(bn, ta, tb, ty, p, g2, st); break;
            default: rc_pair = IMCONV_EDTYPE;
        }
        if (sk_ws) cudaFreeAsync(sk_ws, st);
        return rc_pair;
    }
    int rc_launch;
    switch (a->in_dtype) {
        case IMCONV_BF16:
            rc_launch = a->out_dtype == IMCONV_F32
                       ? dispatch_bn<ELEM_BF16, OUT_F32>(bn, variant, ta, tb, ty, p, grid, st)
                       : dispatch_bn<ELEM_BF16, OUT_BF16>(bn, variant, ta, tb, ty, p, grid, st);
            break;
        case IMCONV_F16:
            rc_launch = a->out_dtype == IMCONV_F32
                            ? dispatch_bn<ELEM_F16, OUT_F32>(bn, variant, ta, tb, ty, p, grid, st)
                            : dispatch_bn<ELEM_F16, OUT_F16>(bn, variant, ta, tb, ty, p, grid, st);
            break;
        case IMCONV_I8: rc_launch = dispatch_bn<ELEM_I8, OUT_I32>(bn, variant, ta, tb, ty, p, grid, st); break;
        default: rc_launch = IMCONV_EDTYPE;
    }
    if (sk_ws) cudaFreeAsync(sk_ws, st);  // stream-ordered: released after the kernel
    if (w_cl) cudaFreeAsync(w_cl, st);
    return rc_launch;
}

int imconv_gemm(const void *A, const void *B, void *Cm, int32_t in_dtype, int32_t out_dtype, int64_t m, int64_t kd,
                int64_t n, void *stream) {
    if (m < 1 || kd < 1 || n < 1) return IMCONV_EINVAL;
    // A (m, kd) row-major is an NHWC image (1, 1, m, kd); B (kd, n) is an
    // HWCN 1x1 filter; the 1x1 stride-1 convolution is exactly A @ B.
    imconv_conv_args a{};
    a.x = A;
    a.w = B;
    a.y = Cm;
    a.in_dtype = in_dtype;
    a.out_dtype = out_dtype;
    a.n = 1;
    a.h = 1;
    a.w_ = m;
    a.c = kd;
    a.k = n;
    a.r = 1;
    a.s = 1;
    a.stride_h = a.stride_w = 1;
    a.dil_h = a.dil_w = 1;
    return imconv_conv2d_nhwc(&a, stream);
}


static int launch_gather(const void *x, void *out, int32_t eb, int64_t n, int64_t h, int64_t w, int64_t c,
                         int32_t hf, int32_t wf, int32_t r_fix, int32_t s_fix, int32_t sh, int32_t sw, int32_t ph,
                         int32_t pw, int32_t dh, int32_t dw, int64_t ho, int64_t wo, int32_t channel_first,
                         cudaStream_t st) {
    const long long M = n * ho * wo;
    const long long taps = r_fix >= 0 ? 1 : static_cast<long long>(hf) * wf;
    if ((c * eb) % 16 == 0 && (channel_first || r_fix >= 0) && aligned16(x) && aligned16(out)) {
        const int c_vec = static_cast<int>(c * eb / 16);
        const long long work = M * taps * c_vec;
        im2col_cf_vec16_kernel<<<grid_for(work), 256, 0, st>>>(
            reinterpret_cast<const uint4 *>(x), reinterpret_cast<uint4 *>(out), M, static_cast<int>(h),
            static_cast<int>(w), c_vec, static_cast<int>(ho), static_cast<int>(wo), r_fix, s_fix,
            static_cast<int>(taps), wf, sh, sw, ph, pw, dh, dw);
    } else {
        const long long work = M * taps * c;
#define IMCONV_GEN(T)                                                                                          \
    im2col_generic_kernel<T><<<grid_for(work), 256, 0, st>>>(                                                   \
        reinterpret_cast<const T *>(x), reinterpret_cast<T *>(out), M, static_cast<int>(h), static_cast<int>(w), \
        static_cast<int>(c), static_cast<int>(ho), static_cast<int>(wo), hf, wf, sh, sw, ph, pw, dh, dw,        \
        channel_first, r_fix, s_fix)
        switch (eb) {
            case 1: IMCONV_GEN(uint8_t); break;
            case 2: IMCONV_GEN(uint16_t); break;
            case 4: IMCONV_GEN(uint32_t); break;
            case 8: IMCONV_GEN(unsigned long long); break;
            default: return IMCONV_EDTYPE;
        }
#undef IMCONV_GEN
    }
    ++g_launches;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : static_cast<int>(e);
}

int imconv_tile_gather_nhwc(const void *x, void *out, int32_t elem_bytes_, int64_t n, int64_t h, int64_t w_,
                            int64_t c, int32_t r, int32_t s, int32_t stride_h, int32_t stride_w, int32_t pad_h,
                            int32_t pad_w, int32_t dil_h, int32_t dil_w, int64_t ho, int64_t wo, void *stream) {
    if (!x || !out || n < 1 || h < 1 || w_ < 1 || c < 1 || ho < 1 || wo < 1 || r < 0 || s < 0) return IMCONV_EINVAL;
    if (stride_h < 1 || stride_w < 1 || dil_h < 1 || dil_w < 1 || pad_h < 0 || pad_w < 0) return IMCONV_EINVAL;
    return launch_gather(x, out, elem_bytes_, n, h, w_, c, 1, 1, r, s, stride_h, stride_w, pad_h, pad_w, dil_h, dil_w,
                         ho, wo, 1, reinterpret_cast<cudaStream_t>(stream));
}

int imconv_im2col_nhwc(const void *x, void *out, int32_t elem_bytes_, int64_t n, int64_t h, int64_t w_, int64_t c,
                       int32_t hf, int32_t wf, int32_t stride_h, int32_t stride_w, int32_t pad_h, int32_t pad_w,
                       int32_t dil_h, int32_t dil_w, int32_t channel_first, void *stream) {
    if (!x || !out || n < 1 || h < 1 || w_ < 1 || c < 1 || hf < 1 || wf < 1) return IMCONV_EINVAL;
    if (stride_h < 1 || stride_w < 1 || dil_h < 1 || dil_w < 1 || pad_h < 0 || pad_w < 0) return IMCONV_EINVAL;
    const int64_t ho = imconv_out_extent(h, hf, stride_h, pad_h, dil_h);
    const int64_t wo = imconv_out_extent(w_, wf, stride_w, pad_w, dil_w);
    if (ho < 1 || wo < 1) return IMCONV_EINVAL;
    return launch_gather(x, out, elem_bytes_, n, h, w_, c, hf, wf, -1, -1, stride_h, stride_w, pad_h, pad_w, dil_h,
                         dil_w, ho, wo, channel_first ? 1 : 0, reinterpret_cast<cudaStream_t>(stream));
}

int imconv_pad_copy(const void *src, void *dst, int32_t eb, int64_t outer, int64_t c, int64_t d, int64_t c_pad,
                    int64_t d_pad, void *stream) {
    if (!src || !dst || outer < 1 || c < 1 || d < 1 || c_pad < c || d_pad < d) return IMCONV_EINVAL;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const long long work = outer * c_pad * d_pad;
#define IMCONV_PAD(T)                                                                                     \
    pad_copy_kernel<T><<<grid_for(work), 256, 0, st>>>(reinterpret_cast<const T *>(src),                  \
                                                       reinterpret_cast<T *>(dst), outer, static_cast<int>(c), \
                                                       static_cast<int>(d), static_cast<int>(c_pad),           \
                                                       static_cast<int>(d_pad))
    switch (eb) {
        case 1: IMCONV_PAD(uint8_t); break;
        case 2: IMCONV_PAD(uint16_t); break;
        case 4: IMCONV_PAD(uint32_t); break;
        default: return IMCONV_EDTYPE;
    }
#undef IMCONV_PAD
    ++g_launches;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : static_cast<int>(e);
}

}  // extern "C"
