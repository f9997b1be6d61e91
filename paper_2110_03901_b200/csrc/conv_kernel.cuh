// conv_kernel.cuh -- the blocked channel-first implicit-im2col convolution
// (arXiv 2110.03901 §5) as a persistent, warp-specialised tcgen05 kernel.
//
// GEMM view: row m = (n*P + p)*Q + q of the output,
// reduction index k = (r*S + s)*C + c (channel-first), B = HWCN filter
// reshaped to (R*S*C, K).  The lowered matrix is never materialised: for
// every (output block, k-subtile) the TMA engine gathers the block's 128
// output pixels for one filter tap <r,s> and one channel chunk straight from
// the NHWC tensor into a swizzled shared-memory tile (im2col mode: the base
// pixel is (q*sw - pw, p*sh - ph) and the tap enters as the im2col offset
// (s*dw, r*dh); out-of-image pixels are zero-filled by the hardware, which is
// the reference's "virtual padding", lowering.py:59-64).
//
// Warp roles (256 threads, one CTA per SM, persistent over output blocks):
//   warp 0      : TMA producer (one elected lane)       -- operand generation
//   warp 1      : tcgen05.mma issuer (one elected lane) -- contraction into TMEM
//   warp 2      : TMEM allocator
//   warps 4..7  : epilogue, TMEM -> registers -> NHWC global stores
// Pipelines: STAGES-deep smem ring (full/empty mbarriers, TMA complete_tx and
// tcgen05.commit), and a 2-deep TMEM accumulator ring (tfull/tempty) so the
// epilogue of block i overlaps the main loop of block i+1.
//
// k-subtile order inside a block follows blocksched.order_subtiles
// (blocksched.py:83-99): REUSE_AWARE = channel chunk outer / tap inner (the
// paper's reordering, consecutive taps re-read ~(S-1)/S of the same input
// window from L1/L2); FILTER_MAJOR = tap outer.  Blocks are rasterised
// m-major with the n-blocks of one m-block adjacent in the schedule, so the
// CTAs working on one input window at the same time share it through L2.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <type_traits>

#include "ptx.cuh"

namespace imconv {

constexpr int kBM = 128;           // output pixels per block (MMA M)
constexpr int kRowBytes = 128;     // bytes of reduction per stage per row (one 128B swizzle span)
constexpr int kAStage = kBM * kRowBytes;  // 16 KiB of A per stage
constexpr int kThreads = 256;

enum ElemKind : int { ELEM_BF16 = 0, ELEM_F16 = 1, ELEM_I8 = 2 };
enum OutKind : int { OUT_BF16 = 0, OUT_F16 = 1, OUT_F32 = 2, OUT_I32 = 3 };
enum ALayout : int { A_NONE = 0, A_SW32 = 1, A_SW64 = 2, A_SW128 = 3 };

struct ConvParams {
    int n, h, w, c;      // input extents (c as stored, 16-byte aligned)
    int k;               // output channels (as stored in y)
    int r, s;            // filter
    int sh, sw, ph, pw, dh, dw;
    int p, q;            // output spatial extents
    long long m;         // n*p*q
    int m_tiles, n_tiles;
    int rs;              // r*s
    int tps;             // filter taps per pipeline stage (1 when c*elem >= 128)
    int c_chunks;        // channel chunks per tap (tps == 1)
    int k_stages;        // pipeline stages per output block
    int a_layout;        // ALayout of the A tile
    int order;           // 0 reuse-aware, 1 filter-major
    void *y;
    long long ldy;       // = k
    long long *dbg;      // optional per-CTA role / wait-cycle counters (instrumentation), else nullptr
    int b_3d;            // 1: the filter map is 3-D {chunk cols, rows, chunks}: one TMA per stage for all of B
};

// Division-free walk over the k-subtiles (filter tap <r,s>, channel chunk) of
// one output block, in the order of blocksched.order_subtiles: REUSE_AWARE =
// chunk outer / tap inner, FILTER_MAJOR = tap outer / chunk inner.  (The
// producer thread's per-stage instruction latency, not TMA bandwidth, bounds
// the pipeline -- tools/tma_bench.cu -- so no runtime divisions here.)
struct KWalk {
    int chunk, r, s, tap;
    __device__ __forceinline__ void reset() { chunk = r = s = tap = 0; }
    __device__ __forceinline__ void next(int order, int R, int S, int c_chunks) {
        if (order == 0) {
            ++tap;
            if (++s == S) {
                s = 0;
                if (++r == R) {
                    r = 0;
                    tap = 0;
                    ++chunk;
                }
            }
        } else {
            if (++chunk == c_chunks) {
                chunk = 0;
                ++tap;
                if (++s == S) {
                    s = 0;
                    ++r;
                }
            }
        }
    }
};

// Instrumentation (IMCONV_INSTRUMENT builds only, libimconv_instr.so): cycles
// spent in blocking waits per role; production builds compile to a plain wait.
__device__ __forceinline__ void timed_wait_g(uint64_t *bar, uint32_t parity, long long &acc) {
#if IMCONV_INSTRUMENT
    const long long t0 = clock64();
    ptx::mbar_wait(bar, parity);
    acc += clock64() - t0;
#else
    (void)acc;
    ptx::mbar_wait(bar, parity);
#endif
}

template <int ELEM>
struct ElemTraits;
template <>
struct ElemTraits<ELEM_BF16> {
    static constexpr int kBytes = 2;
    static constexpr uint32_t kFmt = 1;  // BF16
};
template <>
struct ElemTraits<ELEM_F16> {
    static constexpr int kBytes = 2;
    static constexpr uint32_t kFmt = 0;  // F16
};
template <>
struct ElemTraits<ELEM_I8> {
    static constexpr int kBytes = 1;
    static constexpr uint32_t kFmt = 1;  // signed 8-bit
};

// tcgen05 instruction descriptor: A K-major, B MN-major (HWCN filter rows
// are contiguous over the output channel), M = 128, N = BN.
template <int ELEM, int BN>
__device__ __forceinline__ uint32_t make_idesc() {
    uint32_t d = 0;
    d |= (ELEM == ELEM_I8 ? 2u : 1u) << 4;          // D format: S32 / F32
    d |= ElemTraits<ELEM>::kFmt << 7;               // A format
    d |= ElemTraits<ELEM>::kFmt << 10;              // B format
    d |= 0u << 15;                                  // A major: K
    d |= 1u << 16;                                  // B major: MN
    d |= static_cast<uint32_t>(BN >> 3) << 17;      // N
    d |= static_cast<uint32_t>(kBM >> 4) << 24;     // M
    return d;
}

template <int OUT>
struct OutTraits {
    static constexpr int kBytes = (OUT == OUT_BF16 || OUT == OUT_F16) ? 2 : 4;
    static constexpr int kRowBytes = 32 * kBytes;  // one 32-column epilogue chunk of one output row
};

// Convert one row's 32 accumulator words and write them into the warp's
// staging tile (32 rows x kRowBytes) in the TMA swizzle layout: SW64 for
// 16-bit outputs (Swizzle<2,4,3>), SW128 for 32-bit outputs (Swizzle<3,4,3>).
template <int OUT>
__device__ __forceinline__ void stage_row_chunk(uint8_t *buf, uint32_t row, const uint32_t (&v)[32]) {
    constexpr int RB = OutTraits<OUT>::kRowBytes;
    uint8_t *dst = buf + row * RB;
    if constexpr (OUT == OUT_BF16 || OUT == OUT_F16) {
        uint32_t packed[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const float a = __uint_as_float(v[2 * i]), b = __uint_as_float(v[2 * i + 1]);
            if constexpr (OUT == OUT_BF16) {
                __nv_bfloat162 t = __floats2bfloat162_rn(a, b);
                packed[i] = *reinterpret_cast<uint32_t *>(&t);
            } else {
                __half2 t = __floats2half2_rn(a, b);
                packed[i] = *reinterpret_cast<uint32_t *>(&t);
            }
        }
        const uint32_t swz = (row >> 1) & 3;
#pragma unroll
        for (uint32_t c = 0; c < 4; ++c)
            *reinterpret_cast<uint4 *>(dst + ((c ^ swz) << 4)) =
                make_uint4(packed[4 * c], packed[4 * c + 1], packed[4 * c + 2], packed[4 * c + 3]);
    } else {
        const uint32_t swz = row & 7;
#pragma unroll
        for (uint32_t c = 0; c < 8; ++c)
            *reinterpret_cast<uint4 *>(dst + ((c ^ swz) << 4)) = make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
    }
}

template <int ELEM, int OUT, int BN, int STAGES>
struct ConvCfg {
    static constexpr int kE = ElemTraits<ELEM>::kBytes;
    static constexpr int kBKE = kRowBytes / kE;      // reduction elements per stage
    static constexpr int kNC = kRowBytes / kE;       // n-chunk of one MN-major SW128 atom column
    static constexpr int kBStage = BN * kRowBytes;   // bytes of B per stage
    static constexpr int kMmaK = 32 / kE;            // reduction elements per tcgen05.mma
    static constexpr int kMmaPerStage = kBKE / kMmaK;  // = 4
    static constexpr int kTmemCols = 2 * BN;         // double-buffered accumulator
    static constexpr int kStageOut = 2 * 32 * OutTraits<OUT>::kRowBytes;  // per epilogue warp: 2 buffers
    static constexpr int kSmemBytes = STAGES * (kAStage + kBStage) + 4 * kStageOut + 1024 /*align*/ + 256 /*barriers*/;
    static_assert(BN % kNC == 0, "BN must be a multiple of the swizzle atom width");
    static_assert(kTmemCols == 128 || kTmemCols == 256 || kTmemCols == 512, "TMEM columns");
};

template <int ELEM, int OUT, int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    conv_fwd_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                    const __grid_constant__ CUtensorMap tmap_y, const ConvParams p) {
    using Cfg = ConvCfg<ELEM, OUT, BN, STAGES>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *smem_a = smem;
    uint8_t *smem_b = smem + STAGES * kAStage;
    uint8_t *smem_out = smem_b + STAGES * Cfg::kBStage;  // epilogue staging, 1024-aligned
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_out + 4 * Cfg::kStageOut);
    uint64_t *full = bars;
    uint64_t *empty = bars + STAGES;
    uint64_t *tfull = bars + 2 * STAGES;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const long long total_tiles = static_cast<long long>(p.m_tiles) * p.n_tiles;

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmap_a);
        ptx::prefetch_tmap(&tmap_b);
        ptx::prefetch_tmap(&tmap_y);
        for (int i = 0; i < STAGES; ++i) {
            ptx::mbar_init(&full[i], 2);  // A producer + B producer
            ptx::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&tfull[i], 1);
            ptx::mbar_init(&tempty[i], 4);  // one arrival per epilogue warp
        }
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc<Cfg::kTmemCols>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0 || warp == 3) {
        // ============ TMA producers: warp 0 = activations (im2col), warp 3 = filter ============
        // Two issuing threads so A and B loads leave the SM in parallel; each
        // arms the stage's `full` barrier with its own byte count.
        if (lane == 0) {
            const bool is_a = warp == 0;
            const uint64_t pol = is_a ? ptx::policy_evict_normal() : ptx::policy_evict_last();
            const int pq = p.p * p.q;
            int stage = 0;
            uint32_t phase = 0;
            long long w_empty = 0;
            const long long t_start = clock64();
            KWalk kw;
            for (long long tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
                const long long m_tile = tile / p.n_tiles;
                const int n_tile = static_cast<int>(tile - m_tile * p.n_tiles);
                const long long m0 = m_tile * kBM;
                const int n0 = static_cast<int>(m0 / pq);
                const int rem = static_cast<int>(m0 - static_cast<long long>(n0) * pq);
                const int p0 = rem / p.q;
                const int q0 = rem - p0 * p.q;
                const int w0 = q0 * p.sw - p.pw;  // base pixel (im2col bounding-box coordinates)
                const int h0 = p0 * p.sh - p.ph;
                const int nb0 = n_tile * BN;
                kw.reset();
                for (int kb = 0; kb < p.k_stages; ++kb) {
                    timed_wait_g(&empty[stage], phase ^ 1, w_empty);
                    ptx::mbar_arrive_expect_tx(&full[stage], is_a ? kAStage : Cfg::kBStage);
                    if (p.tps == 1) {
                        const int c0 = kw.chunk * Cfg::kBKE;
                        if (is_a) {
                            ptx::tma_load_im2col_4d(smem_a + stage * kAStage, &tmap_a, &full[stage], c0, w0, h0, n0,
                                                    static_cast<uint16_t>(kw.s * p.dw),
                                                    static_cast<uint16_t>(kw.r * p.dh), pol);
                        } else {
                            const int brow = kw.tap * p.c + c0;
                            uint8_t *b_dst = smem_b + stage * Cfg::kBStage;
                            if (p.b_3d) {
                                ptx::tma_load_3d(b_dst, &tmap_b, &full[stage], 0, brow, nb0 / Cfg::kNC, pol);
                            } else {
#pragma unroll
                                for (int j = 0; j < BN / Cfg::kNC; ++j)
                                    ptx::tma_load_2d(b_dst + j * (Cfg::kBKE * kRowBytes), &tmap_b, &full[stage],
                                                     nb0 + j * Cfg::kNC, brow, pol);
                            }
                        }
                        kw.next(p.order, p.r, p.s, p.c_chunks);
                    } else {
                        // small-C layers: pack tps taps side by side along the
                        // reduction (the paper's multi-tile packing, §4.2)
                        const int tap0 = kb * p.tps;
                        if (is_a) {
                            const int blk = kAStage / p.tps;
                            for (int t = 0; t < p.tps; ++t) {
                                const int tap = min(tap0 + t, p.rs - 1);  // past-the-end taps meet zero filter rows
                                const int r = tap / p.s, s = tap - (tap / p.s) * p.s;
                                ptx::tma_load_im2col_4d(smem_a + stage * kAStage + t * blk, &tmap_a, &full[stage], 0,
                                                        w0, h0, n0, static_cast<uint16_t>(s * p.dw),
                                                        static_cast<uint16_t>(r * p.dh), pol);
                            }
                        } else {
                            const int brow = tap0 * p.c;
                            uint8_t *b_dst = smem_b + stage * Cfg::kBStage;
                            if (p.b_3d) {
                                ptx::tma_load_3d(b_dst, &tmap_b, &full[stage], 0, brow, nb0 / Cfg::kNC, pol);
                            } else {
#pragma unroll
                                for (int j = 0; j < BN / Cfg::kNC; ++j)
                                    ptx::tma_load_2d(b_dst + j * (Cfg::kBKE * kRowBytes), &tmap_b, &full[stage],
                                                     nb0 + j * Cfg::kNC, brow, pol);
                            }
                        }
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
            if (IMCONV_INSTRUMENT && p.dbg && is_a) {
                p.dbg[blockIdx.x * 8 + 0] = clock64() - t_start;
                p.dbg[blockIdx.x * 8 + 1] = w_empty;
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ===================== tcgen05 MMA issuer =====================
        const uint32_t idesc = make_idesc<ELEM, BN>();
        uint32_t a_lbo, a_sbo, a_layout;
        switch (p.a_layout) {
            case A_SW128: a_lbo = 16; a_sbo = 1024; a_layout = ptx::LAYOUT_SW128; break;
            case A_SW64: a_lbo = 16; a_sbo = 512; a_layout = ptx::LAYOUT_SW64; break;
            case A_SW32: a_lbo = 16; a_sbo = 256; a_layout = ptx::LAYOUT_SW32; break;
            default: a_lbo = kBM * 16; a_sbo = 128; a_layout = ptx::LAYOUT_NONE; break;
        }
        // descriptors built once; per MMA only the 14-bit start-address field
        // moves (stage and k-step offsets >> 4 are added to the low word)
        uint32_t a_kk[Cfg::kMmaPerStage];
#pragma unroll
        for (int kk = 0; kk < Cfg::kMmaPerStage; ++kk) {
            uint32_t off;
            switch (p.a_layout) {
                case A_SW128: off = kk * 32; break;
                case A_SW64: off = (kk >> 1) * (kBM * 64) + (kk & 1) * 32; break;
                case A_SW32: off = kk * (kBM * 32); break;
                default: off = kk * 2 * (kBM * 16); break;
            }
            a_kk[kk] = off >> 4;
        }
        const uint64_t adesc0 = ptx::smem_desc(ptx::smem_u32(smem_a), a_lbo, a_sbo, a_layout);
        const uint64_t bdesc0 =
            ptx::smem_desc(ptx::smem_u32(smem_b), Cfg::kBKE * kRowBytes, 1024, ptx::LAYOUT_SW128);
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        long long w_tempty = 0, w_full = 0;
        const long long t_start = clock64();
        for (long long tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
            timed_wait_g(&tempty[acc], acc_phase ^ 1, w_tempty);
            ptx::tc_fence_after();
            const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
            for (int kb = 0; kb < p.k_stages; ++kb) {
                timed_wait_g(&full[stage], phase, w_full);
                ptx::tc_fence_after();
                if (lane == 0) {
                    const uint64_t a_st = adesc0 + static_cast<uint64_t>((stage * kAStage) >> 4);
                    const uint64_t b_st = bdesc0 + static_cast<uint64_t>((stage * Cfg::kBStage) >> 4);
#pragma unroll
                    for (int kk = 0; kk < Cfg::kMmaPerStage; ++kk) {
                        const uint64_t adesc = a_st + a_kk[kk];
                        const uint64_t bdesc = b_st + static_cast<uint64_t>((kk * Cfg::kMmaK * kRowBytes) >> 4);
                        const uint32_t accum = (kb | kk) != 0 ? 1u : 0u;
                        if constexpr (ELEM == ELEM_I8)
                            ptx::mma_i8(d_tmem, adesc, bdesc, idesc, accum);
                        else
                            ptx::mma_f16(d_tmem, adesc, bdesc, idesc, accum);
                    }
                    ptx::mma_commit(&empty[stage]);  // frees the smem slot once these MMAs retire
                }
                __syncwarp();
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (lane == 0) ptx::mma_commit(&tfull[acc]);  // accumulator complete -> epilogue
            __syncwarp();
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
        if (IMCONV_INSTRUMENT && p.dbg && lane == 0) {
            p.dbg[blockIdx.x * 8 + 2] = clock64() - t_start;
            p.dbg[blockIdx.x * 8 + 3] = w_tempty;
            p.dbg[blockIdx.x * 8 + 4] = w_full;
        }
    } else if (warp >= 4) {
        // ============ epilogue: TMEM -> registers -> swizzled smem -> TMA store ============
        const int quarter = warp & 3;  // TMEM lanes [32*quarter, 32*quarter+32) = block rows
        uint8_t *stage_buf = smem_out + quarter * Cfg::kStageOut;
        constexpr int kBuf = 32 * OutTraits<OUT>::kRowBytes;
        int acc = 0;
        uint32_t acc_phase = 0;
        uint32_t chunk_ctr = 0;
        long long w_tfull = 0;
        const long long t_start = clock64();
        for (long long tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
            const long long m_tile = tile / p.n_tiles;
            const int n_tile = static_cast<int>(tile - m_tile * p.n_tiles);
            const int row0 = static_cast<int>(m_tile * kBM) + quarter * 32;
            timed_wait_g(&tfull[acc], acc_phase, w_tfull);
            ptx::tc_fence_after();
#pragma unroll 1
            for (int j = 0; j < BN / 32; ++j) {
                const int col0 = n_tile * BN + j * 32;
                uint32_t v[32];
                const uint32_t taddr =
                    tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(acc * BN + j * 32);
                ptx::tmem_ld_32x32b_x32(taddr, v);
                ptx::tmem_ld_wait();
                if (col0 >= p.k) continue;  // warp-uniform: whole chunk past the last channel
                uint8_t *buf = stage_buf + (chunk_ctr & 1) * kBuf;
                if (lane == 0) ptx::tma_store_wait_read<1>();  // the store issued 2 chunks ago has read buf
                __syncwarp();
                stage_row_chunk<OUT>(buf, lane, v);
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    ptx::tma_store_2d(&tmap_y, buf, col0, row0);  // rows >= M / cols >= K are clipped
                    ptx::tma_store_commit();
                }
                ++chunk_ctr;
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
        if (lane == 0) ptx::tma_store_wait<0>();
        __syncwarp();
        if (IMCONV_INSTRUMENT && p.dbg && lane == 0 && quarter == 0) {
            p.dbg[blockIdx.x * 8 + 5] = clock64() - t_start;
            p.dbg[blockIdx.x * 8 + 6] = w_tfull;
        }
    }

    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<Cfg::kTmemCols>(tmem_base);
    }
}

}  // namespace imconv
