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
// Warp roles (320 threads, one CTA per SM, persistent over output blocks):
//   warps 0, 2  : A (activation) TMA producers, even / odd stages (one lane each)
//   warps 3, 8  : B (filter) TMA producers, even / odd stages
//   warp 1      : tcgen05.mma issuer (warp-uniform issue, one elected lane)
//   warp 2      : also the TMEM allocator
//   warps 4..7  : epilogue, TMEM -> registers -> swizzled smem staging tiles
//   warp 9      : output store issuer (one TMA store per staged 128 x 128-byte tile)
// Pipelines: STAGES-deep smem ring (full/empty mbarriers, TMA complete_tx and
// tcgen05.commit), a 2-deep TMEM accumulator ring (tfull/tempty) so the
// epilogue of block i overlaps the main loop of block i+1, and two staging
// tiles between the epilogue and the store warp (named barriers).  CG = 2
// runs the block on a CTA pair (cta_group::2); split-K tail units and the
// B-stationary mode are described at their code below.
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
constexpr int kThreadsRowband = 320;  // conv_rowband_kernel: plane producers 0/2/3/8, issuer 1, epilogue 4-7, stores 9
constexpr int kThreadsGeneric = 320;  // + warp 8: second filter producer, warp 9: output store issuer

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
    int a_gather;        // 1: 16-byte pixels -- A tap blocks gathered by cp.async warps instead of TMA
    const uint8_t *x;    // NHWC input (gather mode)
    int sk_mode;         // 0 whole tiles, 1 split-K tail, 2 stream-K (UnitWalk)
    int sk_split;        // mode 1: S > 1 splits each of the last (total - sk_first) tiles' k-loop S ways
    long long sk_first;  // modes 1 / 2: first tile of the split / streamed tail
    float *sk_ws;        // fp32 partials [tail tile][S][MT*128 rows][BN]
    unsigned long long *sk_cnt;  // per tail tile ticket counters (monotonic, see sk_arrive)
    int b_resident;      // 1: grid is a multiple of n_tiles (each CTA keeps one output-channel block) --
                         //    when a block's k-subtiles fit the B ring, its filter slice is loaded once
    int a_cl;            // 1: channel-last baseline -- reduction order k = (c*R + r)*S + s, A gathered
                         //    element by element by threads (B = the filter permuted to that order)
    int a_tiled;         // 1: 1x1 / stride 1 / no padding -- A is the plain (M x C) matrix, loaded with
                         //    tiled TMA boxes {128 B of channels, rows} (cheaper per operation than im2col)
    int dbg_flags;       // instrumentation builds only: 1 / 2 = load B / A on a CTA's first tile only
                         // (wrong results; measures what the operand stream costs)
    int b_early;         // 2: independent launch -- no role waits for the preceding grid;
                         // 1: the filter is not written by the preceding grid -- the B producers
                         //    start before griddepcontrol.wait (PDL) and prefetch their ring stages
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

// Work units of one persistent CTA (or CTA pair): every role walks the same
// sequence, unit ul = 0, 1, 2, ... of CTA c out of G.
//
// mode 0: whole tiles round-robin: tile c + ul * G.
// mode 1 (split-K tail, last wave at most half full): the tiles [sk_first, total)
//   are split S ways and their units come FIRST -- global unit v = c + ul * G <
//   tail*S is split v % S of tile sk_first + v / S over k-stages [kb0, kb1) --
//   then the whole tiles [0, sk_first).  A split unit is therefore the first
//   unit of its CTA (tail*S <= G): the splits of a tile start at launch and
//   arrive together, and their partial-sum exchange runs in the epilogue warps
//   while the MMA warp already streams the CTA's next tile into the other TMEM
//   accumulator.
// mode 2 (stream-K, last wave more than half full): the last partial wave plus
//   one full wave, tiles [sk_first, total), are one stream of
//   W = (total - sk_first) * k_stages k-stages cut into G equal contiguous
//   ranges, CTA c taking [c*W/G, (c+1)*W/G) FIRST, then the whole tiles
//   c + j*G < sk_first.  A range is at least one tile long, so a tile is cut at
//   most once: its k-end piece starts some CTA's range (the "writer": partial
//   sums -> workspace, early) and its k-start piece ends the previous CTA's
//   range (the "finisher": adds the writer's partial to its own and stores,
//   while the MMA warp runs the CTA's whole tiles).
struct Unit {
    long long tile;
    int kb0, kb1, split;  // split < 0: the whole tile (or a stream-K piece)
    int sk;               // stream-K piece: 0 none, 1 writer (k-end piece), 2 finisher (k-start piece)
};
struct UnitWalk {
    long long c, G, total, sk_first;
    int mode, S, k_stages;
    long long lo, hi;  // mode 2: this CTA's stream range
    __host__ __device__ __forceinline__ UnitWalk(long long c_, long long G_, long long total_, int mode_, int S_,
                                                  long long sk_first_, int k_stages_)
        : c(c_), G(G_), total(total_), sk_first(sk_first_), mode(mode_), S(S_), k_stages(k_stages_), lo(0), hi(0) {
        if (mode == 2) {
            const long long W = (total - sk_first) * k_stages;
            lo = c * W / G;
            hi = (c + 1) * W / G;
        }
    }
    __host__ __device__ __forceinline__ bool get(long long ul, Unit &w) const {
        w.sk = 0;
        w.split = -1;
        if (mode == 1) {
            const long long u = c + ul * G;
            const long long n_split = (total - sk_first) * S;
            if (u < n_split) {
                w.tile = sk_first + u / S;
                w.split = static_cast<int>(u % S);
                w.kb0 = w.split * k_stages / S;
                w.kb1 = (w.split + 1) * k_stages / S;
                return true;
            }
            const long long t = u - n_split;
            if (t >= sk_first) return false;
            w.tile = t;
            w.kb0 = 0;
            w.kb1 = k_stages;
            return true;
        }
        if (mode == 2) {
            // segments of [lo, hi): the first starts at lo, later ones at tile boundaries
            const long long first_tile = lo / k_stages;
            const long long start = ul == 0 ? lo : (first_tile + ul) * k_stages;
            if (start < hi) {
                const long long t = start / k_stages;
                const long long end = hi < (t + 1) * k_stages ? hi : (t + 1) * k_stages;
                w.tile = sk_first + t;
                w.kb0 = static_cast<int>(start - t * k_stages);
                w.kb1 = static_cast<int>(end - t * k_stages);
                w.sk = (w.kb0 > 0) ? 1 : (w.kb1 < k_stages ? 2 : 0);
                return true;
            }
            const long long n_seg = (hi - 1) / k_stages - first_tile + 1;  // (hi > lo: ranges >= one tile)
            const long long t = c + (ul - n_seg) * G;
            if (t >= sk_first) return false;
            w.tile = t;
            w.kb0 = 0;
            w.kb1 = k_stages;
            return true;
        }
        const long long t = c + ul * G;
        if (t >= total) return false;
        w.tile = t;
        w.kb0 = 0;
        w.kb1 = k_stages;
        return true;
    }
};

// Arrival of one split on its tail tile's ticket counter.  Counters only grow:
// between launches a slot holds a multiple of kSkRound; inside a launch each of
// the S (<= 5) splits adds 1 and the split that completes the set rounds the slot
// up to the next multiple.  Nothing is ever cleared and no launch-specific value
// is baked into the parameters, so a CUDA graph replaying the same launch again
// and again (bench.py's timed step) sees a fresh count every time.  Returns the
// value that proves all S splits of THIS launch have arrived; `last` is set for
// the completing arrival.
constexpr unsigned long long kSkRound = 64;
__device__ __forceinline__ unsigned long long sk_arrive(unsigned long long *slot, int S, bool &last) {
    const unsigned long long old = atomicAdd(slot, 1ull);
    const unsigned long long base = old & ~(kSkRound - 1);
    IMCONV_CHECK(old - base < static_cast<unsigned long long>(S), "split-K ticket: more arrivals than splits in a round",
                 old, S);
    last = old - base == static_cast<unsigned long long>(S - 1);
    if (last) atomicAdd(slot, kSkRound - static_cast<unsigned long long>(S));
    return base + static_cast<unsigned long long>(S);
}

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

// Launch timeline (IMCONV_INSTRUMENT builds, CTA 0 only): globaltimer stamps of
// one launch's phases into dbg[148*20 + 1 + (launch % 64) * 8 + event];
// dbg[148*20] counts launches.  Events: 0 entry, 1 after griddepcontrol.wait,
// 2 first operands landed (MMA warp), 3 last MMA commit, 4 first accumulator
// ready (epilogue), 5 last output store complete, 6 exit.
__device__ __forceinline__ void tl_stamp(long long *dbg, uint32_t idx, int ev) {
#if IMCONV_INSTRUMENT
    if (dbg && blockIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        dbg[148 * 20 + 1 + (idx % 64) * 8 + ev] = static_cast<long long>(t);
    }
#else
    (void)dbg, (void)idx, (void)ev;
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
template <int ELEM, int BN, int M = kBM>
__device__ __forceinline__ uint32_t make_idesc() {
    uint32_t d = 0;
    d |= (ELEM == ELEM_I8 ? 2u : 1u) << 4;          // D format: S32 / F32
    d |= ElemTraits<ELEM>::kFmt << 7;               // A format
    d |= ElemTraits<ELEM>::kFmt << 10;              // B format
    d |= 0u << 15;                                  // A major: K
    d |= 1u << 16;                                  // B major: MN
    d |= static_cast<uint32_t>(BN >> 3) << 17;      // N
    d |= static_cast<uint32_t>(M >> 4) << 24;       // M (256: CTA pair, cta_group::2)
    return d;
}

template <int OUT>
struct OutTraits {
    static constexpr int kBytes = (OUT == OUT_BF16 || OUT == OUT_F16) ? 2 : 4;
    static constexpr int kRowBytes = 32 * kBytes;  // one 32-column epilogue chunk of one output row
};

// One 128-byte row of a 128-row output staging tile in the SW128 TMA layout
// (16-byte chunk c of row r lives at ((c ^ (r & 7)) * 16)): 64 bf16/fp16 or
// 32 fp32/int32 accumulator columns.
template <int OUT>
__device__ __forceinline__ void stage_row128(uint8_t *tile, uint32_t row, const uint32_t *v) {
    uint8_t *dst = tile + row * 128;
    const uint32_t swz = row & 7;
    if constexpr (OUT == OUT_BF16 || OUT == OUT_F16) {
#pragma unroll
        for (uint32_t c = 0; c < 8; ++c) {
            uint32_t w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float a = __uint_as_float(v[8 * c + 2 * i]), b = __uint_as_float(v[8 * c + 2 * i + 1]);
                if constexpr (OUT == OUT_BF16) {
                    __nv_bfloat162 t = __floats2bfloat162_rn(a, b);
                    w[i] = *reinterpret_cast<uint32_t *>(&t);
                } else {
                    __half2 t = __floats2half2_rn(a, b);
                    w[i] = *reinterpret_cast<uint32_t *>(&t);
                }
            }
            *reinterpret_cast<uint4 *>(dst + ((c ^ swz) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
    } else {
#pragma unroll
        for (uint32_t c = 0; c < 8; ++c)
            *reinterpret_cast<uint4 *>(dst + ((c ^ swz) << 4)) =
                make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
    }
}

template <int ELEM, int OUT, int BN, int STAGES, int KSUB = 1, int MT = 1, int CG = 1>
struct ConvCfg {
    static constexpr int kE = ElemTraits<ELEM>::kBytes;
    static constexpr int kBKE = kRowBytes / kE;      // reduction elements per k-subtile
    static constexpr int kNC = kRowBytes / kE;       // n-chunk of one MN-major SW128 atom column
    static constexpr int kRows = MT * kBM;           // output pixels per CTA block (MT accumulators)
    static constexpr int kASub = MT * kAStage;       // bytes of A per k-subtile (one im2col box of kRows pixels)
    static constexpr int kBSub = (BN / CG) * kRowBytes;  // bytes of B per k-subtile (per CTA of a pair)
    static constexpr int kAStageK = KSUB * kASub;    // a pipeline stage carries KSUB k-subtiles
    static constexpr int kBStage = KSUB * kBSub;
    static constexpr int kMmaK = 32 / kE;            // reduction elements per tcgen05.mma
    static constexpr int kMmaPerSub = kBKE / kMmaK;  // = 4
    static constexpr int kMmaPerStage = kMmaPerSub;  // (per k-subtile and m-tile)
    static constexpr int kTmemCols = 2 * MT * BN;    // double-buffered accumulators
    // epilogue: two 128-row x 128-byte staging tiles, one TMA store each
    static constexpr int kOutCols = (OUT == OUT_BF16 || OUT == OUT_F16) ? 64 : 32;
    static constexpr int kOutTile = kBM * 128;
    static constexpr int kStageOut = 2 * 32 * OutTraits<OUT>::kRowBytes;  // (CTA-pair kernel)
    static constexpr int kOutTiles = 2;             // double-buffered epilogue staging
    static constexpr int kSmemBytes =
        STAGES * (kAStageK + kBStage) + kOutTiles * kOutTile + 1024 /*align*/ + 256 /*barriers*/;
    static_assert((BN / CG) % kNC == 0, "each CTA must hold whole swizzle-atom columns of B");
    static_assert(CG == 1 || (MT == 1 && KSUB == 1), "CTA pairs run one m-tile and one k-subtile per stage");
    static_assert(kTmemCols == 128 || kTmemCols == 256 || kTmemCols == 512, "TMEM columns");
    static_assert(kSmemBytes <= 227 * 1024, "shared memory");
};

// Per-stage work is sized so the fixed costs amortise: the MMA issuer's
// handshake (wait, fence, commit ~250-450 cycles, tools/mma_bench.cu) and the
// SM's TMA unit (~200+ cycles per operation whatever its size,
// tools/tma_bench.cu).  MT m-tiles per CTA share every filter load and fetch
// their pixels with ONE im2col box of MT*128 pixels; KSUB k-subtiles per
// stage multiply the MMAs per handshake.
//
// CG = 2 runs the block on a CTA pair (tcgen05 cta_group::2, launched as a
// 2-CTA cluster): CTA r gathers pixels [m0 + 128 r, +128) and HALF of the
// filter tile; the leader issues 256 x BN MMAs reading both CTAs' smem and
// accumulating 128 rows into each CTA's TMEM.  Both CTAs' TMA loads signal
// the leader's `full` barrier (armed with both CTAs' bytes); the leader's
// commits multicast to both CTAs' `empty` / `tfull`; every epilogue warp
// of both CTAs arrives on the leader's `tempty`.
template <int ELEM, int OUT, int BN, int STAGES, int KSUB, int MT, int CG>
__global__ void __launch_bounds__(kThreadsGeneric, 1)
    conv_fwd_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                    const __grid_constant__ CUtensorMap tmap_y, const ConvParams p) {
    using Cfg = ConvCfg<ELEM, OUT, BN, STAGES, KSUB, MT, CG>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *smem_a = smem;
    uint8_t *smem_b = smem + STAGES * Cfg::kAStageK;
    uint8_t *smem_out = smem_b + STAGES * Cfg::kBStage;  // epilogue staging, 1024-aligned
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_out + Cfg::kOutTiles * Cfg::kOutTile);
    uint64_t *full = bars;
    uint64_t *empty = bars + STAGES;
    uint64_t *tfull = bars + 2 * STAGES;
    uint64_t *tempty = tfull + 2;
    uint64_t *bres = tempty + 2;  // resident filter slice landed (B-stationary mode)
    uint64_t *sk_bar = bres + 1;  // split-K: peers' partial blocks landed in the (idle) operand ring
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sk_bar + 1);
    volatile uint32_t *tl_slot = tmem_slot + 2;  // instrumentation: this launch's timeline index

    // broadcast from lane 0: the role branches are then provably warp-uniform and
    // ptxas keeps the MMA issuer's descriptors on the uniform datapath
    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
    const uint32_t lane = threadIdx.x & 31;
    const long long total_tiles = static_cast<long long>(p.m_tiles) * p.n_tiles;  // m_tiles of CG*kRows pixels
    const uint32_t rank = CG == 2 ? ptx::cluster_ctarank() : 0u;  // 0 = leader (issues the MMAs)
    const long long tile_start = CG == 2 ? (blockIdx.x >> 1) : blockIdx.x;
    const long long tile_step = CG == 2 ? (gridDim.x >> 1) : gridDim.x;
    const int k_subs = p.k_stages;                       // k-subtiles per block (host value)
    const int k_stages = (k_subs + KSUB - 1) / KSUB;     // pipeline stages per block
    // bytes of one A row of one tap inside a subtile (128 for >= 64-channel chunks)
    const int rb = kRowBytes / p.tps;
    // B-stationary: this CTA's output-channel block never changes (grid % n_tiles == 0)
    // and all k-subtiles of a block fit the B ring -> the filter slice is loaded
    // once into ring slots 0..k_stages-1 and only A streams (1x1 layers, C*e <= 4*128 B)
    const bool b_res = CG == 1 && KSUB == 1 && p.b_resident && !p.a_gather && k_stages <= STAGES;
    // split-K tail (mode 1) / stream-K (mode 2) over the tiles [sk_first, total) (UnitWalk)
    const int sk_mode = (!p.a_gather && !b_res) ? p.sk_mode : 0;
    const int S = sk_mode == 1 ? p.sk_split : 1;
    const long long full_end = sk_mode ? p.sk_first : total_tiles;
    const UnitWalk walk(tile_start, tile_step, total_tiles, sk_mode, S, full_end, k_stages);

    if (warp == 0 && lane == 0) {
#if IMCONV_INSTRUMENT
        if (p.dbg && blockIdx.x == 0) {
            const uint32_t idx = static_cast<uint32_t>(atomicAdd(reinterpret_cast<unsigned long long *>(p.dbg + 148 * 20), 1ull));
            *tl_slot = idx;
            tl_stamp(p.dbg, idx, 0);
        }
#endif
        ptx::prefetch_tmap(&tmap_a);
        ptx::prefetch_tmap(&tmap_b);
        ptx::prefetch_tmap(&tmap_y);
        for (int i = 0; i < STAGES; ++i) {
            // one A producer + one B producer arm each stage; in gather mode
            // every lane of the A warp arrives once its copies have landed
            ptx::mbar_init(&full[i], (p.a_gather || p.a_cl) ? 33 : (b_res ? 1 : 2));
            ptx::mbar_init(&empty[i], 1);
        }
        ptx::mbar_init(bres, 1);
        ptx::mbar_init(sk_bar, 1);
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&tfull[i], 1);
            ptx::mbar_init(&tempty[i], 4 * CG);  // one arrival per epilogue warp (of both CTAs)
        }
        ptx::fence_barrier_init();
    }
    if (warp == 2) {
        if constexpr (CG == 2)
            ptx::tmem_alloc_2sm<Cfg::kTmemCols>(tmem_slot);
        else
            ptx::tmem_alloc<Cfg::kTmemCols>(tmem_slot);
    }
    ptx::tc_fence_before();
    if constexpr (CG == 2)
        ptx::cluster_sync();
    else
        __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    IMCONV_CHECK((tmem_base >> 16) == 0 && (tmem_base & 0xffffu) + Cfg::kTmemCols <= 512u,
                 "TMEM allocation outside the 512 columns", tmem_base, Cfg::kTmemCols);
    const uint32_t tl_idx = IMCONV_INSTRUMENT ? *tl_slot : 0u;
    volatile uint32_t *dbg_chunks = tmem_slot + 4;  // debug builds: staged / stored chunk counts
    // PDL: setup above overlaps the previous kernel's tail; no global memory is
    // touched before every prerequisite grid has completed
    if (p.b_early == 3) {  // barrier launch: every preceding grid completes before later launches start
        ptx::griddep_wait();
        ptx::griddep_launch_dependents();
    } else {
        ptx::griddep_launch_dependents();
        // B producers touch nothing but the filter and shared memory: with a static
        // filter they fill their ring stages while the previous grid drains
        if (p.b_early < 2 && !(p.b_early && (warp == 3 || warp == 8))) ptx::griddep_wait();
    }
    if (IMCONV_INSTRUMENT && threadIdx.x == 0) tl_stamp(p.dbg, tl_idx, 1);

    if (CG == 1 && STAGES >= 4 && p.a_gather && (warp == 0 || warp == 2)) {  // (>= 2 ring slots per gather warp)
        // ===== A producers for 16-byte pixels (bf16 C = 8: the ResNet stem) =====
        // A 16-byte TMA element costs as much TMA time as a 128-byte one, so the
        // tap blocks (kRows rows x 16 B, no-swizzle K-major core matrices, 8 taps
        // per stage) are gathered by all 32 lanes with cp.async; out-of-image
        // taps are zero-filled (src-size 0).  Warp 0 / 2 take even / odd stages.
        // Completion: wait_group (lagged) -> proxy fence -> per-lane arrive.
        constexpr int kRowsPerLane = Cfg::kRows / 32;
        const int par = warp == 2 ? 1 : 0;
        const int pq = p.p * p.q;
        const size_t img = static_cast<size_t>(p.h) * p.w;
        const uint32_t a0 = ptx::smem_u32(smem_a);
        // completions are retired one stage late: each warp owns only STAGES/2
        // ring slots, so a longer lag would wait on its own un-arrived stage
        constexpr int kLag = 1;
        int pend[kLag + 1];
        int npend = 0;
        uint32_t it = 0;
        int stage = 0;
        uint32_t phase = 0;
        for (long long tile = tile_start; tile < total_tiles; tile += tile_step) {
            const long long m_tile = tile / p.n_tiles;
            const long long m0 = m_tile * Cfg::kRows;
            // this lane's rows: lane + 32 i
            int hb[kRowsPerLane], wb[kRowsPerLane];
            const uint8_t *base[kRowsPerLane];
#pragma unroll
            for (int i = 0; i < kRowsPerLane; ++i) {
                const long long m = m0 + lane + 32 * i;
                const bool ok = m < p.m;
                const int n = ok ? static_cast<int>(m / pq) : 0;
                const int rem = ok ? static_cast<int>(m - static_cast<long long>(n) * pq) : 0;
                const int op = rem / p.q, oq = rem - (rem / p.q) * p.q;
                hb[i] = ok ? op * p.sh - p.ph : -(1 << 20);  // never in range when past M
                wb[i] = oq * p.sw - p.pw;
                base[i] = p.x + static_cast<size_t>(n) * img * 16;
            }
            for (int kb = 0; kb < k_stages; ++kb) {
                const bool mine = ((it++) & 1u) == static_cast<uint32_t>(par);
                if (mine) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    const uint32_t dst0 = a0 + stage * Cfg::kAStageK;
                    for (int t = 0; t < p.tps; ++t) {
                        const int tap = min(kb * p.tps + t, p.rs - 1);  // past-the-end taps meet zero filter rows
                        const int r = tap / p.s, sx = tap - (tap / p.s) * p.s;
                        const uint32_t dblk = dst0 + t * (Cfg::kRows * 16);
#pragma unroll
                        for (int i = 0; i < kRowsPerLane; ++i) {
                            const int hh = hb[i] + r * p.dh, ww = wb[i] + sx * p.dw;
                            const bool ok = hh >= 0 && hh < p.h && ww >= 0 && ww < p.w;
                            const uint8_t *src = ok ? base[i] + (static_cast<size_t>(hh) * p.w + ww) * 16 : p.x;
                            ptx::cp_async_16(dblk + (lane + 32 * i) * 16, src, ok ? 16u : 0u);
                        }
                    }
                    ptx::cp_async_commit();
                    pend[npend++] = stage;
                    if (npend > kLag) {
                        ptx::cp_async_wait<kLag>();
                        ptx::fence_proxy_async_smem();  // generic-proxy writes -> visible to tcgen05
                        ptx::mbar_arrive(&full[pend[0]]);
                        for (int u = 0; u < kLag; ++u) pend[u] = pend[u + 1];
                        --npend;
                    }
                }
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
        ptx::cp_async_wait<0>();
        ptx::fence_proxy_async_smem();
        for (int u = 0; u < npend; ++u) ptx::mbar_arrive(&full[pend[u]]);
    } else if (CG == 1 && KSUB == 1 && MT == 1 && p.a_cl && (warp == 0 || warp == 2)) {
        // ===== A producers, channel-last baseline =====
        // With the reduction ordered k = (c*R + r)*S + s, one 64-element k-subtile mixes
        // several channels and taps: every 2-byte element of an A row comes from a
        // different (pixel, channel), and TMA boxes need >= 16-byte rows, so the lanes
        // gather element by element (8 per 16-byte chunk) into the SW128 K-major tile.
        // This is the channel-last lowering whose locality -- and cost -- degrades with
        // the convolution stride, against which the channel-first kernel is measured.
        // Warps 0 / 2 take even / odd stages; completion: proxy fence -> per-lane arrive.
        constexpr int kRowsPerLane = Cfg::kRows / 32;
        const int par = warp == 2 ? 1 : 0;
        const int pq = p.p * p.q;
        const int rs = p.rs;
        const long long ksz = static_cast<long long>(rs) * p.c;
        const unsigned short *xs = reinterpret_cast<const unsigned short *>(p.x);
        const uint32_t a0 = ptx::smem_u32(smem_a);
        uint32_t it = 0;
        int stage = 0;
        uint32_t phase = 0;
        for (long long tile = tile_start; tile < total_tiles; tile += tile_step) {
            const long long m_tile = tile / p.n_tiles;
            const long long m0 = m_tile * Cfg::kRows;
            int hb[kRowsPerLane], wb[kRowsPerLane];
            long long nb[kRowsPerLane];
#pragma unroll
            for (int i = 0; i < kRowsPerLane; ++i) {
                const long long m = m0 + lane + 32 * i;
                const bool ok = m < p.m;
                const int n = ok ? static_cast<int>(m / pq) : 0;
                const int rem = ok ? static_cast<int>(m - static_cast<long long>(n) * pq) : 0;
                const int op = rem / p.q, oq = rem - (rem / p.q) * p.q;
                hb[i] = ok ? op * p.sh - p.ph : -(1 << 20);  // never in range when past M
                wb[i] = oq * p.sw - p.pw;
                nb[i] = static_cast<long long>(n) * p.h;
            }
            for (int kb = 0; kb < k_stages; ++kb) {
                const bool mine = ((it++) & 1u) == static_cast<uint32_t>(par);
                if (mine) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    const uint32_t dst0 = a0 + stage * Cfg::kAStageK;
#pragma unroll 1
                    for (int j = 0; j < 8; ++j) {  // 16-byte chunk j of every row = k in [kb*64 + 8j, +8)
                        int ec[8], er[8], es[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            const long long k = static_cast<long long>(kb) * 64 + j * 8 + e;
                            const int c = static_cast<int>(k / rs), tap = static_cast<int>(k - static_cast<long long>(c) * rs);
                            ec[e] = k < ksz ? c : -1;
                            er[e] = (tap / p.s) * p.dh;
                            es[e] = (tap - (tap / p.s) * p.s) * p.dw;
                        }
#pragma unroll
                        for (int i = 0; i < kRowsPerLane; ++i) {
                            uint32_t w4[4];
#pragma unroll
                            for (int e = 0; e < 8; e += 2) {
                                uint32_t v2 = 0;
#pragma unroll
                                for (int h2 = 0; h2 < 2; ++h2) {
                                    const int hh = hb[i] + er[e + h2], ww = wb[i] + es[e + h2];
                                    uint32_t v = 0;
                                    if (ec[e + h2] >= 0 && hh >= 0 && hh < p.h && ww >= 0 && ww < p.w)
                                        v = __ldg(xs + ((nb[i] + hh) * p.w + ww) * p.c + ec[e + h2]);
                                    v2 |= v << (16 * h2);
                                }
                                w4[e / 2] = v2;
                            }
                            const uint32_t row = lane + 32 * i;
                            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(
                                             dst0 + row * 128 + ((static_cast<uint32_t>(j) ^ (row & 7)) << 4)),
                                         "r"(w4[0]), "r"(w4[1]), "r"(w4[2]), "r"(w4[3])
                                         : "memory");
                        }
                    }
                    ptx::fence_proxy_async_smem();  // generic-proxy writes -> visible to tcgen05
                    ptx::mbar_arrive(&full[stage]);
                }
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 0 || warp == 2 || warp == 3 || warp == 8) {
        // ============ TMA producers ============
        // A (activations, im2col): warps 0 / 2 take even / odd stages;
        // B (filter): warps 3 / 8 take even / odd stages.  A TMA costs its
        // issuing thread ~450 cycles whatever the box size (tools/tma_bench.cu),
        // so two issuing threads per operand double the fill rate; each stage's
        // `full` barrier is armed by exactly one A and one B producer.
        if (lane == 0 && b_res && (warp == 3 || warp == 8)) {
            // B-stationary: warp 3 loads the block's whole filter slice once; warp 8 idles
            if (warp == 3) {
                const uint64_t pol = ptx::policy_evict_last();
                const int nb0 = static_cast<int>(tile_start % p.n_tiles) * BN;
                ptx::mbar_arrive_expect_tx(bres, static_cast<uint32_t>(k_stages * Cfg::kBSub));
                KWalk kw;
                kw.reset();
                for (int kb = 0; kb < k_stages; ++kb) {
                    // filter rows of k-subtile kb: one tap's channel chunk, or tps packed taps
                    const int brow = p.tps == 1 ? kw.tap * p.c + kw.chunk * Cfg::kBKE : kb * p.tps * p.c;
                    uint8_t *b_dst = smem_b + kb * Cfg::kBStage;
                    if (p.b_3d) {
                        ptx::tma_load_3d(b_dst, &tmap_b, bres, 0, brow, nb0 / Cfg::kNC, pol);
                    } else {
#pragma unroll
                        for (int j = 0; j < BN / Cfg::kNC; ++j)
                            ptx::tma_load_2d(b_dst + j * (Cfg::kBKE * kRowBytes), &tmap_b, bres, nb0 + j * Cfg::kNC,
                                             brow, pol);
                    }
                    kw.next(p.order, p.r, p.s, p.c_chunks);
                }
            }
        } else if (lane == 0) {
            const bool is_a = warp == 0 || warp == 2;
            const int par = (warp == 2 || warp == 8) ? 1 : 0;
            uint32_t it = 0;
            const uint64_t pol = is_a ? ptx::policy_evict_normal() : ptx::policy_evict_last();
            const int pq = p.p * p.q;
            int stage = 0;
            uint32_t phase = 0;
            long long w_empty = 0;
            const long long t_start = clock64();
            KWalk kw;
            Unit wu;
            for (long long ul = 0; walk.get(ul, wu); ++ul) {
                const long long tile = wu.tile;
                const long long m_tile = tile / p.n_tiles;
                const int n_tile = static_cast<int>(tile - m_tile * p.n_tiles);
                const long long m0 = m_tile * (CG * Cfg::kRows) + rank * Cfg::kRows;
                const int n0 = static_cast<int>(m0 / pq);
                const int rem = static_cast<int>(m0 - static_cast<long long>(n0) * pq);
                const int p0 = rem / p.q;
                const int q0 = rem - p0 * p.q;
                const int w0 = q0 * p.sw - p.pw;  // base pixel (im2col bounding-box coordinates)
                const int h0 = p0 * p.sh - p.ph;
                const int nb0 = n_tile * BN + static_cast<int>(rank) * (BN / CG);
                kw.reset();
                for (int i = 0; i < wu.kb0 * KSUB && p.tps == 1; ++i) kw.next(p.order, p.r, p.s, p.c_chunks);
                for (int kb = wu.kb0; kb < wu.kb1; ++kb) {
                    const bool mine = ((it++) & 1u) == static_cast<uint32_t>(par);
                    const int nsub = min(KSUB, k_subs - kb * KSUB);
                    // completion barrier: own `full` (single CTA) or the leader's (pair)
                    const uint32_t fb = CG == 2 ? ptx::mapa(ptx::smem_u32(&full[stage]), 0)
                                                : ptx::smem_u32(&full[stage]);
                    // instrumentation: skip this operand's loads after the CTA's first tile
                    const bool skip = IMCONV_INSTRUMENT && tile != tile_start &&
                                      (p.dbg_flags & (is_a ? 2 : 1)) != 0;
                    if (mine) {
                        timed_wait_g(&empty[stage], phase ^ 1, w_empty);
                        if (rank == 0)
                            ptx::mbar_arrive_expect_tx(&full[stage],
                                                       skip ? 0u : CG * nsub * (is_a ? Cfg::kASub : Cfg::kBSub));
                    }
                    uint8_t *a_st = smem_a + stage * Cfg::kAStageK;
                    uint8_t *b_st = smem_b + stage * Cfg::kBStage;
                    for (int u = 0; u < nsub; ++u) {
                        int brow;
                        if (p.tps == 1) {
                            const int c0 = kw.chunk * Cfg::kBKE;
                            if (is_a && mine && !skip) {
                                if (p.a_tiled) {
                                    if constexpr (CG == 2)
                                        ptx::tma_load_2d_2sm(a_st + u * Cfg::kASub, &tmap_a, fb, c0,
                                                             static_cast<int>(m0), pol);
                                    else
                                        ptx::tma_load_2d(a_st + u * Cfg::kASub, &tmap_a, &full[stage], c0,
                                                         static_cast<int>(m0), pol);
                                } else if constexpr (CG == 2) {
                                    ptx::tma_load_im2col_4d_2sm(a_st + u * Cfg::kASub, &tmap_a, fb, c0, w0, h0, n0,
                                                                static_cast<uint16_t>(kw.s * p.dw),
                                                                static_cast<uint16_t>(kw.r * p.dh), pol);
                                } else {
                                    ptx::tma_load_im2col_4d(a_st + u * Cfg::kASub, &tmap_a, &full[stage], c0, w0, h0,
                                                            n0, static_cast<uint16_t>(kw.s * p.dw),
                                                            static_cast<uint16_t>(kw.r * p.dh), pol);
                                }
                            }
                            brow = p.a_cl ? (kb * KSUB + u) * Cfg::kBKE : kw.tap * p.c + c0;
                            kw.next(p.order, p.r, p.s, p.c_chunks);
                        } else {
                            // small-C layers: pack tps taps side by side along the
                            // reduction (the paper's multi-tile packing, §4.2); tap t
                            // occupies a (kRows x rb) block
                            const int tap0 = (kb * KSUB + u) * p.tps;
                            if (is_a && mine && !skip) {
                                for (int t = 0; t < p.tps; ++t) {
                                    const int tap = min(tap0 + t, p.rs - 1);  // past-the-end taps meet zero filter rows
                                    const int r = tap / p.s, s = tap - (tap / p.s) * p.s;
                                    if constexpr (CG == 2)
                                        ptx::tma_load_im2col_4d_2sm(a_st + u * Cfg::kASub + t * (Cfg::kRows * rb),
                                                                    &tmap_a, fb, 0, w0, h0, n0,
                                                                    static_cast<uint16_t>(s * p.dw),
                                                                    static_cast<uint16_t>(r * p.dh), pol);
                                    else
                                        ptx::tma_load_im2col_4d(a_st + u * Cfg::kASub + t * (Cfg::kRows * rb), &tmap_a,
                                                                &full[stage], 0, w0, h0, n0,
                                                                static_cast<uint16_t>(s * p.dw),
                                                                static_cast<uint16_t>(r * p.dh), pol);
                                }
                            }
                            brow = tap0 * p.c;
                        }
                        if (!is_a && mine && !skip) {
                            uint8_t *b_dst = b_st + u * Cfg::kBSub;
                            if constexpr (CG == 2) {
                                if (p.b_3d) {
                                    ptx::tma_load_3d_2sm(b_dst, &tmap_b, fb, 0, brow, nb0 / Cfg::kNC, pol);
                                } else {
#pragma unroll
                                    for (int j = 0; j < (BN / CG) / Cfg::kNC; ++j)
                                        ptx::tma_load_2d_2sm(b_dst + j * (Cfg::kBKE * kRowBytes), &tmap_b, fb,
                                                             nb0 + j * Cfg::kNC, brow, pol);
                                }
                            } else if (p.b_3d) {
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
            if (IMCONV_INSTRUMENT && p.dbg && warp == 0) {
                p.dbg[blockIdx.x * 8 + 0] = clock64() - t_start;
                p.dbg[blockIdx.x * 8 + 1] = w_empty;
            }
        }
        __syncwarp();
    } else if (warp == 1 && rank == 0) {
        // ===================== tcgen05 MMA issuer (the leader CTA of a pair) =====================
        const uint32_t idesc = make_idesc<ELEM, BN, CG * kBM>();
        // A layout of one (tap, m-tile) operand: 128 rows x rb bytes; tap blocks
        // of kRows rows; m-tile mt starts mt*128 rows into its tap block
        uint32_t a_lbo, a_sbo, a_layout;
        switch (p.a_layout) {
            case A_SW128: a_lbo = 16; a_sbo = 1024; a_layout = ptx::LAYOUT_SW128; break;
            case A_SW64: a_lbo = 16; a_sbo = 512; a_layout = ptx::LAYOUT_SW64; break;
            case A_SW32: a_lbo = 16; a_sbo = 256; a_layout = ptx::LAYOUT_SW32; break;
            default: a_lbo = Cfg::kRows * 16; a_sbo = 128; a_layout = ptx::LAYOUT_NONE; break;
        }
        // descriptors built once; per MMA only the 14-bit start-address field
        // moves (stage, subtile, m-tile and k-step offsets >> 4)
        uint32_t a_kk[Cfg::kMmaPerSub];
#pragma unroll
        for (int kk = 0; kk < Cfg::kMmaPerSub; ++kk) {
            uint32_t off;
            switch (p.a_layout) {
                case A_SW128: off = kk * 32; break;
                case A_SW64: off = (kk >> 1) * (Cfg::kRows * 64) + (kk & 1) * 32; break;
                case A_SW32: off = kk * (Cfg::kRows * 32); break;
                default: off = kk * 2 * (Cfg::kRows * 16); break;
            }
            a_kk[kk] = off >> 4;
        }
        const uint32_t a_mt = static_cast<uint32_t>((kBM * rb) >> 4);  // m-tile step inside a tap block
        // The whole warp runs the issue loop on warp-uniform values (lane-0
        // broadcasts below) and one elected lane issues each MMA: ptxas then
        // keeps every descriptor in uniform registers (no per-MMA R2UR
        // broadcast / single-lane waterfall loop around each UTCHMMA).
        const uint64_t adesc0 =
            ptx::smem_desc(__shfl_sync(0xffffffffu, ptx::smem_u32(smem_a), 0), a_lbo, a_sbo, a_layout);
        const uint64_t bdesc0 = ptx::smem_desc(__shfl_sync(0xffffffffu, ptx::smem_u32(smem_b), 0),
                                               Cfg::kBKE * kRowBytes, 1024, ptx::LAYOUT_SW128);
        const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem_base, 0);
        const uint32_t a_lo0 = static_cast<uint32_t>(adesc0), a_hi = static_cast<uint32_t>(adesc0 >> 32);
        const uint32_t b_lo0 = static_cast<uint32_t>(bdesc0), b_hi = static_cast<uint32_t>(bdesc0 >> 32);
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        long long w_tempty = 0, w_full = 0;
        if (b_res) ptx::mbar_wait(bres, 0);
        const long long t_start = clock64();
        Unit wu;
        for (long long ul = 0; walk.get(ul, wu); ++ul) {
            IMCONV_CHECK(wu.kb0 < wu.kb1 && wu.kb1 <= k_stages && wu.tile >= 0 && wu.tile < total_tiles,
                         "work unit outside the tile / k-stage space", wu.tile, wu.kb0 * 65536 + wu.kb1);
            timed_wait_g(&tempty[acc], acc_phase ^ 1, w_tempty);
            ptx::tc_fence_after();
            const uint32_t d_base = tmem_u + static_cast<uint32_t>(acc * MT * BN);
            for (int kb = wu.kb0; kb < wu.kb1; ++kb) {
                timed_wait_g(&full[stage], phase, w_full);
                if (IMCONV_INSTRUMENT && ul == 0 && kb == wu.kb0 && lane == 0) tl_stamp(p.dbg, tl_idx, 2);
                ptx::tc_fence_after();
                {
                    // descriptors as (low, high) words: only the start-address field moves
                    const int nsub = min(KSUB, k_subs - kb * KSUB);
                    const uint32_t a_st = a_lo0 + static_cast<uint32_t>((stage * Cfg::kAStageK) >> 4);
                    const uint32_t b_st = b_lo0 + static_cast<uint32_t>(((b_res ? kb : stage) * Cfg::kBStage) >> 4);
#pragma unroll
                    for (int u = 0; u < KSUB; ++u) {
                        if (u < nsub) {
#pragma unroll
                            for (int kk = 0; kk < Cfg::kMmaPerSub; ++kk) {
                                const uint32_t bdesc =
                                    b_st + static_cast<uint32_t>((u * Cfg::kBSub + kk * Cfg::kMmaK * kRowBytes) >> 4);
                                const uint32_t accum = (kb != wu.kb0 || (u | kk) != 0) ? 1u : 0u;
#pragma unroll
                                for (int mt = 0; mt < MT; ++mt) {
                                    const uint32_t adesc =
                                        a_st + static_cast<uint32_t>((u * Cfg::kASub) >> 4) + mt * a_mt + a_kk[kk];
                                    if constexpr (CG == 2) {
                                        if constexpr (ELEM == ELEM_I8)
                                            ptx::mma_i8_2sm_elect_lh(d_base + mt * BN, adesc, a_hi, bdesc, b_hi, idesc, accum);
                                        else
                                            ptx::mma_f16_2sm_elect_lh(d_base + mt * BN, adesc, a_hi, bdesc, b_hi, idesc, accum);
                                    } else if constexpr (ELEM == ELEM_I8) {
                                        ptx::mma_i8_elect_lh(d_base + mt * BN, adesc, a_hi, bdesc, b_hi, idesc, accum);
                                    } else {
                                        ptx::mma_f16_elect_lh(d_base + mt * BN, adesc, a_hi, bdesc, b_hi, idesc, accum);
                                    }
                                }
                            }
                        }
                    }
                    // frees the smem slot (in both CTAs of a pair) once these MMAs retire
                    if constexpr (CG == 2)
                        ptx::mma_commit_2sm_elect(&empty[stage]);
                    else
                        ptx::mma_commit_elect(&empty[stage]);
                }
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            // accumulators complete -> epilogue(s)
            if constexpr (CG == 2)
                ptx::mma_commit_2sm_elect(&tfull[acc]);
            else
                ptx::mma_commit_elect(&tfull[acc]);
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
        if (IMCONV_INSTRUMENT && lane == 0) tl_stamp(p.dbg, tl_idx, 3);
        if (IMCONV_INSTRUMENT && p.dbg && lane == 0) {
            p.dbg[blockIdx.x * 8 + 2] = clock64() - t_start;
            p.dbg[blockIdx.x * 8 + 3] = w_tempty;
            p.dbg[blockIdx.x * 8 + 4] = w_full;
        }
    } else if (warp >= 4 && warp < 8) {
        // ===== epilogue: TMEM -> registers -> one swizzled 128-row tile per 128-byte column chunk =====
        // The four warps stage a whole 128 x 128-byte tile (one TMA store: the
        // SM's TMA unit costs ~200+ cycles per operation whatever its size,
        // tools/tma_bench.cu) and hand it to the store warp, which issues the
        // store -- a TMA issue blocks its thread ~400 cycles, which must not sit
        // on the critical path of the warps draining TMEM.  Handshake per
        // staging tile b (named barriers, 128 epilogue + 32 store threads):
        // FULL(b) = staged, EMPTY(b) = the store that last read b has finished.
        const int quarter = warp & 3;  // TMEM lanes [32*quarter, 32*quarter+32) = block rows
        const uint32_t row = quarter * 32 + lane;
        constexpr int kOC = Cfg::kOutCols;
        int acc = 0;
        uint32_t acc_phase = 0;
        uint32_t chunk_ctr = 0;
        long long w_tfull = 0, t_ld = 0, t_bar = 0, t_st = 0;
        const long long t_start = clock64();
        // hand one staged 128 x 128-byte chunk (fp32 / int32 words v) to the store warp
        auto stage_chunk = [&](const uint32_t *v) {
            const uint32_t b = chunk_ctr & 1;
            if (chunk_ctr >= 2) ptx::named_bar_sync(3 + b, 160);  // EMPTY(b)
            stage_row128<OUT>(smem_out + b * Cfg::kOutTile, row, v);
            ptx::fence_proxy_async_smem();
            ptx::named_bar_arrive(1 + b, 160);  // FULL(b)
            ++chunk_ctr;
        };
        Unit wu;
        for (long long ul = 0; walk.get(ul, wu); ++ul) {
            const long long tile = wu.tile;
            const long long m_tile = tile / p.n_tiles;
            const int n_tile = static_cast<int>(tile - m_tile * p.n_tiles);
            timed_wait_g(&tfull[acc], acc_phase, w_tfull);
            if (IMCONV_INSTRUMENT && ul == 0 && warp == 4 && lane == 0) tl_stamp(p.dbg, tl_idx, 4);
            ptx::tc_fence_after();
            if (wu.split < 0 && wu.sk == 0) {
                // ---- whole tile: TMEM -> staged 128 x 128-byte chunks -> the store warp ----
#pragma unroll 1
                for (int mt = 0; mt < MT; ++mt) {
                    const long long row0 = m_tile * (CG * Cfg::kRows) + rank * Cfg::kRows + mt * kBM;
#pragma unroll 1
                    for (int j = 0; j < BN / kOC; ++j) {
                        const int col0 = n_tile * BN + j * kOC;
                        if (col0 >= p.k || row0 >= p.m) continue;  // uniform (the store warp skips it too)
                        uint32_t v[kOC];
                        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) +
                                               static_cast<uint32_t>(acc * MT * BN + mt * BN + j * kOC);
                        const long long e0 = IMCONV_INSTRUMENT ? clock64() : 0;
#pragma unroll
                        for (int h = 0; h < kOC / 32; ++h)
                            ptx::tmem_ld_32x32b_x32(taddr + h * 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32 * h));
                        ptx::tmem_ld_wait();
                        const long long e1 = IMCONV_INSTRUMENT ? clock64() : 0;
                        stage_chunk(v);
                        if (IMCONV_INSTRUMENT) {
                            t_ld += e1 - e0;
                            t_st += clock64() - e1;
                        }
                    }
                }
                // every TMEM load of this accumulator has completed: release it
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if constexpr (CG == 2)
                        ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&tempty[acc]), 0));
                    else
                        ptx::mbar_arrive(&tempty[acc]);
                }
            } else if (wu.split < 0) {
                // ---- stream-K piece (UnitWalk mode 2; kept out of the whole-tile loop above, whose
                // code generation the output-heavy layers are sensitive to) ----
                // The writer (k-end piece) parks its partial sums in the tile's workspace slot
                // ([block][kOC/4 quads][128 rows][4 words] per CTA of a pair); the finisher (k-start
                // piece, later in its CTA's range) waits for it and adds it to its own accumulator
                // (fixed order: finisher + writer, deterministic).
                constexpr uint32_t kBlkWords = kBM * kOC;
                const long long tt = (tile - full_end) * CG + rank;
                uint32_t *ws_sk = reinterpret_cast<uint32_t *>(p.sk_ws) + tt * (Cfg::kRows * BN);
                unsigned long long *sk_slot = p.sk_cnt + tt;
                if (wu.sk == 2) {
                    if (warp == 4 && lane == 0) {
                        bool last = false;
                        const unsigned long long target = sk_arrive(sk_slot, 2, last);
                        if (!last) {
                            const long long t0 = clock64();
                            uint32_t tries = 0;
                            while (ptx::ld_acquire_gpu(sk_slot) < target) {
                                __nanosleep(32);
                                if ((++tries & 1023u) == 0 && clock64() - t0 > (1ll << 34)) __trap();
                            }
                        }
                        __threadfence();
                    }
                    ptx::named_bar_sync(5, 128);  // the writer's partial is visible to all epilogue warps
                }
#pragma unroll 1
                for (int mt = 0; mt < MT; ++mt) {
                    const long long row0 = m_tile * (CG * Cfg::kRows) + rank * Cfg::kRows + mt * kBM;
#pragma unroll 1
                    for (int j = 0; j < BN / kOC; ++j) {
                        const int col0 = n_tile * BN + j * kOC;
                        if (col0 >= p.k || row0 >= p.m) continue;  // uniform (the store warp skips it too)
                        uint32_t v[kOC];
                        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) +
                                               static_cast<uint32_t>(acc * MT * BN + mt * BN + j * kOC);
#pragma unroll
                        for (int h = 0; h < kOC / 32; ++h)
                            ptx::tmem_ld_32x32b_x32(taddr + h * 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32 * h));
                        ptx::tmem_ld_wait();
                        uint4 *blk = reinterpret_cast<uint4 *>(ws_sk + (mt * (BN / kOC) + j) * kBlkWords) + row;
                        if (wu.sk == 1) {
#pragma unroll
                            for (int q = 0; q < kOC / 4; ++q)
                                blk[q * kBM] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                            continue;
                        }
#pragma unroll
                        for (int q = 0; q < kOC / 4; ++q) {
                            const uint4 u4 = ptx::ld_global_cg_v4(blk + q * kBM);
                            const uint32_t t[4] = {u4.x, u4.y, u4.z, u4.w};
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                if constexpr (OUT == OUT_I32)
                                    v[4 * q + e] += t[e];
                                else
                                    v[4 * q + e] = __float_as_uint(__uint_as_float(v[4 * q + e]) + __uint_as_float(t[e]));
                            }
                        }
                        stage_chunk(v);
                    }
                }
                if (wu.sk == 1) {
                    __threadfence();              // this thread's partials are visible GPU-wide ...
                    ptx::named_bar_sync(5, 128);  // ... for all four epilogue warps: publish
                    if (warp == 4 && lane == 0) {
                        bool last = false;
                        sk_arrive(sk_slot, 2, last);  // the writer never waits
                    }
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if constexpr (CG == 2)
                        ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&tempty[acc]), 0));
                    else
                        ptx::mbar_arrive(&tempty[acc]);
                }
            } else {
                // ---- split-K unit (always its CTA's FIRST unit, see UnitWalk) ----
                // The tile's output blocks (block b = mt * (BN / kOC) + j: m-tile mt, kOC-column
                // chunk j) are owned round-robin by the splits (owner = b % S).  Each split writes
                // the raw 32-bit partial sums of the blocks it does NOT own to the workspace,
                // arrives on the tile's ticket counter and waits for the other splits (they all
                // started at launch); it then adds the peers' partials of its own blocks, in
                // split order (deterministic sums), to its accumulator -- still in TMEM -- and
                // stores them.  Meanwhile the MMA warp already runs the CTA's next unit in the
                // other TMEM accumulator, so the exchange is hidden behind a whole tile.
                // Workspace per (tail tile, CTA of a pair): [split][block][kOC/4 quads][128 rows]
                // [4 words]: one warp-wide store / load of a quad covers 512 contiguous bytes.
                constexpr int kBlocks = MT * (BN / kOC);
                constexpr uint32_t kBlkWords = kBM * kOC;  // 32 KiB (16-bit out) / 16 KiB (32-bit out)
                const long long tt = (tile - full_end) * CG + rank;
                const uint32_t *ws_tile = reinterpret_cast<const uint32_t *>(p.sk_ws) + tt * S * (Cfg::kRows * BN);
                uint32_t *ws_mine = const_cast<uint32_t *>(ws_tile) + static_cast<long long>(wu.split) * (Cfg::kRows * BN);
                const long long rbase = m_tile * (CG * Cfg::kRows) + rank * Cfg::kRows;
                const uint32_t tacc = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) +
                                      static_cast<uint32_t>(acc * MT * BN);
                long long ts[6];
                ts[0] = IMCONV_INSTRUMENT ? clock64() : 0;
#pragma unroll 1
                for (int b = 0; b < kBlocks; ++b) {
                    const int mt = b / (BN / kOC), j = b - mt * (BN / kOC);
                    if (b % S == wu.split) continue;  // owned: stays in TMEM
                    if (n_tile * BN + j * kOC >= p.k || rbase + mt * kBM >= p.m) continue;
                    uint32_t v[kOC];
#pragma unroll
                    for (int h = 0; h < kOC / 32; ++h)
                        ptx::tmem_ld_32x32b_x32(tacc + static_cast<uint32_t>(mt * BN + j * kOC + h * 32),
                                                *reinterpret_cast<uint32_t(*)[32]>(v + 32 * h));
                    ptx::tmem_ld_wait();
                    uint4 *dst = reinterpret_cast<uint4 *>(ws_mine + b * kBlkWords) + row;
#pragma unroll
                    for (int q = 0; q < kOC / 4; ++q) dst[q * kBM] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                }
                ts[1] = IMCONV_INSTRUMENT ? clock64() : 0;
                __threadfence();                      // this thread's partials are visible GPU-wide ...
                ptx::named_bar_sync(5, 128);          // ... for all four epilogue warps
                ts[2] = IMCONV_INSTRUMENT ? clock64() : 0;
                if (warp == 4 && lane == 0) {
                    // arrive, then wait for the tile's other splits (co-resident: every split is
                    // the first unit of a distinct persistent CTA, grid <= resident CTAs)
                    unsigned long long *slot = p.sk_cnt + tt;
                    bool last = false;
                    const unsigned long long target = sk_arrive(slot, S, last);
                    if (!last) {
                        const long long t0 = clock64();
                        uint32_t tries = 0;
                        while (ptx::ld_acquire_gpu(slot) < target) {
                            __nanosleep(32);
                            // a peer that never arrives is a planner bug (non-resident split): fail loudly
                            if ((++tries & 1023u) == 0 && clock64() - t0 > (1ll << 34)) __trap();
                        }
                    }
                    __threadfence();
                }
                ptx::named_bar_sync(6, 160);          // all partials visible -> epilogue warps and the store warp
                ts[3] = IMCONV_INSTRUMENT ? clock64() : 0;
                ts[4] = ts[3];
#pragma unroll 1
                for (int b = wu.split; b < kBlocks; b += S) {
                    const int mt = b / (BN / kOC), j = b - mt * (BN / kOC);
                    if (n_tile * BN + j * kOC >= p.k || rbase + mt * kBM >= p.m) continue;
                    uint32_t v[kOC];
#pragma unroll
                    for (int q = 0; q < kOC; ++q) v[q] = 0u;
                    for (int s2 = 0; s2 < S; ++s2) {  // fixed split order: deterministic sums
                        uint32_t t[kOC];
                        if (s2 == wu.split) {
#pragma unroll
                            for (int h = 0; h < kOC / 32; ++h)
                                ptx::tmem_ld_32x32b_x32(tacc + static_cast<uint32_t>(mt * BN + j * kOC + h * 32),
                                                        *reinterpret_cast<uint32_t(*)[32]>(t + 32 * h));
                            ptx::tmem_ld_wait();
                        } else {
                            const uint4 *src = reinterpret_cast<const uint4 *>(
                                                   ws_tile + static_cast<long long>(s2) * (Cfg::kRows * BN) + b * kBlkWords) + row;
#pragma unroll
                            for (int q = 0; q < kOC / 4; ++q) {
                                const uint4 u4 = ptx::ld_global_cg_v4(src + q * kBM);
                                t[4 * q] = u4.x;
                                t[4 * q + 1] = u4.y;
                                t[4 * q + 2] = u4.z;
                                t[4 * q + 3] = u4.w;
                            }
                        }
#pragma unroll
                        for (int e = 0; e < kOC; ++e) {
                            if constexpr (OUT == OUT_I32)
                                v[e] += t[e];  // int32 two's complement
                            else
                                v[e] = __float_as_uint(__uint_as_float(v[e]) + __uint_as_float(t[e]));
                        }
                    }
                    stage_chunk(v);
                }
                // every TMEM load of this accumulator has completed: release it
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if constexpr (CG == 2)
                        ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&tempty[acc]), 0));
                    else
                        ptx::mbar_arrive(&tempty[acc]);
                }
                if (IMCONV_INSTRUMENT && p.dbg && warp == 4 && lane == 0) {
                    ts[5] = clock64();
                    for (int i = 0; i < 5; ++i) p.dbg[148 * 12 + blockIdx.x * 8 + i] = ts[i + 1] - ts[i];
                    p.dbg[148 * 12 + blockIdx.x * 8 + 5] = ts[0] - t_start;
                    p.dbg[148 * 12 + blockIdx.x * 8 + 6] = wu.split;
                }
            }
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
        // the store warp frees the second-to-last tile after the last chunk: consume
        // that arrival so no named barrier is left half-arrived at exit
        if (chunk_ctr >= 2) ptx::named_bar_sync(3 + (chunk_ctr & 1), 160);
        if (IMCONV_DEBUG && warp == 4 && lane == 0) dbg_chunks[0] = chunk_ctr;
        if (IMCONV_INSTRUMENT && p.dbg && lane == 0 && quarter == 0) {
            p.dbg[blockIdx.x * 8 + 5] = clock64() - t_start;
            p.dbg[blockIdx.x * 8 + 6] = w_tfull;
            p.dbg[blockIdx.x * 8 + 7] = t_ld;
            p.dbg[148 * 8 + blockIdx.x * 4 + 0] = t_bar;
            p.dbg[148 * 8 + blockIdx.x * 4 + 1] = t_st;
        }
    } else if (warp == 9) {
        // ===== output store issuer: one TMA store per staged 128 x 128-byte tile =====
        constexpr int kOC = Cfg::kOutCols;
        uint32_t chunk_ctr = 0;
        Unit wu;
        for (long long ul = 0; walk.get(ul, wu); ++ul) {
            const long long tile = wu.tile;
            const long long m_tile = tile / p.n_tiles;
            const int n_tile = static_cast<int>(tile - m_tile * p.n_tiles);
            // split-K unit: this split stores the blocks it owns (b % S == split);
            // a stream-K writer piece stores nothing (its finisher does)
            if (wu.sk == 1) continue;
            if (wu.split >= 0) ptx::named_bar_sync(6, 160);
            for (int mt = 0; mt < MT; ++mt) {
                const long long row0 = m_tile * (CG * Cfg::kRows) + rank * Cfg::kRows + mt * kBM;
                for (int j = 0; j < BN / kOC; ++j) {
                    const int col0 = n_tile * BN + j * kOC;
                    if (col0 >= p.k || row0 >= p.m) continue;
                    if (wu.split >= 0 && (mt * (BN / kOC) + j) % S != wu.split) continue;
                    const uint32_t b = chunk_ctr & 1;
                    ptx::named_bar_sync(1 + b, 160);  // FULL(b)
                    if (lane == 0) {
                        ptx::tma_store_2d(&tmap_y, smem_out + b * Cfg::kOutTile, col0,
                                          static_cast<int>(row0));  // clipped at M / K
                        ptx::tma_store_commit();
                        ptx::tma_store_wait_read<1>();  // the previous chunk's store has read its tile
                    }
                    __syncwarp();
                    if (chunk_ctr >= 1) ptx::named_bar_arrive(3 + (b ^ 1), 160);  // EMPTY(b ^ 1)
                    ++chunk_ctr;
                }
            }
        }
        // only the staging reads must finish before exit: the grid's completion (what a
        // dependent launch waits on) covers the global writes still in flight
        if (lane == 0) ptx::tma_store_wait_read<0>();
        if (IMCONV_DEBUG && lane == 0) dbg_chunks[1] = chunk_ctr;
        if (IMCONV_INSTRUMENT && lane == 0) tl_stamp(p.dbg, tl_idx, 5);
        __syncwarp();
    }

    if constexpr (CG == 2) {
        ptx::tc_fence_before();
        ptx::cluster_sync();  // neither CTA of the pair releases TMEM / smem while its peer still uses them
        if (warp == 2) {
            ptx::tc_fence_after();
            ptx::tmem_dealloc_2sm<Cfg::kTmemCols>(tmem_base);
        }
    } else {
        __syncthreads();
        if (warp == 2) {
            ptx::tc_fence_after();
            ptx::tmem_dealloc<Cfg::kTmemCols>(tmem_base);
        }
    }
    // every chunk the epilogue staged was stored exactly once (debug builds)
    if (IMCONV_DEBUG && threadIdx.x == 0)
        IMCONV_CHECK(dbg_chunks[0] == dbg_chunks[1], "epilogue staged / store warp stored chunk counts differ",
                     dbg_chunks[0], dbg_chunks[1]);
    if (IMCONV_INSTRUMENT && threadIdx.x == 0) tl_stamp(p.dbg, tl_idx, 6);
}

}  // namespace imconv
