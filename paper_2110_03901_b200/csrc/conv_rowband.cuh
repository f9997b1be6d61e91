// conv_rowband.cuh -- implicit im2col for layers whose pixel vector is exactly
// 16 bytes (bf16/fp16 C = 8, e.g. the ResNet stem with C = 3 padded to 8).
//
// The generic kernel gathers every filter tap separately (one im2col TMA load
// per tap), which for 16-byte pixels degenerates into 16-byte TMA elements and
// re-reads each input pixel R*S times.  Here each input row is loaded ONCE
// per output block as `sw` stride-phase planes (TMA tiled load with element
// stride sw along W: plane e holds columns sw*j + e), and every tap <r,s> of
// the row is formed by the tensor core straight from those planes:
//
//   input column of output q, tap s:  q*sw + s*dw - pw = sw*(q + t_s) + e_s
//
// so tap s's (128 x 16 B) operand is plane e_s starting at pixel q0 + t_s --
// a contiguous run of 16-byte rows, i.e. a no-swizzle K-major UMMA operand
// whose descriptor simply points into the plane.  Two taps fill one
// K = 16 MMA: the second core-matrix column is addressed through the
// descriptor's leading-byte offset (the distance between the two taps' runs).
// Nothing is duplicated in shared memory; the paper's channel-first tap
// decomposition (lowering.py:136-143) becomes descriptor arithmetic.
//
// A block is TP consecutive output rows x 128 output columns of one image;
// the TP accumulators (TP*BN TMEM columns, double-buffered) share the
// (TP-1)*sh + (R-1)*dh + 1 input rows, each loaded once per block.  The
// filter (R x taps x 8 channels x K) stays resident in shared memory for the
// whole persistent kernel, packed in tap-pair order.
#pragma once
#include <cstdint>
#include <cuda.h>

#include "conv_kernel.cuh"
#include "ptx.cuh"

namespace imconv {

constexpr int kMaxPairs = 8;  // S <= 16
constexpr int kProducers = 128;  // warps 0, 2, 3 and 8 gather the planes
constexpr int kMaxEntPerThread = 4;  // sw * needed <= 512 plane pixels per input row

struct RowbandParams {
    int b_early;  // 1: static filter -- warp 0 loads it before griddepcontrol.wait; 2: no role waits
    int n, h, w, k;
    int r, s, sh, sw, ph, pw, dh, dw;
    int p, q;
    int p_groups, q_blocks;
    long long tiles;          // n * p_groups * q_blocks
    int t_min;                // min_s floor((s*dw - pw) / sw)
    int needed;               // plane pixels loaded per input row: min(Q,128) + t_max - t_min
    int plane_bytes;          // smem bytes per plane (covers 128 + t_max - t_min pixels)
    int a_stage_bytes;        // rps * sw * plane_bytes
    int rps;                  // input rows per pipeline stage (2: halves the per-stage handshakes)
    int row_bytes_planes;     // sw * plane_bytes: one input row's planes
    int n_stages;
    int in_rows;              // (TP-1)*sh + (R-1)*dh + 1, rounded up to a multiple of rps
    int npairs;
    int b_bytes;              // resident filter bytes
    int b_chunk_bytes;        // bytes of one 64-column (128 B) n-chunk of the resident filter
    int pair_a_off[kMaxPairs];  // A byte offset of the pair's first tap run inside a stage
    int pair_lbo[kMaxPairs];    // byte distance to the second tap's run (> 0)
    int pair_s0[kMaxPairs];     // tap index (0..S-1) of the first / second half; -1 = zero tap
    int pair_s1[kMaxPairs];
    int row_pair_lbo;         // > 0: output rows j, j+1 share one N = 2*BN MMA (B = two filter rows
                              // sh apart, the second at this byte distance); 0 = off
    const uint8_t *x;         // NHWC input, 16 bytes per pixel
    long long *dbg;           // optional per-CTA wait-cycle counters (instrumentation), else nullptr
    int dbg_flags;            // instrumentation: 1 = epilogue skips TMEM/stores, 2 = producer skips copies,
                              // 4 = one MMA per (row, filter row) instead of npairs, 8 = issuer skips MMAs,
                              // 16 = producer skips the proxy fence, 32 = one full-barrier arrive per warp,
                              // 64 / 128 = epilogue / producer waits back off with nanosleep, 1 << 28 = no output stores
};

// instrumentation: cycles spent in a blocking wait, accumulated per role
__device__ __forceinline__ void timed_wait(uint64_t *bar, uint32_t parity, long long &acc, int sleep_ns = 0) {
#if IMCONV_INSTRUMENT
    const long long t0 = clock64();
    if (sleep_ns) {
        while (!ptx::mbar_try_wait(ptx::smem_u32(bar), parity)) __nanosleep(sleep_ns);
    } else {
        ptx::mbar_wait(bar, parity);
    }
    acc += clock64() - t0;
#else
    (void)acc;
    (void)sleep_ns;
    ptx::mbar_wait(bar, parity);
#endif
}

template <int ELEM, int OUT, int BN, int TP>
struct RowbandCfg {
    static constexpr int kTmemCols = 2 * TP * BN;
    static constexpr int kNChunks = BN / 64;
    static constexpr int kOutCols = (OUT == OUT_BF16 || OUT == OUT_F16) ? 64 : 32;  // one 128-byte chunk
    static constexpr int kOutTile = kBM * 128;                                       // staging tile (x2)
    static_assert(ELEM != ELEM_I8, "row-band path is for 16-bit pixels of 8 channels");
    static_assert(kTmemCols == 128 || kTmemCols == 256 || kTmemCols == 512, "TMEM columns");
};

// STEM = 1: the ResNet-50 stem geometry (7x7, stride 2, dilation 1, 64 channels, 7 input rows per
// stage, 14 per block) as compile-time constants of the MMA issuer (the host checks the layer matches)
constexpr int kStemR = 7, kStemSh = 2, kStemRps = 7, kStemInRows = 14;

template <int ELEM, int OUT, int BN, int TP, int NP, int STEM = 0>
__global__ void __launch_bounds__(kThreadsRowband, 1)
    conv_rowband_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_y,
                        const RowbandParams p) {
    using Cfg = RowbandCfg<ELEM, OUT, BN, TP>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *smem_b = smem;                                   // resident filter
    uint8_t *smem_out = smem + p.b_bytes;                     // epilogue staging (b_bytes is 1024-aligned)
    uint8_t *smem_a = smem_out + 2 * Cfg::kOutTile;           // plane ring
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_a + p.n_stages * p.a_stage_bytes);
    uint64_t *full = bars;
    uint64_t *empty = bars + p.n_stages;
    uint64_t *tfull = bars + 2 * p.n_stages;
    uint64_t *tempty = tfull + 2;
    uint64_t *bfull = tempty + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bfull + 1);
    uint64_t *adesc_tab = reinterpret_cast<uint64_t *>(tmem_slot + 2);          // kMaxPairs entries
    int8_t *rr_tab = reinterpret_cast<int8_t *>(adesc_tab + kMaxPairs);         // in_rows * TP entries (<= 256)

    // broadcast from lane 0: the role branches are then provably warp-uniform and
    // ptxas keeps the MMA issuer's descriptors on the uniform datapath
    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
    const uint32_t lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmap_w);
        ptx::prefetch_tmap(&tmap_y);
        for (int i = 0; i < p.n_stages; ++i) {
            // one arrival per plane-producer thread (instrumentation flag 32: per warp)
            ptx::mbar_init(&full[i], (IMCONV_INSTRUMENT && (p.dbg_flags & 32)) ? kProducers / 32 : kProducers);
            ptx::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&tfull[i], 1);
            ptx::mbar_init(&tempty[i], 4);
        }
        ptx::mbar_init(bfull, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc<Cfg::kTmemCols>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    IMCONV_CHECK((tmem_base >> 16) == 0 && (tmem_base & 0xffffu) + (Cfg::kTmemCols) <= 512u,
                 "TMEM allocation outside the 512 columns", tmem_base, (Cfg::kTmemCols));
    // PDL: setup above overlaps the previous kernel's tail; no global memory is
    // touched before every prerequisite grid has completed
    if (p.b_early == 3) {  // barrier launch: every preceding grid completes before later launches start
        ptx::griddep_wait();
        ptx::griddep_launch_dependents();
    } else {
        ptx::griddep_launch_dependents();
        if (p.b_early < 2 && !(p.b_early && warp == 0)) ptx::griddep_wait();
    }

    if (warp == 0) {
        if (lane == 0) {
            // ---- resident filter: (r, pair, half) groups of 8 channel rows ----
            const uint64_t pol_w = ptx::policy_evict_last();
            ptx::mbar_arrive_expect_tx(bfull, static_cast<uint32_t>(p.b_bytes));
            const int rsc = p.r * p.s * 8;
            for (int r = 0; r < p.r; ++r)
                for (int pr = 0; pr < p.npairs; ++pr)
                    for (int half = 0; half < 2; ++half) {
                        const int s = half ? p.pair_s1[pr] : p.pair_s0[pr];
                        const int row = s >= 0 ? (r * p.s + s) * 8 : rsc;  // rsc: out of range -> zeros
                        // filter rows stored in DESCENDING order, so filter row r - sh (the
                        // next output row's) sits a positive descriptor LBO after row r
                        const int grp = ((p.r - 1 - r) * p.npairs + pr) * 2 + half;
                        for (int j = 0; j < Cfg::kNChunks; ++j)
                            ptx::tma_load_2d(smem_b + j * p.b_chunk_bytes + grp * 1024, &tmap_w, bfull, j * 64, row,
                                             pol_w);
                    }
        }
        __syncwarp();
        if (p.b_early == 1) ptx::griddep_wait();  // the planes read the previous grid's output
    }
    if (warp == 0 || warp == 2 || warp == 3 || warp == 8) {
        // ---- plane producers: cp.async 16-byte pixels into the stride-phase planes ----
        // (LSU path: a 16-byte TMA element costs as much TMA time as a 128-byte
        // one, so strided 16-byte pixels are gathered by threads instead; warp 0
        // joins after issuing the resident-filter load)
        // consecutive lanes copy consecutive input pixels (each 8-lane phase reads one 128-byte
        // line); the planes' pitch is 128 / sw bytes off a multiple of 128 (host), so the phase's
        // sw interleaved plane slots land on disjoint banks: one shared-memory wavefront per phase
        const int t = (warp == 0 ? 0 : warp == 8 ? 3 : warp - 1) * 32 + static_cast<int>(lane);
        const int entries = (IMCONV_INSTRUMENT && (p.dbg_flags & 2)) ? 0 : p.sw * p.needed;
        const uint32_t a0 = ptx::smem_u32(smem_a);
        // this thread's (plane, pixel) entries, fixed for the whole kernel:
        // smem offset inside a stage and column offset relative to the block
        uint32_t e_dst[kMaxEntPerThread];
        int e_col[kMaxEntPerThread];
        int n_ent = 0;
#pragma unroll
        for (int u = 0; u < kMaxEntPerThread; ++u) {
            // entry k = input column col0 + k (consecutive lanes read consecutive
            // pixels: whole 128-byte lines) -> plane k % sw, slot k / sw
            const int k = t + u * kProducers;
            const int j = k / p.sw, e = k - j * p.sw;
            e_dst[u] = static_cast<uint32_t>(e * p.plane_bytes + j * 16);
            e_col[u] = k;
            n_ent += k < entries ? 1 : 0;
        }
        const size_t row_bytes = static_cast<size_t>(p.w) * 16;
        // cp.async groups (stages) kept in flight per thread; must stay below
        // n_stages - 1 or the arrival for a stage would wait on its own slot
        constexpr int kLag = 4;
        const int lag = p.n_stages - 2 < kLag ? p.n_stages - 2 : kLag;
        int npend = 0;      // committed cp.async groups not yet signalled
        int arr_stage = 0;  // oldest of them (stages are committed and signalled in ring order)
        int stage = 0;
        uint32_t phase = 0;
        long long w_empty = 0, t_wg = 0, t_fa = 0;
        const long long t_start = clock64();
        auto signal_oldest = [&]() {
            if (IMCONV_INSTRUMENT && (p.dbg_flags & 32)) {
                __syncwarp();
                if ((t & 31) == 0) ptx::mbar_arrive(&full[arr_stage]);
            } else {
                ptx::mbar_arrive(&full[arr_stage]);
            }
            if (++arr_stage == p.n_stages) arr_stage = 0;
            --npend;
        };
        for (long long tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
            const int qb = static_cast<int>(tile % p.q_blocks);
            const long long rest = tile / p.q_blocks;
            const int pg = static_cast<int>(rest % p.p_groups);
            const int n = static_cast<int>(rest / p.p_groups);
            const int col0 = p.sw * (qb * 128 + p.t_min);
            const int h0 = pg * TP * p.sh - p.ph;
            // per-tile column validity of this thread's entries (rows are checked per row)
            uint32_t col_ok = 0;
            int e_src[kMaxEntPerThread];
#pragma unroll
            for (int u = 0; u < kMaxEntPerThread; ++u) {
                const int col = col0 + e_col[u];
                const bool ok = u < n_ent && col >= 0 && col < p.w;
                col_ok |= ok ? (1u << u) : 0u;
                e_src[u] = (ok ? col : 0) * 16;
            }
            for (int i0 = 0; i0 < p.in_rows; i0 += p.rps) {
                timed_wait(&empty[stage], phase ^ 1, w_empty, (p.dbg_flags & 128) ? 100 : 0);
                for (int ri = 0; ri < p.rps; ++ri) {
                    const int h = h0 + i0 + ri;
                    const bool row_ok = h >= 0 && h < p.h;
                    const uint8_t *xrow = p.x + (static_cast<size_t>(n) * p.h + (row_ok ? h : 0)) * row_bytes;
                    const uint32_t dst0 = a0 + stage * p.a_stage_bytes + ri * p.row_bytes_planes;
                    const uint32_t ok_mask = row_ok ? col_ok : 0u;
#pragma unroll
                    for (int u = 0; u < kMaxEntPerThread; ++u) {
                        if (u < n_ent)
                            ptx::cp_async_16(dst0 + e_dst[u], xrow + e_src[u], ((ok_mask >> u) & 1u) ? 16u : 0u);
                    }
                }
                ptx::cp_async_commit();
                ++npend;
                if (npend > lag) {
#if IMCONV_INSTRUMENT
                    const long long tw0 = clock64();
#endif
                    switch (lag) {  // wait_group takes an immediate
                        case 1: ptx::cp_async_wait<1>(); break;
                        case 2: ptx::cp_async_wait<2>(); break;
                        case 3: ptx::cp_async_wait<3>(); break;
                        default: ptx::cp_async_wait<kLag>(); break;
                    }
#if IMCONV_INSTRUMENT
                    const long long tw1 = clock64();
                    t_wg += tw1 - tw0;
#endif
                    if (!(IMCONV_INSTRUMENT && (p.dbg_flags & 16)))
                        ptx::fence_proxy_async_smem();  // generic-proxy writes -> visible to tcgen05 (async proxy)
                    signal_oldest();
#if IMCONV_INSTRUMENT
                    t_fa += clock64() - tw1;
#endif
                }
                if (++stage == p.n_stages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
        ptx::cp_async_wait<0>();
        ptx::fence_proxy_async_smem();
        while (npend > 0) signal_oldest();
        if (IMCONV_INSTRUMENT && p.dbg && t == 0) {
            p.dbg[blockIdx.x * 8 + 0] = clock64() - t_start;
            p.dbg[blockIdx.x * 8 + 1] = w_empty;
            p.dbg[148 * 8 + blockIdx.x * 4 + 2] = t_fa;
            p.dbg[148 * 8 + blockIdx.x * 4 + 3] = t_wg;
        }
    } else if (warp == 1) {
        // ---- MMA issuer ----
        // Per-MMA work is two 64-bit adds: descriptors are built once (the
        // 14-bit start-address field absorbs stage / filter-row offsets >> 4)
        // and the (output row j, filter row r) pairs of every input row are
        // tabulated, so the single issuing thread keeps up with N = 64 MMAs.
        const uint32_t idesc = make_idesc<ELEM, BN>();
        for (int u = lane; u < p.in_rows * TP; u += 32) {
            const int i = u / TP, j = u - (u / TP) * TP;
            int rr = i - j * p.sh;
            rr = (rr >= 0 && rr % p.dh == 0 && rr / p.dh < p.r) ? rr / p.dh : -1;
            rr_tab[u] = static_cast<int8_t>(rr);
        }
        // Every operand below is provably warp-uniform (kernel parameters,
        // uniform loop counters, and values broadcast from lane 0 with
        // __shfl_sync), so ptxas keeps the descriptors in uniform registers and
        // each MMA is ~2 uniform adds + UTCHMMA -- no per-MMA elect / R2UR
        // broadcast, which otherwise made this single issuing warp (not the
        // tensor pipe) the stem's bottleneck at ~100 cycles per MMA.
        const uint32_t a_base = __shfl_sync(0xffffffffu, ptx::smem_u32(smem_a), 0);
        const uint32_t b_base = __shfl_sync(0xffffffffu, ptx::smem_u32(smem_b), 0);
        const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem_base, 0);
        const int npairs = (IMCONV_INSTRUMENT && (p.dbg_flags & 8)) ? 0 : (IMCONV_INSTRUMENT && (p.dbg_flags & 4)) ? 1 : p.npairs;
        uint64_t adesc_r[NP];
#pragma unroll
        for (int k = 0; k < NP; ++k) {
            const int kk = k < p.npairs ? k : 0;
            adesc_r[k] = ptx::smem_desc(a_base + p.pair_a_off[kk], p.pair_lbo[kk], 128, ptx::LAYOUT_NONE);
        }
        const uint64_t bdesc0 = ptx::smem_desc(b_base, p.b_chunk_bytes, 1024, ptx::LAYOUT_SW128);
        // Row pairing (BN = 64): input row i feeds output row j through filter row rr and
        // row j+1 through rr - sh with the SAME A operand, and the two rows' accumulators
        // are adjacent in TMEM -- so one N = 128 MMA whose B is [W(rr) | W(rr - sh)] (two
        // 64-column atoms LBO apart) does both: 64 instead of 2 x 48 cycles of A+B reads.
        const bool row_pairs = BN == 64 && TP >= 2 && (STEM || p.row_pair_lbo > 0);
        const int g_sh = STEM ? kStemSh : p.sh;  // filter-row step between output rows
        const int g_r = STEM ? kStemR : p.r;
        const uint32_t idesc2 = make_idesc<ELEM, (BN == 64 ? 128 : BN)>();
        const uint64_t bdesc2 = ptx::smem_desc(b_base, static_cast<uint32_t>(p.row_pair_lbo > 0 ? p.row_pair_lbo : 16),
                                               1024, ptx::LAYOUT_SW128);
        // low / high descriptor words (the high words -- SBO, version, layout -- never change)
        uint32_t a_lo[NP];
#pragma unroll
        for (int k = 0; k < NP; ++k) a_lo[k] = static_cast<uint32_t>(adesc_r[k]);
        const uint32_t a_hi = static_cast<uint32_t>(adesc_r[0] >> 32);
        const uint32_t b_lo0 = static_cast<uint32_t>(bdesc0), b_lo2 = static_cast<uint32_t>(bdesc2);
        const uint32_t b_hi = static_cast<uint32_t>(bdesc0 >> 32);
        const uint32_t stage_enc = static_cast<uint32_t>(p.a_stage_bytes >> 4);
        const uint32_t row_enc = static_cast<uint32_t>(p.row_bytes_planes >> 4);
        ptx::mbar_wait(bfull, 0);
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        long long w_tempty = 0, w_full = 0, t_loop = 0, t_commit = 0;
        const long long t_start = clock64();
        for (long long tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
            timed_wait(&tempty[acc], acc_phase ^ 1, w_tempty);
            ptx::tc_fence_after();
            const uint32_t d_base = tmem_u + static_cast<uint32_t>(acc * TP * BN);
            // one input row i (ri-th of its pipeline stage): every (output row, filter row) pair it
            // feeds, as MMAs over the stage's planes
            auto issue_input_row = [&](const int i, const int ri) {
                    const uint64_t a_add = static_cast<uint64_t>(stage * stage_enc + ri * row_enc);
                    int rrs[TP];
                    if (STEM || p.dh == 1) {  // filter row of output row j fed by input row i (no table read)
#pragma unroll
                        for (int j = 0; j < TP; ++j) {
                            const int rr = i - j * g_sh;
                            rrs[j] = (rr >= 0 && rr < g_r) ? rr : -1;
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < TP; ++j) rrs[j] = __shfl_sync(0xffffffffu, rr_tab[i * TP + j], 0);
                    }
                    // descriptors as (low, high) words: per MMA only the low words move
                    const uint32_t a_add32 = static_cast<uint32_t>(a_add);
                    // (the tap-pair loop compiles branch-free when the kernel's NP equals the
                    // layer's pair count -- the stem -- instead of testing every MMA)
                    auto issue_row = [&](auto full_c) {
                        constexpr bool FULL = decltype(full_c)::value;
                        const int np = FULL ? NP : npairs;
                        bool skip = false;
#pragma unroll
                        for (int j = 0; j < TP; ++j) {
                            const int rr = rrs[j];
                            if (skip || rr < 0) {  // warp-uniform
                                skip = false;
                                continue;
                            }
                            const uint32_t b_off = static_cast<uint32_t>((g_r - 1 - rr) * np * 128);
                            if (row_pairs && j + 1 < TP && rrs[j + 1] >= 0) {
                                // rows j and j+1 (filter rows rr and rr - sh >= 0; rr >= sh >= 1)
                                skip = true;
                                const int rr1 = rrs[j + 1];
#pragma unroll
                                for (int pr = 0; pr < NP; ++pr) {
                                    if (!FULL && pr >= np) continue;
                                    if (pr == 0 && rr1 == 0) {
                                        // row j+1's first product initialises its accumulator: issue apart
                                        ptx::mma_f16_elect_lh(d_base + j * BN, a_lo[pr] + a_add32, a_hi, b_lo0 + b_off, b_hi,
                                                              idesc, 1u);
                                        ptx::mma_f16_elect_lh(d_base + (j + 1) * BN, a_lo[pr] + a_add32, a_hi,
                                                              b_lo0 + static_cast<uint32_t>((g_r - 1) * np * 128), b_hi,
                                                              idesc, 0u);
                                    } else {
                                        ptx::mma_f16_elect_lh(d_base + j * BN, a_lo[pr] + a_add32, a_hi,
                                                              b_lo2 + b_off + static_cast<uint32_t>(pr * 128), b_hi, idesc2, 1u);
                                    }
                                }
                                continue;
                            }
#pragma unroll
                            for (int pr = 0; pr < NP; ++pr) {
                                if (FULL || pr < np)
                                    ptx::mma_f16_elect_lh(d_base + j * BN, a_lo[pr] + a_add32, a_hi,
                                                          b_lo0 + b_off + static_cast<uint32_t>(pr * 128), b_hi, idesc,
                                                          (rr | pr) != 0 ? 1u : 0u);
                            }
                        }
                    };
                    if (STEM || npairs == NP)
                        issue_row(std::true_type{});
                    else
                        issue_row(std::false_type{});
            };
            auto issue_stage = [&](auto body) {
                timed_wait(&full[stage], phase, w_full);
                ptx::tc_fence_after();
#if IMCONV_INSTRUMENT
                const long long tm0 = clock64();
#endif
                body();
#if IMCONV_INSTRUMENT
                const long long tm1 = clock64();
                t_loop += tm1 - tm0;
#endif
                ptx::mma_commit_elect(&empty[stage]);
#if IMCONV_INSTRUMENT
                t_commit += clock64() - tm1;
#endif
                if (++stage == p.n_stages) {
                    stage = 0;
                    phase ^= 1;
                }
            };
            if constexpr (STEM) {
                // the ResNet stem geometry is compile-time (2 stages of 7 input rows): every
                // (row, filter row, tap pair) decision folds away and the issue is straight-line
#pragma unroll
                for (int i0 = 0; i0 < kStemInRows; i0 += kStemRps)
                    issue_stage([&] {
#pragma unroll
                        for (int ri = 0; ri < kStemRps; ++ri) issue_input_row(i0 + ri, ri);
                    });
            } else {
                for (int i0 = 0; i0 < p.in_rows; i0 += p.rps)
                    issue_stage([&] {
                        for (int ri = 0; ri < p.rps; ++ri) issue_input_row(i0 + ri, ri);
                    });
            }
            ptx::mma_commit_elect(&tfull[acc]);
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
        if (IMCONV_INSTRUMENT && p.dbg && lane == 0) {
            p.dbg[blockIdx.x * 8 + 2] = clock64() - t_start;
            p.dbg[blockIdx.x * 8 + 3] = w_tempty;
            p.dbg[blockIdx.x * 8 + 4] = w_full;
            p.dbg[148 * 8 + blockIdx.x * 4 + 0] = t_commit;
            p.dbg[148 * 8 + blockIdx.x * 4 + 1] = t_loop;
        }
    } else if (warp >= 4 && warp < 8) {
        // ---- epilogue: per output row j and 128-byte channel chunk, the four warps stage
        // the block's 128 pixels as one SW128 tile and the store warp writes it with ONE
        // 4-D TMA store {chunk, 128 pixels (clipped at Q), 1 row, 1 image}; handshake as in
        // conv_fwd_kernel (named barriers FULL(b) = 1 + b, EMPTY(b) = 3 + b) ----
        const int quarter = warp & 3;
        const uint32_t row = quarter * 32 + lane;
        constexpr int kOC = Cfg::kOutCols;
        int acc = 0;
        uint32_t acc_phase = 0;
        uint32_t chunk_ctr = 0;
        long long w_tfull = 0;
        const long long t_start = clock64();
        for (long long tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
            const long long rest = tile / p.q_blocks;
            const int pg = static_cast<int>(rest % p.p_groups);
            timed_wait(&tfull[acc], acc_phase, w_tfull, (p.dbg_flags & 64) ? 200 : 0);
            ptx::tc_fence_after();
#pragma unroll 1
            for (int j = 0; j < TP; ++j) {
                if (pg * TP + j >= p.p) continue;  // uniform (the store warp skips it too)
#pragma unroll 1
                for (int c = 0; c < BN / kOC; ++c) {
                    if (c * kOC >= p.k) continue;
                    uint32_t v[kOC];
                    const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) +
                                           static_cast<uint32_t>(acc * TP * BN + j * BN + c * kOC);
#pragma unroll
                    for (int h = 0; h < kOC / 32; ++h)
                        ptx::tmem_ld_32x32b_x32(taddr + h * 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32 * h));
                    ptx::tmem_ld_wait();
                    const uint32_t b = chunk_ctr & 1;
                    if (chunk_ctr >= 2) ptx::named_bar_sync(3 + b, 160);  // EMPTY(b)
                    if (!(IMCONV_INSTRUMENT && (p.dbg_flags & 1))) stage_row128<OUT>(smem_out + b * Cfg::kOutTile, row, v);
                    ptx::fence_proxy_async_smem();
                    ptx::named_bar_arrive(1 + b, 160);  // FULL(b)
                    ++chunk_ctr;
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
        if (chunk_ctr >= 2) ptx::named_bar_sync(3 + (chunk_ctr & 1), 160);
        if (IMCONV_INSTRUMENT && p.dbg && lane == 0 && quarter == 0) {
            p.dbg[blockIdx.x * 8 + 5] = clock64() - t_start;
            p.dbg[blockIdx.x * 8 + 6] = w_tfull;
        }
    } else if (warp == 9) {
        // ---- output store issuer ----
        constexpr int kOC = Cfg::kOutCols;
        uint32_t chunk_ctr = 0;
        for (long long tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
            const int qb = static_cast<int>(tile % p.q_blocks);
            const long long rest = tile / p.q_blocks;
            const int pg = static_cast<int>(rest % p.p_groups);
            const int n = static_cast<int>(rest / p.p_groups);
            for (int j = 0; j < TP; ++j) {
                const int prow = pg * TP + j;
                if (prow >= p.p) continue;
                for (int c = 0; c < BN / kOC; ++c) {
                    if (c * kOC >= p.k) continue;
                    const uint32_t b = chunk_ctr & 1;
                    ptx::named_bar_sync(1 + b, 160);  // FULL(b)
                    if (lane == 0) {
                        if (!(IMCONV_INSTRUMENT && (p.dbg_flags & (1 << 28))))  // instrumentation: skip the output stores
                            ptx::tma_store_4d(&tmap_y, smem_out + b * Cfg::kOutTile, c * kOC, qb * 128, prow, n);
                        ptx::tma_store_commit();
                        ptx::tma_store_wait_read<1>();
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
        __syncwarp();
    }

    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<Cfg::kTmemCols>(tmem_base);
    }
}

}  // namespace imconv
