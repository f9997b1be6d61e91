// conv_halo.cuh -- stride-1 convolutions whose pixel is exactly one 128-byte
// swizzle row (bf16/fp16 C = 64, int8 C = 128) and whose whole filter fits in
// shared memory (e.g. the ResNet-50 stage-2 3x3 layers).
//
// The generic kernel gathers every filter tap separately: one im2col TMA box
// of 128 output pixels per tap, so each input pixel crosses the SM's shared
// memory R*S times.  For these N = 64 layers shared-memory bandwidth (operand
// writes + tensor-core reads), not the tensor core, is the bound.  Here a block
// is TPR whole output rows of one image laid out with a padded row pitch
// QP = Q + (S-1)*dw:
//
//   accumulator row m = p_rel * QP + q        (q >= Q: halo columns, discarded)
//
// and ONE 4-D TMA box loads the TR = TPR + (R-1)*dh input rows x QP pixels the
// block needs (out-of-image rows / columns are zero-filled by the hardware:
// the reference's virtual padding, lowering.py:59-64).  Input pixel
// (p_rel + r*dh, q + s*dw) of that tile is smem row m + r*dh*QP + s*dw, so
// filter tap <r,s> is the same tile read through a descriptor whose start
// moves by that many 128-byte rows -- the tensor core applies the SW128
// swizzle by absolute shared-memory address (tools/desc_probe.cu), so shifted
// descriptors need no re-layout.  The paper's channel-first tap decomposition
// (lowering.py:136-143) becomes descriptor arithmetic, and each input pixel
// is written to shared memory once per block instead of once per tap.
//
// HB = 2 (BN = 64): a block is two such sub-blocks stacked (2*TPR output rows, one input tile of
// 2*TPR + (R-1)*dh rows).  Sub-block 1's tap <r',s> reads the tile at the same shift as sub-block
// 0's tap <r'+TPR/dh, s>, and the two accumulators are adjacent in TMEM, so those taps run as ONE
// N = 128 MMA whose B is [W(r'+TPR/dh, s) | W(r', s)] (two 64-column atoms one LBO apart; the
// resident filter is stored filter-row-descending): A is read once for both sub-blocks.
//
// The filter (R*S taps x 128-byte k-rows x BN) stays resident.  Warp roles as
// in conv_fwd_kernel: 0 = TMA producer, 1 = MMA issuer, 2 = TMEM allocator,
// 4-7 = epilogue (TMEM -> swizzled staging of the TPR*Q valid pixels), 9 =
// store issuer (one 4-D TMA store {128 B of channels, Q, TPR, 1} per chunk).
#pragma once
#include <cstdint>
#include <cuda.h>

#include "conv_kernel.cuh"
#include "ptx.cuh"

namespace imconv {

struct HaloParams {
    int b_early;  // 1: static filter -- warp 0 loads it before griddepcontrol.wait; 2: no role waits
    int n, h, w, k;
    int r, s, ph, pw, dh, dw;
    int p, q;
    int qp;                 // padded row pitch of the tile (Q + (S-1)*dw)
    int tpr;                // output rows per sub-block (floor(128 / qp))
    int tr;                 // input rows per block (HB*tpr + (R-1)*dh)
    int p_tiles;            // ceil(P / (HB*tpr))
    long long tiles;        // n * p_tiles * n_tiles
    int n_tiles;            // output-channel blocks of BN
    int a_stage_bytes;      // tr * qp * 128 rounded up to 1024 (+ slack rows the last taps over-read)
    int a_box_bytes;        // tr * qp * 128 (bytes the TMA delivers)
    int n_stages;
    int b_bytes;            // resident filter bytes (R*S taps; CTA pairs: this CTA's two regions)
    int pair_dr;            // CTA pairs: filter-row distance of the taps the two sub-blocks share (0 = none)
    int b_single_off;       // CTA pairs: byte offset of the half-column (SW64) single-tap region
};

template <int ELEM, int OUT, int BN, int HB = 1>
struct HaloCfg {
    static constexpr int kE = ElemTraits<ELEM>::kBytes;
    static constexpr int kBKE = kRowBytes / kE;           // k-rows (channels) per tap
    static constexpr int kNC = kRowBytes / kE;            // columns per 128-byte B chunk
    static constexpr int kBTap = BN * kRowBytes;          // resident B bytes per tap (BN/kNC chunks x kBKE rows x 128 B)
    static constexpr int kBChunk = kBKE * kRowBytes;      // one column chunk of one tap
    static constexpr int kMmaK = 32 / kE;
    static constexpr int kMmaPerTap = kBKE / kMmaK;       // = 4
    static constexpr int kTmemCols = 2 * HB * BN;
    static constexpr int kOutCols = (OUT == OUT_BF16 || OUT == OUT_F16) ? 64 : 32;
    static constexpr int kOutTile = kBM * 128;
    static_assert(kTmemCols == 128 || kTmemCols == 256 || kTmemCols == 512, "TMEM columns");
};

// CG = 2 (BN = 64, HB = 2, 16-bit): a CTA pair runs two blocks with M = 256 MMAs -- each CTA loads
// its own block's input tile -- and the filter columns are split between the pair, so the tensor
// core reads half of every B operand from each CTA:
//   * taps shared by the stacked sub-blocks (N = 128 = [W(r) | W(r - dr)]): CTA 0 holds W(r, s),
//     CTA 1 holds W(r - dr, s), each a full 64-column SW128 atom (slot (r - dr)*S + s);
//   * the other taps (N = 64): each CTA holds 32 of the 64 columns of every W(r, s) as one SW64
//     atom (the b_single_off region, slot r*S + s), loaded through the half-column map tmap_b64.
// Per SM and 128 x 64 x 16 of work the tensor core then reads 5 KB instead of 6 KB (single taps)
// and 6 instead of 8 KB per N = 128 shared tap; both CTAs' loads complete on the leader's
// barriers, its commits multicast to both CTAs, and both CTAs' epilogue warps arrive on its tempty.
template <int ELEM, int OUT, int BN, int HB = 1, int CG = 1>
__global__ void __launch_bounds__(kThreadsGeneric, 1)
    conv_halo_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                     const __grid_constant__ CUtensorMap tmap_y, const __grid_constant__ CUtensorMap tmap_b64,
                     const HaloParams p) {
    static_assert(HB == 1 || BN == 64, "stacked sub-blocks share MMAs through one 64-column atom per tap");
    static_assert(CG == 1 || (HB == 2 && BN == 64 && ELEM != ELEM_I8), "CTA pairs: stacked bf16/fp16 BN = 64 only");
    using Cfg = HaloCfg<ELEM, OUT, BN, HB>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *smem_b = smem;                                 // resident filter (1024-aligned size)
    uint8_t *smem_out = smem_b + p.b_bytes;                 // 2 staging tiles
    uint8_t *smem_a = smem_out + 2 * Cfg::kOutTile;         // input-tile ring
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_a + p.n_stages * p.a_stage_bytes);
    uint64_t *full = bars;
    uint64_t *empty = bars + p.n_stages;
    uint64_t *tfull = bars + 2 * p.n_stages;
    uint64_t *tempty = tfull + 2;
    uint64_t *bfull = tempty + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bfull + 1);

    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t rank = CG == 2 ? ptx::cluster_ctarank() : 0u;  // 0 = leader (issues the MMAs)
    // a pair's (or a single CTA's) block group g covers blocks g*CG + rank; a CTA whose block is
    // past the end (odd block count) recomputes its partner's block and stores nothing
    const long long groups = (p.tiles + CG - 1) / CG;
    const long long g_start = CG == 2 ? (blockIdx.x >> 1) : blockIdx.x;
    const long long g_step = CG == 2 ? (gridDim.x >> 1) : gridDim.x;
    auto block_of = [&](long long g, uint32_t r) {
        const long long t = g * CG + r;
        return t < p.tiles ? t : p.tiles - 1;
    };

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmap_a);
        ptx::prefetch_tmap(&tmap_b);
        ptx::prefetch_tmap(&tmap_y);
        if (CG == 2) ptx::prefetch_tmap(&tmap_b64);
        for (int i = 0; i < p.n_stages; ++i) {
            ptx::mbar_init(&full[i], 1);
            ptx::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&tfull[i], 1);
            ptx::mbar_init(&tempty[i], 4 * CG);
        }
        ptx::mbar_init(bfull, 1);
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
    const int rs = p.r * p.s;

    if (warp == 0) {
        if (lane == 0) {
            // ---- resident filter: per tap, all BN/kNC column chunks in one 3-D box ----
            const uint64_t pol_w = ptx::policy_evict_last();
            if constexpr (CG == 2) {
                // this CTA's share (class comment): shared taps as full atoms, the rest as 32 columns;
                // completion on the leader's bfull, armed for both CTAs
                if (rank == 0) ptx::mbar_arrive_expect_tx(bfull, static_cast<uint32_t>(2 * p.b_bytes));
                const uint32_t bar = ptx::mapa(ptx::smem_u32(bfull), 0);
                const int dr = p.pair_dr;
                for (int r = dr; dr > 0 && r < p.r; ++r)
                    for (int s_ = 0; s_ < p.s; ++s_) {
                        const int src_r = rank == 0 ? r : r - dr;
                        ptx::tma_load_3d_2sm(smem_b + ((r - dr) * p.s + s_) * Cfg::kBTap, &tmap_b, bar, 0,
                                             (src_r * p.s + s_) * Cfg::kBKE, 0, pol_w);
                    }
                for (int t = 0; t < rs; ++t)
                    ptx::tma_load_2d_2sm(smem_b + p.b_single_off + t * (Cfg::kBTap / 2), &tmap_b64, bar,
                                         static_cast<int>(rank) * (BN / 2), t * Cfg::kBKE, pol_w);
            } else {
                ptx::mbar_arrive_expect_tx(bfull, static_cast<uint32_t>(p.b_bytes));
                // (the resident filter covers all K = BN output channels: n_tiles == 1)
                // tap <r,s> goes to slot (R-1-r)*S + s (filter rows descending: a lower filter row sits
                // a positive descriptor LBO after a higher one)
                for (int t = 0; t < rs; ++t) {
                    const int r = t / p.s, s_ = t - r * p.s;
                    ptx::tma_load_3d(smem_b + ((p.r - 1 - r) * p.s + s_) * Cfg::kBTap, &tmap_b, bfull, 0,
                                     t * Cfg::kBKE, 0, pol_w);
                }
            }
            if (p.b_early == 1) ptx::griddep_wait();  // the input tiles depend on the previous grid
            // ---- input tiles: one 4-D box {128 B of channels, QP pixels, TR rows, 1 image} ----
            const uint64_t pol_a = ptx::policy_evict_normal();
            int stage = 0;
            uint32_t phase = 0;
            for (long long g = g_start; g < groups; g += g_step) {
                const long long tile = block_of(g, rank);
                const int pt = static_cast<int>(tile % p.p_tiles);
                const int n = static_cast<int>(tile / p.p_tiles);
                ptx::mbar_wait(&empty[stage], phase ^ 1);
                if (rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], static_cast<uint32_t>(CG * p.a_box_bytes));
                if constexpr (CG == 2)
                    ptx::tma_load_4d_2sm(smem_a + stage * p.a_stage_bytes, &tmap_a,
                                         ptx::mapa(ptx::smem_u32(&full[stage]), 0), 0, -p.pw,
                                         pt * (HB * p.tpr) - p.ph, n, pol_a);
                else
                    ptx::tma_load_4d(smem_a + stage * p.a_stage_bytes, &tmap_a, &full[stage], 0, -p.pw,
                                     pt * (HB * p.tpr) - p.ph, n, pol_a);
                if (++stage == p.n_stages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
        __syncwarp();
    } else if (warp == 1 && CG == 2) {
        // ---- MMA issuer of a CTA pair (the leader): M = 256 over the two CTAs' blocks ----
        if (rank == 0) {
            const uint32_t idesc1 = make_idesc<ELEM, BN, 2 * kBM>();       // single tap, N = 64
            const uint32_t idesc2 = make_idesc<ELEM, 2 * BN, 2 * kBM>();   // shared tap, N = 128
            const uint32_t a_base = __shfl_sync(0xffffffffu, ptx::smem_u32(smem_a), 0);
            const uint32_t b_base = __shfl_sync(0xffffffffu, ptx::smem_u32(smem_b), 0);
            const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem_base, 0);
            const uint64_t adesc0 = ptx::smem_desc(a_base, 16, 1024, ptx::LAYOUT_SW128);
            // shared taps: one 64-column SW128 atom per CTA; single taps: one 32-column SW64 atom per CTA
            const uint64_t bdesc_sh = ptx::smem_desc(b_base, Cfg::kBChunk, 1024, ptx::LAYOUT_SW128);
            const uint64_t bdesc_1 = ptx::smem_desc(b_base + static_cast<uint32_t>(p.b_single_off), Cfg::kBChunk / 2,
                                                    512, ptx::LAYOUT_SW64);
            const uint32_t a_lo0 = static_cast<uint32_t>(adesc0), a_hi = static_cast<uint32_t>(adesc0 >> 32);
            const uint32_t bs_lo = static_cast<uint32_t>(bdesc_sh), bs_hi = static_cast<uint32_t>(bdesc_sh >> 32);
            const uint32_t b1_lo = static_cast<uint32_t>(bdesc_1), b1_hi = static_cast<uint32_t>(bdesc_1 >> 32);
            ptx::mbar_wait(bfull, 0);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            const int dr = p.pair_dr;
            for (long long g = g_start; g < groups; g += g_step) {
                ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem_u + static_cast<uint32_t>(acc * HB * BN);
                ptx::mbar_wait(&full[stage], phase);
                ptx::tc_fence_after();
                const uint32_t a_st = a_lo0 + static_cast<uint32_t>((stage * p.a_stage_bytes) >> 4);
                // one tap: A = the tile shifted by `rows` 128-byte rows; B = this tap's slot (both CTAs)
                auto tap_mmas = [&](uint32_t d_tap, int rows, int r, int s_, bool both, bool first) {
                    const uint32_t a_tap = a_st + static_cast<uint32_t>(rows * 8);
                    const uint32_t b_tap = both ? bs_lo + static_cast<uint32_t>((((r - dr) * p.s + s_) * Cfg::kBTap) >> 4)
                                                : b1_lo + static_cast<uint32_t>(((r * p.s + s_) * (Cfg::kBTap / 2)) >> 4);
#pragma unroll
                    for (int kk = 0; kk < Cfg::kMmaPerTap; ++kk) {
                        const uint32_t accum = (first && kk == 0) ? 0u : 1u;
                        const uint32_t ad = a_tap + static_cast<uint32_t>(kk * 2);  // +32 bytes along K
                        // K advances by kMmaK rows of the MN-major atom: 128-byte (shared) / 64-byte rows
                        const uint32_t bd = b_tap + static_cast<uint32_t>((kk * Cfg::kMmaK * (both ? kRowBytes : kRowBytes / 2)) >> 4);
                        ptx::mma_f16_2sm_elect_lh(d_tap, ad, a_hi, bd, both ? bs_hi : b1_hi, both ? idesc2 : idesc1, accum);
                    }
                };
                // as in the single-CTA issue below: unpartnered sub-block 1 taps, unpartnered
                // sub-block 0 taps (both initialise), then the shared N = 128 taps
                const int r1_lo = dr > 0 ? p.r - dr : 0;
                for (int r = r1_lo; r < p.r; ++r)
                    for (int s_ = 0; s_ < p.s; ++s_)
                        tap_mmas(d + BN, (p.tpr + r * p.dh) * p.qp + s_ * p.dw, r, s_, false, r == r1_lo && s_ == 0);
                const int r0_hi = dr > 0 ? dr : p.r;
                for (int r = 0; r < r0_hi; ++r)
                    for (int s_ = 0; s_ < p.s; ++s_)
                        tap_mmas(d, (r * p.dh) * p.qp + s_ * p.dw, r, s_, false, (r | s_) == 0);
                for (int r = dr; dr > 0 && r < p.r; ++r)
                    for (int s_ = 0; s_ < p.s; ++s_) tap_mmas(d, (r * p.dh) * p.qp + s_ * p.dw, r, s_, true, false);
                ptx::mma_commit_2sm_elect(&empty[stage]);
                ptx::mma_commit_2sm_elect(&tfull[acc]);
                if (++stage == p.n_stages) {
                    stage = 0;
                    phase ^= 1;
                }
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
    } else if (warp == 1) {
        // ---- MMA issuer: R*S taps x kMmaPerTap MMAs per block, all operands warp-uniform ----
        const uint32_t idesc = make_idesc<ELEM, BN>();
        const uint32_t a_base = __shfl_sync(0xffffffffu, ptx::smem_u32(smem_a), 0);
        const uint32_t b_base = __shfl_sync(0xffffffffu, ptx::smem_u32(smem_b), 0);
        const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem_base, 0);
        const uint64_t adesc0 = ptx::smem_desc(a_base, 16, 1024, ptx::LAYOUT_SW128);
        const uint64_t bdesc0 = ptx::smem_desc(b_base, Cfg::kBChunk, 1024, ptx::LAYOUT_SW128);
        const uint32_t a_lo0 = static_cast<uint32_t>(adesc0), a_hi = static_cast<uint32_t>(adesc0 >> 32);
        const uint32_t b_lo0 = static_cast<uint32_t>(bdesc0), b_hi = static_cast<uint32_t>(bdesc0 >> 32);
        // stacked sub-blocks (HB = 2): shared taps pair filter rows dr = TPR/dh apart; their B atoms
        // are dr*S tap slots apart in the row-descending filter (the LBO of the N = 128 descriptor)
        const int share_dr = (HB == 2 && p.tpr % p.dh == 0 && p.tpr / p.dh < p.r) ? p.tpr / p.dh : 0;
        const uint64_t bdesc2 = ptx::smem_desc(b_base, static_cast<uint32_t>((share_dr > 0 ? share_dr : 1) * p.s * Cfg::kBTap),
                                               1024, ptx::LAYOUT_SW128);
        const uint32_t b_lo2 = static_cast<uint32_t>(bdesc2), b_hi2 = static_cast<uint32_t>(bdesc2 >> 32);
        const uint32_t idesc2 = make_idesc<ELEM, 2 * BN <= 256 ? 2 * BN : BN>();
        ptx::mbar_wait(bfull, 0);
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (long long tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
            ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
            ptx::tc_fence_after();
            const uint32_t d = tmem_u + static_cast<uint32_t>(acc * HB * BN);
            ptx::mbar_wait(&full[stage], phase);
            ptx::tc_fence_after();
            // descriptors as (low, high) words: only the start-address field moves
            const uint32_t a_st = a_lo0 + static_cast<uint32_t>((stage * p.a_stage_bytes) >> 4);
            // one tap of one (or both) sub-blocks: A = the tile shifted by `rows` 128-byte rows,
            // B = the resident filter slot of <r,s> (N = 2*BN over both sub-blocks when `both`)
            auto tap_mmas = [&](uint32_t d_tap, int rows, int r, int s, bool both, bool first) {
                const uint32_t a_tap = a_st + static_cast<uint32_t>(rows * 8);
                const uint32_t b_tap = b_lo0 + static_cast<uint32_t>((((p.r - 1 - r) * p.s + s) * Cfg::kBTap) >> 4);
#pragma unroll
                for (int kk = 0; kk < Cfg::kMmaPerTap; ++kk) {
                    const uint32_t accum = (first && kk == 0) ? 0u : 1u;
                    const uint32_t ad = a_tap + static_cast<uint32_t>(kk * 2);  // +32 bytes along K
                    const uint32_t bd = b_tap + static_cast<uint32_t>((kk * Cfg::kMmaK * kRowBytes) >> 4);
                    if constexpr (ELEM == ELEM_I8)
                        ptx::mma_i8_elect_lh(d_tap, ad, a_hi, both ? bd - b_lo0 + b_lo2 : bd, both ? b_hi2 : b_hi,
                                             both ? idesc2 : idesc, accum);
                    else
                        ptx::mma_f16_elect_lh(d_tap, ad, a_hi, both ? bd - b_lo0 + b_lo2 : bd, both ? b_hi2 : b_hi,
                                              both ? idesc2 : idesc, accum);
                }
            };
            if constexpr (HB == 1) {
                for (int r = 0; r < p.r; ++r)
                    for (int s = 0; s < p.s; ++s)
                        tap_mmas(d, (r * p.dh) * p.qp + s * p.dw, r, s, false, (r | s) == 0);
            } else {
                // sub-block 1's tap <r',s> = sub-block 0's tap <r'+dr, s> (same tile shift):
                // 1) sub-block 1 taps without a partner (r' >= R - dr), 2) sub-block 0 taps without a
                // partner (r < dr) -- both initialise their accumulators here -- 3) shared N = 128 taps
                const int dr = share_dr;
                const int r1_lo = dr > 0 ? p.r - dr : 0;
                for (int r = r1_lo; r < p.r; ++r)
                    for (int s = 0; s < p.s; ++s)
                        tap_mmas(d + BN, (p.tpr + r * p.dh) * p.qp + s * p.dw, r, s, false, r == r1_lo && s == 0);
                const int r0_hi = dr > 0 ? dr : p.r;
                for (int r = 0; r < r0_hi; ++r)
                    for (int s = 0; s < p.s; ++s)
                        tap_mmas(d, (r * p.dh) * p.qp + s * p.dw, r, s, false, (r | s) == 0);
                for (int r = dr; dr > 0 && r < p.r; ++r)
                    for (int s = 0; s < p.s; ++s) tap_mmas(d, (r * p.dh) * p.qp + s * p.dw, r, s, true, false);
            }
            ptx::mma_commit_elect(&empty[stage]);
            ptx::mma_commit_elect(&tfull[acc]);
            if (++stage == p.n_stages) {
                stage = 0;
                phase ^= 1;
            }
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
    } else if (warp >= 4 && warp < 8) {
        // ---- epilogue: TMEM row m = p_rel*QP + q -> staging row p_rel*Q + q (halo columns dropped) ----
        const int quarter = warp & 3;
        const int m = quarter * 32 + static_cast<int>(lane);
        const int p_rel = m / p.qp;
        const int qq = m - p_rel * p.qp;
        const bool valid = qq < p.q && p_rel < p.tpr;
        const uint32_t srow = static_cast<uint32_t>(p_rel * p.q + qq);
        constexpr int kOC = Cfg::kOutCols;
        int acc = 0;
        uint32_t acc_phase = 0;
        uint32_t chunk_ctr = 0;
        for (long long g = g_start; g < groups; g += g_step) {
            const bool live = g * CG + rank < p.tiles;
            const int pt = static_cast<int>(block_of(g, rank) % p.p_tiles);
            ptx::mbar_wait(&tfull[acc], acc_phase);
            ptx::tc_fence_after();
#pragma unroll 1
            for (int jj = 0; jj < HB * (BN / kOC); ++jj) {
                const int hb = jj / (BN / kOC), j = jj - hb * (BN / kOC);
                // uniform (the store warp skips the same chunks)
                if (!live || j * kOC >= p.k || (pt * HB + hb) * p.tpr >= p.p) continue;
                uint32_t v[kOC];
                const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) +
                                       static_cast<uint32_t>(acc * HB * BN + hb * BN + j * kOC);
#pragma unroll
                for (int hh = 0; hh < kOC / 32; ++hh)
                    ptx::tmem_ld_32x32b_x32(taddr + hh * 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32 * hh));
                ptx::tmem_ld_wait();
                const uint32_t b = chunk_ctr & 1;
                if (chunk_ctr >= 2) ptx::named_bar_sync(3 + b, 160);  // EMPTY(b)
                if (valid) stage_row128<OUT>(smem_out + b * Cfg::kOutTile, srow, v);
                ptx::fence_proxy_async_smem();
                ptx::named_bar_arrive(1 + b, 160);  // FULL(b)
                ++chunk_ctr;
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (CG == 2)
                    ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&tempty[acc]), 0));
                else
                    ptx::mbar_arrive(&tempty[acc]);
            }
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
        if (chunk_ctr >= 2) ptx::named_bar_sync(3 + (chunk_ctr & 1), 160);
    } else if (warp == 9) {
        // ---- store issuer: one 4-D box {128 B of channels, Q, TPR rows, 1} per staged chunk ----
        constexpr int kOC = Cfg::kOutCols;
        uint32_t chunk_ctr = 0;
        for (long long g = g_start; g < groups; g += g_step) {
            if (g * CG + rank >= p.tiles) continue;
            const long long tile = g * CG + rank;
            const int pt = static_cast<int>(tile % p.p_tiles);
            const int n = static_cast<int>(tile / p.p_tiles);
            for (int jj = 0; jj < HB * (BN / kOC); ++jj) {
                const int hb = jj / (BN / kOC), j = jj - hb * (BN / kOC);
                const int row0 = (pt * HB + hb) * p.tpr;
                if (j * kOC >= p.k || row0 >= p.p) continue;
                const uint32_t b = chunk_ctr & 1;
                ptx::named_bar_sync(1 + b, 160);  // FULL(b)
                if (lane == 0) {
                    ptx::tma_store_4d(&tmap_y, smem_out + b * Cfg::kOutTile, j * kOC, 0, row0, n);  // clipped at P
                    ptx::tma_store_commit();
                    ptx::tma_store_wait_read<1>();
                }
                __syncwarp();
                if (chunk_ctr >= 1) ptx::named_bar_arrive(3 + (b ^ 1), 160);  // EMPTY(b ^ 1)
                ++chunk_ctr;
            }
        }
        // only the staging reads must finish before exit: the grid's completion (what a
        // dependent launch waits on) covers the global writes still in flight
        if (lane == 0) ptx::tma_store_wait_read<0>();
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
}

}  // namespace imconv
