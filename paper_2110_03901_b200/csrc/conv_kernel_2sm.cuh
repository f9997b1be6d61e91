// conv_kernel_2sm.cuh -- the implicit-im2col convolution on CTA pairs
// (tcgen05 cta_group::2).  A thread-block cluster of 2 CTAs on one TPC owns a
// 256-pixel output block: CTA r gathers pixels [m0 + 128 r, m0 + 128 r + 128)
// (its own im2col TMA loads) and HALF of the filter tile (columns
// [n0 + r BN/2, n0 + (r+1) BN/2)); the leader CTA issues one
// 256 x BN x K MMA per k-step that reads A from both CTAs and B from both
// halves, accumulating 128 rows x BN columns into each CTA's TMEM.
//
// Why: the kernel is bound by the L2 -> shared-memory fill rate (TMA), not by
// the tensor cores (tools/run_layer.py --waits: the MMA warp waits on `full`
// ~75% of the time in the 1-CTA kernel).  Splitting B across the pair halves
// the filter bytes every SM pulls per MAC.
//
// Protocol (per stage): both producers TMA into their own smem and signal the
// LEADER's full[stage] (expect_tx armed by the leader with both CTAs' bytes);
// the leader's MMA warp commits to empty[stage] in BOTH CTAs (multicast), so
// each producer refills its own slot; the accumulator handshake is the same
// (tfull multicast to both, tempty = 8 epilogue-warp arrivals on the leader).
#pragma once
#include <cstdint>
#include <cuda.h>

#include "conv_kernel.cuh"
#include "ptx.cuh"

namespace imconv {

template <int ELEM, int OUT, int BN, int STAGES>
struct Conv2smCfg {
    static constexpr int kE = ElemTraits<ELEM>::kBytes;
    static constexpr int kBKE = kRowBytes / kE;
    static constexpr int kNC = kRowBytes / kE;
    static constexpr int kBHalf = BN / 2;                  // filter columns held by each CTA
    static constexpr int kBStage = kBHalf * kRowBytes;     // bytes of B per stage per CTA
    static constexpr int kMmaK = 32 / kE;
    static constexpr int kMmaPerStage = kBKE / kMmaK;
    static constexpr int kTmemCols = 2 * BN;
    static constexpr int kStageOut = 2 * 32 * OutTraits<OUT>::kRowBytes;
    static constexpr int kSmemBytes = STAGES * (kAStage + kBStage) + 4 * kStageOut + 1024 + 256;
    static_assert(kBHalf % kNC == 0, "each CTA must hold whole swizzle-atom columns of B");
    static_assert(kTmemCols == 256 || kTmemCols == 512, "TMEM columns");
};

// M = 256 pair MMA
template <int ELEM, int BN>
__device__ __forceinline__ uint32_t make_idesc_2sm() {
    uint32_t d = 0;
    d |= (ELEM == ELEM_I8 ? 2u : 1u) << 4;
    d |= ElemTraits<ELEM>::kFmt << 7;
    d |= ElemTraits<ELEM>::kFmt << 10;
    d |= 1u << 16;                                   // B MN-major
    d |= static_cast<uint32_t>(BN >> 3) << 17;
    d |= static_cast<uint32_t>(256 >> 4) << 24;
    return d;
}

template <int ELEM, int OUT, int BN, int STAGES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    conv_fwd_2sm_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                        const __grid_constant__ CUtensorMap tmap_y, const ConvParams p) {
    using Cfg = Conv2smCfg<ELEM, OUT, BN, STAGES>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *smem_a = smem;
    uint8_t *smem_b = smem + STAGES * kAStage;
    uint8_t *smem_out = smem_b + STAGES * Cfg::kBStage;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_out + 4 * Cfg::kStageOut);
    uint64_t *full = bars;
    uint64_t *empty = bars + STAGES;
    uint64_t *tfull = bars + 2 * STAGES;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t rank = ptx::cluster_ctarank();  // 0 = leader (issues the pair MMAs)
    const long long pair_tiles = static_cast<long long>((p.m_tiles + 1) / 2) * p.n_tiles;
    const long long cluster_id = blockIdx.x >> 1;
    const long long n_clusters = gridDim.x >> 1;

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmap_a);
        ptx::prefetch_tmap(&tmap_b);
        ptx::prefetch_tmap(&tmap_y);
        for (int i = 0; i < STAGES; ++i) {
            ptx::mbar_init(&full[i], 2);  // leader's A and B producers arm it (with both CTAs' bytes)
            ptx::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&tfull[i], 1);
            ptx::mbar_init(&tempty[i], 8);  // 4 epilogue warps x 2 CTAs (leader's copy is used)
        }
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc_2sm<Cfg::kTmemCols>(tmem_slot);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0 || warp == 3) {
        // ===== TMA producers (both CTAs): warp 0 = own 128 pixels, warp 3 = own half of the filter =====
        if (lane == 0) {
            const bool is_a = warp == 0;
            const uint64_t pol = is_a ? ptx::policy_evict_normal() : ptx::policy_evict_last();
            const int pq = p.p * p.q;
            int stage = 0;
            uint32_t phase = 0;
            KWalk kw;
            for (long long t = cluster_id; t < pair_tiles; t += n_clusters) {
                const long long mp = t / p.n_tiles;
                const int n_tile = static_cast<int>(t - mp * p.n_tiles);
                const long long m0 = mp * 2 * kBM + rank * kBM;
                const int n0 = static_cast<int>(m0 / pq);
                const int rem = static_cast<int>(m0 - static_cast<long long>(n0) * pq);
                const int p0 = rem / p.q;
                const int q0 = rem - p0 * p.q;
                const int w0 = q0 * p.sw - p.pw;
                const int h0 = p0 * p.sh - p.ph;
                const int nb0 = n_tile * BN + static_cast<int>(rank) * Cfg::kBHalf;
                kw.reset();
                for (int kb = 0; kb < p.k_stages; ++kb) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    const uint32_t fb = ptx::mapa(ptx::smem_u32(&full[stage]), 0);
                    if (rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], is_a ? 2 * kAStage : 2 * Cfg::kBStage);
                    int brow;
                    if (p.tps == 1) {
                        const int c0 = kw.chunk * Cfg::kBKE;
                        if (is_a)
                            ptx::tma_load_im2col_4d_2sm(smem_a + stage * kAStage, &tmap_a, fb, c0, w0, h0, n0,
                                                        static_cast<uint16_t>(kw.s * p.dw),
                                                        static_cast<uint16_t>(kw.r * p.dh), pol);
                        brow = kw.tap * p.c + c0;
                        kw.next(p.order, p.r, p.s, p.c_chunks);
                    } else {
                        const int tap0 = kb * p.tps;
                        if (is_a) {
                            const int blk = kAStage / p.tps;
                            for (int tt = 0; tt < p.tps; ++tt) {
                                const int tap = min(tap0 + tt, p.rs - 1);
                                const int r = tap / p.s, s = tap - (tap / p.s) * p.s;
                                ptx::tma_load_im2col_4d_2sm(smem_a + stage * kAStage + tt * blk, &tmap_a, fb, 0, w0, h0,
                                                            n0, static_cast<uint16_t>(s * p.dw),
                                                            static_cast<uint16_t>(r * p.dh), pol);
                            }
                        }
                        brow = tap0 * p.c;
                    }
                    if (!is_a) {
                        uint8_t *b_dst = smem_b + stage * Cfg::kBStage;
                        if (p.b_3d) {
                            ptx::tma_load_3d_2sm(b_dst, &tmap_b, fb, 0, brow, nb0 / Cfg::kNC, pol);
                        } else {
#pragma unroll
                            for (int j = 0; j < Cfg::kBHalf / Cfg::kNC; ++j)
                                ptx::tma_load_2d_2sm(b_dst + j * (Cfg::kBKE * kRowBytes), &tmap_b, fb,
                                                     nb0 + j * Cfg::kNC, brow, pol);
                        }
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ===================== pair MMA issuer (leader CTA) =====================
        if (rank == 0) {
            const uint32_t idesc = make_idesc_2sm<ELEM, BN>();
            uint32_t a_lbo, a_sbo, a_layout;
            switch (p.a_layout) {
                case A_SW128: a_lbo = 16; a_sbo = 1024; a_layout = ptx::LAYOUT_SW128; break;
                case A_SW64: a_lbo = 16; a_sbo = 512; a_layout = ptx::LAYOUT_SW64; break;
                case A_SW32: a_lbo = 16; a_sbo = 256; a_layout = ptx::LAYOUT_SW32; break;
                default: a_lbo = kBM * 16; a_sbo = 128; a_layout = ptx::LAYOUT_NONE; break;
            }
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (long long t = cluster_id; t < pair_tiles; t += n_clusters) {
                ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
                for (int kb = 0; kb < p.k_stages; ++kb) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    if (lane == 0) {
                        const uint32_t a_base = ptx::smem_u32(smem_a + stage * kAStage);
                        const uint32_t b_base = ptx::smem_u32(smem_b + stage * Cfg::kBStage);
#pragma unroll
                        for (int kk = 0; kk < Cfg::kMmaPerStage; ++kk) {
                            uint32_t a_off;
                            switch (p.a_layout) {
                                case A_SW128: a_off = kk * 32; break;
                                case A_SW64: a_off = (kk >> 1) * (kBM * 64) + (kk & 1) * 32; break;
                                case A_SW32: a_off = kk * (kBM * 32); break;
                                default: a_off = kk * 2 * (kBM * 16); break;
                            }
                            const uint64_t adesc = ptx::smem_desc(a_base + a_off, a_lbo, a_sbo, a_layout);
                            const uint64_t bdesc = ptx::smem_desc(b_base + kk * (Cfg::kMmaK * kRowBytes),
                                                                  Cfg::kBKE * kRowBytes, 1024, ptx::LAYOUT_SW128);
                            const uint32_t accum = (kb | kk) != 0 ? 1u : 0u;
                            if constexpr (ELEM == ELEM_I8)
                                ptx::mma_i8_2sm(d_tmem, adesc, bdesc, idesc, accum);
                            else
                                ptx::mma_f16_2sm(d_tmem, adesc, bdesc, idesc, accum);
                        }
                        ptx::mma_commit_2sm(&empty[stage]);  // frees the slot in both CTAs
                    }
                    __syncwarp();
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (lane == 0) ptx::mma_commit_2sm(&tfull[acc]);
                __syncwarp();
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
    } else if (warp >= 4) {
        // ============ epilogue (both CTAs): own 128 rows x BN columns ============
        const int quarter = warp & 3;
        uint8_t *stage_buf = smem_out + quarter * Cfg::kStageOut;
        constexpr int kBuf = 32 * OutTraits<OUT>::kRowBytes;
        const uint32_t tempty_leader0 = ptx::mapa(ptx::smem_u32(&tempty[0]), 0);
        int acc = 0;
        uint32_t acc_phase = 0;
        uint32_t chunk_ctr = 0;
        for (long long t = cluster_id; t < pair_tiles; t += n_clusters) {
            const long long mp = t / p.n_tiles;
            const int n_tile = static_cast<int>(t - mp * p.n_tiles);
            const long long rowl = mp * 2 * kBM + rank * kBM + quarter * 32;
            ptx::mbar_wait(&tfull[acc], acc_phase);
            ptx::tc_fence_after();
#pragma unroll 1
            for (int j = 0; j < BN / 32; ++j) {
                const int col0 = n_tile * BN + j * 32;
                uint32_t v[32];
                const uint32_t taddr =
                    tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(acc * BN + j * 32);
                ptx::tmem_ld_32x32b_x32(taddr, v);
                ptx::tmem_ld_wait();
                if (col0 >= p.k || rowl >= p.m) continue;  // warp-uniform
                uint8_t *buf = stage_buf + (chunk_ctr & 1) * kBuf;
                if (lane == 0) ptx::tma_store_wait_read<1>();
                __syncwarp();
                stage_row_chunk<OUT>(buf, lane, v);
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    ptx::tma_store_2d(&tmap_y, buf, col0, static_cast<int>(rowl));
                    ptx::tma_store_commit();
                }
                ++chunk_ctr;
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_cluster(tempty_leader0 + acc * 8);
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
        if (lane == 0) ptx::tma_store_wait<0>();
        __syncwarp();
    }

    ptx::tc_fence_before();
    ptx::cluster_sync();  // no CTA of the pair may release TMEM / smem while its peer still uses them
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_2sm<Cfg::kTmemCols>(tmem_base);
    }
}

}  // namespace imconv
