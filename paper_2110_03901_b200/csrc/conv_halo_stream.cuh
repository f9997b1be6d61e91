// conv_halo_stream.cuh -- halo tiles for stride-1 convolutions whose pixel spans SEVERAL
// 128-byte channel chunks (bf16/fp16 C = 128, 192, ...), with the filter streamed.
//
// The generic kernel loads one im2col box per (filter tap, channel chunk): every input pixel
// crosses L2 -> SM R*S times per chunk.  For the stage-3 ResNet 3x3 layers (C = K = 128) that
// operand stream (~12 TB/s L2 -> SM, the practical ceiling) is the bound.  Here, as in
// conv_halo.cuh, a block is HB stacked sub-blocks of TPR whole output rows at padded pitch
// QP = Q + (S-1)*dw; per channel chunk ONE 4-D TMA box brings the block's TR = HB*TPR +
// (R-1)*dh input rows x QP pixels, and filter tap <r,s> is that tile read through a descriptor
// shifted by r*dh*QP + s*dw rows.  The filter does not fit in shared memory, so it streams
// through its own ring: one 64-row x BN-column stage per (chunk, tap), consumed by the HB
// sub-blocks' MMAs.  Per output pixel the SM receives ~half the operand bytes of the generic
// kernel.
//
// Warp roles: 0 = A producer (one TMA per block and chunk), 3 = B producer (one TMA per
// chunk and tap), 1 = MMA issuer, 2 = TMEM allocator, 4-7 = epilogue, 9 = store issuer
// (as in conv_halo.cuh).
#pragma once
#include <cstdint>
#include <cuda.h>

#include "conv_halo.cuh"
#include "conv_kernel.cuh"
#include "ptx.cuh"

namespace imconv {

struct HaloStreamParams {
    int b_early;  // 1: static filter -- the B producer (warp 3) starts before griddepcontrol.wait; 2: no wait
    int n, h, w, c, k;
    int r, s, ph, pw, dh, dw;
    int p, q;
    int qp;                 // padded row pitch (Q + (S-1)*dw)
    int tpr;                // output rows per sub-block (floor(128 / qp))
    int tr;                 // input rows per block (HB*tpr + (R-1)*dh)
    int p_tiles;            // ceil(P / (HB*tpr))
    long long tiles;        // n * p_tiles
    int chunks;             // 128-byte channel chunks per pixel
    int a_slot_bytes;       // one chunk's tile incl. rows the last taps over-read, 1024-aligned
    int a_box_bytes;        // tr * qp * 128 (bytes the TMA delivers)
    int na, nb;             // A slots / B stages
};

template <int ELEM, int OUT, int BN, int HB, int CG = 1>
struct HaloStreamCfg {
    static constexpr int kE = ElemTraits<ELEM>::kBytes;
    static constexpr int kBKE = kRowBytes / kE;       // k-rows per chunk
    static constexpr int kNC = kRowBytes / kE;        // columns per 128-byte B atom
    static constexpr int kBStage = (BN / CG) * kRowBytes;  // one (chunk, tap) filter slice (this CTA's columns)
    static constexpr int kMmaK = 32 / kE;
    static constexpr int kMmaPerTap = kBKE / kMmaK;   // = 4
    static constexpr int kTmemCols = 2 * HB * BN;
    static constexpr int kOutCols = (OUT == OUT_BF16 || OUT == OUT_F16) ? 64 : 32;
    static constexpr int kOutTile = kBM * 128;
    static_assert(kTmemCols == 128 || kTmemCols == 256 || kTmemCols == 512, "TMEM columns");
    static_assert((BN / CG) % kNC == 0, "each CTA of a pair holds whole 128-byte filter column atoms");
};

// CG = 2: a CTA pair (cta_group::2, 2-CTA cluster) runs TWO blocks -- each CTA loads its own
// block's input tile -- with M = 256 MMAs issued by the leader: the filter slice of each
// (chunk, tap) is split by columns, each CTA loading and holding half, so per SM the tensor
// core reads 4 KB of pixels + 2 KB of filter per 256 x BN x 16 MMA instead of 4 + 4 KB, and
// the filter crosses L2 -> SM once per pair.  Both CTAs' TMA loads complete on the leader's
// barriers (armed for both), the leader's commits multicast to both CTAs' empty / tfull
// barriers, and every epilogue warp of both CTAs arrives on the leader's tempty.
template <int ELEM, int OUT, int BN, int HB, int CG = 1>
__global__ void __launch_bounds__(kThreadsGeneric, 1)
    conv_halo_stream_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                            const __grid_constant__ CUtensorMap tmap_y, const HaloStreamParams p) {
    using Cfg = HaloStreamCfg<ELEM, OUT, BN, HB, CG>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *smem_out = smem;                                  // 2 staging tiles
    uint8_t *smem_b = smem_out + 2 * Cfg::kOutTile;            // filter ring
    uint8_t *smem_a = smem_b + p.nb * Cfg::kBStage;            // input-tile ring
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_a + p.na * p.a_slot_bytes);
    uint64_t *a_full = bars;
    uint64_t *a_empty = a_full + p.na;
    uint64_t *b_full = a_empty + p.na;
    uint64_t *b_empty = b_full + p.nb;
    uint64_t *tfull = b_empty + p.nb;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
    const uint32_t lane = threadIdx.x & 31;
    const int rs = p.r * p.s;
    const uint32_t rank = CG == 2 ? ptx::cluster_ctarank() : 0u;  // 0 = leader (issues the MMAs)
    // a pair's (or a single CTA's) block group g covers blocks g*CG + rank
    const long long groups = (p.tiles + CG - 1) / CG;
    const long long g_start = CG == 2 ? (blockIdx.x >> 1) : blockIdx.x;
    const long long g_step = CG == 2 ? (gridDim.x >> 1) : gridDim.x;
    // a CTA whose block is past the end (odd block count) computes its partner's last block
    // again and stores nothing
    auto block_of = [&](long long g, uint32_t r) {
        const long long t = g * CG + r;
        return t < p.tiles ? t : p.tiles - 1;
    };

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmap_a);
        ptx::prefetch_tmap(&tmap_b);
        ptx::prefetch_tmap(&tmap_y);
        for (int i = 0; i < p.na; ++i) {
            ptx::mbar_init(&a_full[i], 1);
            ptx::mbar_init(&a_empty[i], 1);
        }
        for (int i = 0; i < p.nb; ++i) {
            ptx::mbar_init(&b_full[i], 1);
            ptx::mbar_init(&b_empty[i], 1);
        }
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
    IMCONV_CHECK((tmem_base >> 16) == 0 && (tmem_base & 0xffffu) + (Cfg::kTmemCols) <= 512u,
                 "TMEM allocation outside the 512 columns", tmem_base, (Cfg::kTmemCols));
    // PDL: setup above overlaps the previous kernel's tail
    if (p.b_early == 3) {  // barrier launch: every preceding grid completes before later launches start
        ptx::griddep_wait();
        ptx::griddep_launch_dependents();
    } else {
        ptx::griddep_launch_dependents();
        if (p.b_early < 2 && !(p.b_early && warp == 3)) ptx::griddep_wait();
    }

    if (warp == 0) {
        if (lane == 0) {
            // ---- A: per block and channel chunk, one 4-D box {128 B, QP pixels, TR rows, 1 image} ----
            const uint64_t pol = ptx::policy_evict_normal();
            int slot = 0;
            uint32_t phase = 0;
            for (long long g = g_start; g < groups; g += g_step) {
                const long long tile = block_of(g, rank);
                const int pt = static_cast<int>(tile % p.p_tiles);
                const int n = static_cast<int>(tile / p.p_tiles);
                for (int c = 0; c < p.chunks; ++c) {
                    ptx::mbar_wait(&a_empty[slot], phase ^ 1);
                    if (rank == 0)
                        ptx::mbar_arrive_expect_tx(&a_full[slot], static_cast<uint32_t>(CG * p.a_box_bytes));
                    if constexpr (CG == 2)
                        ptx::tma_load_4d_2sm(smem_a + slot * p.a_slot_bytes, &tmap_a,
                                             ptx::mapa(ptx::smem_u32(&a_full[slot]), 0), c * Cfg::kNC, -p.pw,
                                             pt * (HB * p.tpr) - p.ph, n, pol);
                    else
                        ptx::tma_load_4d(smem_a + slot * p.a_slot_bytes, &tmap_a, &a_full[slot], c * Cfg::kNC, -p.pw,
                                         pt * (HB * p.tpr) - p.ph, n, pol);
                    if (++slot == p.na) {
                        slot = 0;
                        phase ^= 1;
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 3) {
        if (lane == 0) {
            // ---- B: per (chunk, tap), the filter's 64 k-rows x this CTA's BN / CG columns in one 3-D box ----
            const uint64_t pol = ptx::policy_evict_last();
            int stage = 0;
            uint32_t phase = 0;
            for (long long g = g_start; g < groups; g += g_step) {
                for (int c = 0; c < p.chunks; ++c) {
                    for (int t = 0; t < rs; ++t) {
                        ptx::mbar_wait(&b_empty[stage], phase ^ 1);
                        if (rank == 0)
                            ptx::mbar_arrive_expect_tx(&b_full[stage], static_cast<uint32_t>(CG * Cfg::kBStage));
                        // filter row of (tap t, chunk c): HWCN rows are (r*S + s)*C + channel
                        if constexpr (CG == 2)
                            ptx::tma_load_3d_2sm(smem_b + stage * Cfg::kBStage, &tmap_b,
                                                 ptx::mapa(ptx::smem_u32(&b_full[stage]), 0), 0,
                                                 t * p.c + c * Cfg::kBKE, static_cast<int>(rank) * (BN / CG / Cfg::kNC),
                                                 pol);
                        else
                            ptx::tma_load_3d(smem_b + stage * Cfg::kBStage, &tmap_b, &b_full[stage], 0,
                                             t * p.c + c * Cfg::kBKE, 0, pol);
                        if (++stage == p.nb) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1 && rank == 0) {
        // ---- MMA issuer (the leader of a pair): per (chunk, tap) one B stage, HB sub-blocks x 4 MMAs ----
        const uint32_t idesc = make_idesc<ELEM, BN, CG * kBM>();
        const uint32_t a_base = __shfl_sync(0xffffffffu, ptx::smem_u32(smem_a), 0);
        const uint32_t b_base = __shfl_sync(0xffffffffu, ptx::smem_u32(smem_b), 0);
        const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem_base, 0);
        const uint64_t adesc0 = ptx::smem_desc(a_base, 16, 1024, ptx::LAYOUT_SW128);
        const uint64_t bdesc0 = ptx::smem_desc(b_base, Cfg::kBKE * kRowBytes, 1024, ptx::LAYOUT_SW128);
        const uint32_t a_lo0 = static_cast<uint32_t>(adesc0), a_hi = static_cast<uint32_t>(adesc0 >> 32);
        const uint32_t b_lo0 = static_cast<uint32_t>(bdesc0), b_hi = static_cast<uint32_t>(bdesc0 >> 32);
        int aslot = 0, bstage = 0;
        uint32_t aphase = 0, bphase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (long long g = g_start; g < groups; g += g_step) {
            // sub-blocks past the last output row (the last block of an image) need no MMAs -- unless
            // the partner's block still has them: the epilogue and the store warp skip them too
            int hb_live = 0;
#pragma unroll
            for (int r2 = 0; r2 < CG; ++r2) {
                const int pt = static_cast<int>(block_of(g, r2) % p.p_tiles);
                hb_live = max(hb_live, min(HB, (p.p - pt * HB * p.tpr + p.tpr - 1) / p.tpr));
            }
            ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
            ptx::tc_fence_after();
            const uint32_t d = tmem_u + static_cast<uint32_t>(acc * HB * BN);
            for (int c = 0; c < p.chunks; ++c) {
                ptx::mbar_wait(&a_full[aslot], aphase);
                ptx::tc_fence_after();
                const uint32_t a_st = a_lo0 + static_cast<uint32_t>((aslot * p.a_slot_bytes) >> 4);
                for (int r = 0; r < p.r; ++r) {
                    for (int s = 0; s < p.s; ++s) {
                        ptx::mbar_wait(&b_full[bstage], bphase);
                        ptx::tc_fence_after();
                        const uint32_t b_st = b_lo0 + static_cast<uint32_t>((bstage * Cfg::kBStage) >> 4);
                        const bool first = c == 0 && r == 0 && s == 0;
#pragma unroll
                        for (int hb = 0; hb < HB; ++hb) {
                            if (hb >= hb_live) continue;  // warp-uniform
                            // sub-block hb, tap <r,s>: the chunk's tile shifted by (hb*TPR + r*dh) rows of QP
                            const uint32_t a_tap =
                                a_st + static_cast<uint32_t>(((hb * p.tpr + r * p.dh) * p.qp + s * p.dw) * 8);
#pragma unroll
                            for (int kk = 0; kk < Cfg::kMmaPerTap; ++kk) {
                                const uint32_t ad = a_tap + static_cast<uint32_t>(kk * 2);  // +32 bytes along K
                                const uint32_t bd = b_st + static_cast<uint32_t>((kk * Cfg::kMmaK * kRowBytes) >> 4);
                                const uint32_t accum = (first && kk == 0) ? 0u : 1u;
                                if constexpr (CG == 2)
                                    ptx::mma_f16_2sm_elect_lh(d + hb * BN, ad, a_hi, bd, b_hi, idesc, accum);
                                else
                                    ptx::mma_f16_elect_lh(d + hb * BN, ad, a_hi, bd, b_hi, idesc, accum);
                            }
                        }
                        if constexpr (CG == 2)
                            ptx::mma_commit_2sm_elect(&b_empty[bstage]);
                        else
                            ptx::mma_commit_elect(&b_empty[bstage]);
                        if (++bstage == p.nb) {
                            bstage = 0;
                            bphase ^= 1;
                        }
                    }
                }
                if constexpr (CG == 2)
                    ptx::mma_commit_2sm_elect(&a_empty[aslot]);
                else
                    ptx::mma_commit_elect(&a_empty[aslot]);
                if (++aslot == p.na) {
                    aslot = 0;
                    aphase ^= 1;
                }
            }
            if constexpr (CG == 2)
                ptx::mma_commit_2sm_elect(&tfull[acc]);
            else
                ptx::mma_commit_elect(&tfull[acc]);
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
                // uniform (the store warp skips it too)
                if (!live || j * kOC >= p.k || (pt * HB + hb) * p.tpr >= p.p) continue;
                uint32_t v[kOC];
                const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) +
                                       static_cast<uint32_t>(acc * HB * BN + hb * BN + j * kOC);
#pragma unroll
                for (int h2 = 0; h2 < kOC / 32; ++h2)
                    ptx::tmem_ld_32x32b_x32(taddr + h2 * 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32 * h2));
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
