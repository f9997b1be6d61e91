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

struct RowbandParams {
    int n, h, w, k;
    int r, s, sh, sw, ph, pw, dh, dw;
    int p, q;
    int p_groups, q_blocks;
    long long tiles;          // n * p_groups * q_blocks
    int t_min;                // min_s floor((s*dw - pw) / sw)
    int box_pix;              // pixels per plane TMA box (box W extent = box_pix * sw <= 256)
    int n_boxes;              // boxes loaded per plane
    int plane_bytes;          // smem bytes per plane (covers 128 + t_max - t_min pixels)
    int a_stage_bytes;        // sw * plane_bytes
    int n_stages;
    int in_rows;              // (TP-1)*sh + (R-1)*dh + 1
    int npairs;
    int b_bytes;              // resident filter bytes
    int b_chunk_bytes;        // bytes of one 64-column (128 B) n-chunk of the resident filter
    int pair_a_off[kMaxPairs];  // A byte offset of the pair's first tap run inside a stage
    int pair_lbo[kMaxPairs];    // byte distance to the second tap's run (> 0)
    int pair_s0[kMaxPairs];     // tap index (0..S-1) of the first / second half; -1 = zero tap
    int pair_s1[kMaxPairs];
};

template <int ELEM, int OUT, int BN, int TP>
struct RowbandCfg {
    static constexpr int kTmemCols = 2 * TP * BN;
    static constexpr int kNChunks = BN / 64;
    static constexpr int kStageOut = 2 * 32 * OutTraits<OUT>::kRowBytes;
    static_assert(ELEM != ELEM_I8, "row-band path is for 16-bit pixels of 8 channels");
    static_assert(kTmemCols == 128 || kTmemCols == 256 || kTmemCols == 512, "TMEM columns");
};

template <int ELEM, int OUT, int BN, int TP>
__global__ void __launch_bounds__(kThreads, 1)
    conv_rowband_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_w,
                        const __grid_constant__ CUtensorMap tmap_y, const RowbandParams p) {
    using Cfg = RowbandCfg<ELEM, OUT, BN, TP>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *smem_b = smem;                                   // resident filter
    uint8_t *smem_out = smem + p.b_bytes;                     // epilogue staging (b_bytes is 1024-aligned)
    uint8_t *smem_a = smem_out + 4 * Cfg::kStageOut;          // plane ring
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_a + p.n_stages * p.a_stage_bytes);
    uint64_t *full = bars;
    uint64_t *empty = bars + p.n_stages;
    uint64_t *tfull = bars + 2 * p.n_stages;
    uint64_t *tempty = tfull + 2;
    uint64_t *bfull = tempty + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bfull + 1);

    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) {
        ptx::prefetch_tmap(&tmap_x);
        ptx::prefetch_tmap(&tmap_w);
        ptx::prefetch_tmap(&tmap_y);
        for (int i = 0; i < p.n_stages; ++i) {
            ptx::mbar_init(&full[i], 1);
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
                        const int grp = (r * p.npairs + pr) * 2 + half;
                        for (int j = 0; j < Cfg::kNChunks; ++j)
                            ptx::tma_load_2d(smem_b + j * p.b_chunk_bytes + grp * 1024, &tmap_w, bfull, j * 64, row,
                                             pol_w);
                    }
            // ---- input planes, one stage per input row of a block ----
            const uint64_t pol_x = ptx::policy_evict_normal();
            const uint32_t stage_tx = static_cast<uint32_t>(p.sw * p.n_boxes * p.box_pix * 16);
            int stage = 0;
            uint32_t phase = 0;
            for (long long tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
                const int qb = static_cast<int>(tile % p.q_blocks);
                const long long rest = tile / p.q_blocks;
                const int pg = static_cast<int>(rest % p.p_groups);
                const int n = static_cast<int>(rest / p.p_groups);
                const int q0 = qb * 128;
                const int h0 = pg * TP * p.sh - p.ph;
                for (int i = 0; i < p.in_rows; ++i) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    ptx::mbar_arrive_expect_tx(&full[stage], stage_tx);
                    uint8_t *dst = smem_a + stage * p.a_stage_bytes;
                    for (int e = 0; e < p.sw; ++e)
                        for (int b = 0; b < p.n_boxes; ++b)
                            ptx::tma_load_4d(dst + e * p.plane_bytes + b * p.box_pix * 16, &tmap_x, &full[stage], 0,
                                             p.sw * (q0 + p.t_min + b * p.box_pix) + e, h0 + i, n, pol_x);
                    if (++stage == p.n_stages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ---- MMA issuer ----
        const uint32_t idesc = make_idesc<ELEM, BN>();
        ptx::mbar_wait(bfull, 0);
        const uint32_t b_base = ptx::smem_u32(smem_b);
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (long long tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
            ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
            ptx::tc_fence_after();
            const uint32_t d_base = tmem_base + static_cast<uint32_t>(acc * TP * BN);
            for (int i = 0; i < p.in_rows; ++i) {
                ptx::mbar_wait(&full[stage], phase);
                ptx::tc_fence_after();
                if (lane == 0) {
                    const uint32_t a_base = ptx::smem_u32(smem_a + stage * p.a_stage_bytes);
#pragma unroll
                    for (int j = 0; j < TP; ++j) {
                        int rr = i - j * p.sh;
                        if (rr < 0 || rr % p.dh != 0) continue;
                        rr /= p.dh;
                        if (rr >= p.r) continue;
                        for (int pr = 0; pr < p.npairs; ++pr) {
                            const uint64_t adesc =
                                ptx::smem_desc(a_base + p.pair_a_off[pr], p.pair_lbo[pr], 128, ptx::LAYOUT_NONE);
                            const uint64_t bdesc = ptx::smem_desc(b_base + ((rr * p.npairs + pr) * 2) * 1024,
                                                                  p.b_chunk_bytes, 1024, ptx::LAYOUT_SW128);
                            ptx::mma_f16(d_base + j * BN, adesc, bdesc, idesc, (rr | pr) != 0 ? 1u : 0u);
                        }
                    }
                    ptx::mma_commit(&empty[stage]);
                }
                __syncwarp();
                if (++stage == p.n_stages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (lane == 0) ptx::mma_commit(&tfull[acc]);
            __syncwarp();
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
    } else if (warp >= 4) {
        // ---- epilogue: TP accumulators -> NHWC via 4-D TMA stores ----
        const int quarter = warp & 3;
        uint8_t *stage_buf = smem_out + quarter * Cfg::kStageOut;
        constexpr int kBuf = 32 * OutTraits<OUT>::kRowBytes;
        int acc = 0;
        uint32_t acc_phase = 0;
        uint32_t chunk_ctr = 0;
        for (long long tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
            const int qb = static_cast<int>(tile % p.q_blocks);
            const long long rest = tile / p.q_blocks;
            const int pg = static_cast<int>(rest % p.p_groups);
            const int n = static_cast<int>(rest / p.p_groups);
            const int qrow = qb * 128 + quarter * 32;
            ptx::mbar_wait(&tfull[acc], acc_phase);
            ptx::tc_fence_after();
#pragma unroll 1
            for (int j = 0; j < TP; ++j) {
                const int prow = pg * TP + j;
#pragma unroll 1
                for (int c = 0; c < BN / 32; ++c) {
                    uint32_t v[32];
                    const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) +
                                           static_cast<uint32_t>(acc * TP * BN + j * BN + c * 32);
                    ptx::tmem_ld_32x32b_x32(taddr, v);
                    ptx::tmem_ld_wait();
                    if (prow >= p.p || qrow >= p.q || c * 32 >= p.k) continue;  // warp-uniform
                    uint8_t *buf = stage_buf + (chunk_ctr & 1) * kBuf;
                    if (lane == 0) ptx::tma_store_wait_read<1>();
                    __syncwarp();
                    stage_row_chunk<OUT>(buf, lane, v);
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        ptx::tma_store_4d(&tmap_y, buf, c * 32, qrow, prow, n);
                        ptx::tma_store_commit();
                    }
                    ++chunk_ctr;
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
        if (lane == 0) ptx::tma_store_wait<0>();
        __syncwarp();
    }

    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<Cfg::kTmemCols>(tmem_base);
    }
}

}  // namespace imconv
