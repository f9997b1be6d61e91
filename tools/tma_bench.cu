// tma_bench.cu -- per-SM TMA load throughput from L2-resident data, by box
// shape / mode (tiled vs im2col).  One producer thread per CTA (148 CTAs)
// streams loads into an 8-slot ring; one consumer thread frees slots as soon
// as they land.  Prints bytes per SM-cycle.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2110_03901_b200/csrc tools/tma_bench.cu -o tools/tma_bench
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include "ptx.cuh"

using namespace imconv;

constexpr int kSlots = 8;

// mode 0: 2-D tiled, mode 1: 4-D im2col, mode 2: 4-D tiled (pixel row)
__global__ void __launch_bounds__(128, 1) tma_stream(const __grid_constant__ CUtensorMap m, int mode, int loads,
                                                    int box_bytes, int c_extent, int w_extent, int h_extent,
                                                    long long *out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full_all[2][kSlots], empty_all[2][kSlots];
    if (threadIdx.x == 0) {
        for (int i = 0; i < kSlots; ++i)
            for (int j = 0; j < 2; ++j) {
                ptx::mbar_init(&full_all[j][i], 1);
                ptx::mbar_init(&empty_all[j][i], 1);
            }
        ptx::fence_barrier_init();
    }
    __syncthreads();
    const uint64_t pol = ptx::policy_evict_normal();
    const int nprod = loads < 0 ? 2 : 1;
    if (loads < 0) loads = -loads;
    const int per = loads / nprod;
    const int grp = threadIdx.x >> 6;          // producer/consumer group (0 or 1)
    const int slots = kSlots / nprod;
    uint64_t *full = full_all[grp], *empty = empty_all[grp];
    smem += grp * slots * box_bytes;
    if ((threadIdx.x & 63) == 0 && grp < nprod) {
        for (int i = 0; i < per; ++i) {
            const int s = i % slots;
            ptx::mbar_wait(&empty[s], ((i / slots) & 1) ^ 1);
            ptx::mbar_arrive_expect_tx(&full[s], box_bytes);
            const int k = (blockIdx.x * 7919 + i * 131) & 1023;
            uint8_t *dst = smem + s * box_bytes;
            if (mode == 0) {
                ptx::tma_load_2d(dst, &m, &full[s], 0, (k * 64) % (c_extent - 128), pol);
            } else if (mode == 1) {
                ptx::tma_load_im2col_4d(dst, &m, &full[s], 0, (k % w_extent) - 1, (k / w_extent) % h_extent - 1,
                                        k % 8, static_cast<uint16_t>(i % 3), static_cast<uint16_t>((i / 3) % 3), pol);
            } else {
                ptx::tma_load_4d(dst, &m, &full[s], 0, 0, k % h_extent, k % 8, pol);
            }
        }
    } else if ((threadIdx.x & 63) == 32 && grp < nprod) {
        const long long t0 = clock64();
        for (int i = 0; i < per; ++i) {
            const int s = i % slots;
            ptx::mbar_wait(&full[s], (i / slots) & 1);
            ptx::mbar_arrive(&empty[s]);
        }
        const long long t1 = clock64();
        if (blockIdx.x == 0 && grp == 0) out[0] = t1 - t0;
    }
}

int main() {
    PFN_cuTensorMapEncodeTiled_v12000 enc_tiled;
    PFN_cuTensorMapEncodeIm2col_v12000 enc_im2col;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc_tiled, cudaEnableDefault, &q);
    cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", (void **)&enc_im2col, cudaEnableDefault, &q);
    // 8 x 56 x 58 x 64 bf16 NHWC (~3.3 MB, L2 resident)
    const int N = 8, H = 56, W = 56, C = 64;
    void *x;
    cudaMalloc(&x, size_t(N) * H * W * C * 2 + (1 << 20));
    cudaMemset(x, 0, size_t(N) * H * W * C * 2 + (1 << 20));
    long long *d;
    cudaMalloc(&d, 8);
    const int loads = 20000;
    auto run = [&](const char *name, const CUtensorMap &m, int mode, int box_bytes) {
        cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, kSlots * box_bytes + 1024);
        for (int np = 1; np <= 2; ++np) {
        const int ld = np == 1 ? loads : -loads;
        tma_stream<<<148, 128, kSlots * box_bytes + 1024>>>(m, mode, ld, box_bytes, N * H * W, W, H, d);
        tma_stream<<<148, 128, kSlots * box_bytes + 1024>>>(m, mode, ld, box_bytes, N * H * W, W, H, d);
        cudaError_t e = cudaDeviceSynchronize();
        long long c = 0;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        printf("%-40s box %6d B, %d producer(s): %6.1f cyc/load  %6.1f B/cyc/SM  (%s)\n", name, box_bytes, np,
               double(c) / loads, double(box_bytes) * loads / c, cudaGetErrorString(e));
        }
    };
    {  // 2-D tiled: rows of 128 B (64 bf16), box 64 x R rows
        for (int rows : {32, 64, 128, 256}) {
            CUtensorMap m;
            cuuint64_t gd[2] = {64, cuuint64_t(N) * H * W};
            cuuint64_t gs[1] = {128};
            cuuint32_t box[2] = {64, cuuint32_t(rows)};
            cuuint32_t es[2] = {1, 1};
            enc_tiled(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            char nm[64];
            snprintf(nm, 64, "tiled 2D 128B x %d rows (SW128)", rows);
            run(nm, m, 0, rows * 128);
        }
    }
    {  // im2col: 128 pixels x 64 ch
        for (int px : {64, 128, 256}) {
            CUtensorMap m;
            cuuint64_t gd[4] = {cuuint64_t(C), cuuint64_t(W), cuuint64_t(H), cuuint64_t(N)};
            cuuint64_t gs[3] = {cuuint64_t(C * 2), cuuint64_t(W * C * 2), cuuint64_t(H * W * C * 2)};
            int lo[2] = {-1, -1}, up[2] = {-1, -1};
            cuuint32_t es[4] = {1, 1, 1, 1};
            enc_im2col(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, x, gd, gs, lo, up, 64, px, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            char nm[64];
            snprintf(nm, 64, "im2col 4D %d px x 64 ch (SW128)", px);
            run(nm, m, 1, px * 128);
        }
    }
    {  // 4-D tiled pixel row: {64 ch, W px, 1, 1}
        CUtensorMap m;
        cuuint64_t gd[4] = {cuuint64_t(C), cuuint64_t(W), cuuint64_t(H), cuuint64_t(N)};
        cuuint64_t gs[3] = {cuuint64_t(C * 2), cuuint64_t(W * C * 2), cuuint64_t(H * W * C * 2)};
        cuuint32_t box[4] = {64, 56, 1, 1};
        cuuint32_t es[4] = {1, 1, 1, 1};
        enc_tiled(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, x, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        run("tiled 4D pixel row 56 px x 64 ch (SW128)", m, 2, 56 * 128);
    }
    return 0;
}
