// l2_bench.cu -- aggregate L2 -> SM bandwidth of TMA tile loads, by footprint and
// sharing pattern.  Every CTA (one per SM) streams 2-D tiled boxes of a
// (rows x 128 B) matrix into a deep shared-memory ring (2 producer threads, the
// consumer frees a slot as soon as it lands), so the ring is never the limit:
// kRingBytes / latency stays well above the per-SM rate the conv kernels need.
//
//   mode 0  distinct : CTA b loads box (b + i * G) -- every SM a different box (the A stream)
//   mode 1  shared   : every CTA loads box i       -- all SMs the same box at about the same time (the B stream)
//   mode 3  pairs    : SM pairs share (box (b/2 + i * G/2))
//   mode 4  window   : CTA b cycles through its own 512 KB window
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2110_03901_b200/csrc tools/l2_bench.cu -o tools/l2_bench -lcuda
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include "ptx.cuh"

using namespace imconv;

constexpr int kRingBytes = 192 * 1024;
constexpr int kWindow = 512 * 1024;  // mode 4: each CTA re-reads its own 512 KB window (one 2 MB page: no TLB misses)

// kind 0: 2-D tiled box {128 B, box_rows}; kind 1: 4-D im2col box of box_rows pixels x 128 B over an
// NHWC (C = 64) tensor with 3x3 taps; kind 2: 3-D tiled box {128 B, 64 rows, box_rows / 64}
__global__ void __launch_bounds__(256, 1) l2_stream(const __grid_constant__ CUtensorMap m, int mode, int loads,
                                                   int box_rows, int nboxes, int slots, int nprod, int kind) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[64], empty[64];
    if (threadIdx.x == 0) {
        for (int i = 0; i < slots; ++i) {
            ptx::mbar_init(&full[i], 1);
            ptx::mbar_init(&empty[i], 1);
        }
        ptx::fence_barrier_init();
    }
    __syncthreads();
    const uint64_t pol = ptx::policy_evict_normal();
    const int box_bytes = box_rows * 128;
    const int G = gridDim.x, b = blockIdx.x;
    // producer warp g (lane 0) owns ring slots [g * spp, (g + 1) * spp) and takes loads g, g + nprod, ...;
    // consumer warp 4 + g (lane 0) frees them.  No divisions inside the loops.
    const int grp = (threadIdx.x >> 5) & 3;
    const int spp = slots / nprod;
    const bool producer = (threadIdx.x & 31) == 0 && (threadIdx.x >> 5) < nprod;
    const bool consumer = (threadIdx.x & 31) == 0 && (threadIdx.x >> 5) >= 4 && grp < nprod;
    if (producer) {
        const int win = kWindow / box_bytes;
        int s = 0;
        uint32_t ph = 1;
        // box index of load i = grp, stepping by `step` per load of this producer, wrapping at nboxes
        int bx, step;
        switch (mode) {
            case 0: bx = (b + grp * G) % nboxes; step = (nprod * G) % nboxes; break;
            case 1: bx = grp % nboxes; step = nprod; break;
            case 3: bx = ((b >> 1) + grp * (G >> 1)) % nboxes; step = (nprod * (G >> 1)) % nboxes; break;
            default: bx = grp % win; step = nprod % win; break;
        }
        const int wrap = mode == 4 ? win : nboxes;
        const int base = mode == 4 ? b * win : 0;
        int tap = grp % 9;
        for (int i = grp; i < loads; i += nprod) {
            uint64_t *fb = &full[grp * spp + s], *eb = &empty[grp * spp + s];
            ptx::mbar_wait(eb, ph);
            ptx::mbar_arrive_expect_tx(fb, box_bytes);
            uint8_t *dst = smem + (grp * spp + s) * box_bytes;
            const int bb = base + bx;
            if (kind == 0) {
                ptx::tma_load_2d(dst, &m, fb, 0, bb * box_rows, pol);
            } else if (kind == 1) {
                // pixel bb * box_rows of the (N, 56, 56) grid, 3x3 taps, pad 1 (box_rows divides 3136 * 8)
                const int px = bb * box_rows;
                const int n = px / 3136, rem = px - n * 3136;
                const int hh = rem / 56;
                ptx::tma_load_im2col_4d(dst, &m, fb, 0, rem - hh * 56 - 1, hh - 1, n,
                                        static_cast<uint16_t>(tap % 3), static_cast<uint16_t>(tap / 3), pol);
                tap = tap + 1 == 9 ? 0 : tap + 1;
            } else {
                ptx::tma_load_3d(dst, &m, fb, 0, 0, bb * (box_rows / 64), pol);
            }
            bx += step;
            if (bx >= wrap) bx -= wrap;
            if (++s == spp) {
                s = 0;
                ph ^= 1;
            }
        }
    } else if (consumer) {
        int s = 0;
        uint32_t ph = 0;
        for (int i = grp; i < loads; i += nprod) {
            ptx::mbar_wait(&full[grp * spp + s], ph);
            ptx::mbar_arrive(&empty[grp * spp + s]);
            if (++s == spp) {
                s = 0;
                ph ^= 1;
            }
        }
    }
}

int main(int argc, char **argv) {
    PFN_cuTensorMapEncodeTiled_v12000 enc_tiled;
    PFN_cuTensorMapEncodeIm2col_v12000 enc_im2col;
    cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", (void **)&enc_im2col, cudaEnableDefault, nullptr);
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc_tiled, cudaEnableDefault, &q);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t cap = size_t(2) << 30;
    void *x;
    cudaMalloc(&x, cap);
    cudaMemset(x, 1, cap);
    cudaFuncSetAttribute(l2_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, kRingBytes + 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char *names[5] = {"distinct", "shared", "mixed", "sm-pairs", "own 512 KB window"};
    const char *kinds[3] = {"tiled 2-D", "im2col 4-D", "tiled 3-D"};
    printf("| kind | footprint | box | slots | producers | CTAs | pattern | GB/s aggregate | B/clk/SM @1.965 GHz | clk/op |\n|---|---|---|---|---|---|---|---|---|---|\n");
    auto run = [&](int kind, size_t fp_mb, int box_rows, int ring_kb, int nprod, int ctas, int mode) {
        const int box_bytes = box_rows * 128;
        int slots = ring_kb * 1024 / box_bytes;
        slots -= slots % nprod;  // a slot always belongs to the same producer
        if (slots < 2) return;
        const size_t fp = fp_mb << 20;
        const int nboxes = static_cast<int>(fp / box_bytes);
        CUtensorMap m;
        cuuint32_t es[4] = {1, 1, 1, 1};
        if (kind == 0) {
            cuuint64_t gd[2] = {64, cuuint64_t(fp / 128)};
            cuuint64_t gs[1] = {128};
            cuuint32_t box[2] = {64, cuuint32_t(box_rows)};
            enc_tiled(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else if (kind == 1) {
            cuuint64_t gd[4] = {64, 56, 56, cuuint64_t(fp / (3136 * 128))};
            cuuint64_t gs[3] = {128, 56 * 128, 3136 * 128};
            int lo[2] = {-1, -1}, up[2] = {-1, -1};
            enc_im2col(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, x, gd, gs, lo, up, 64, box_rows, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
            cuuint64_t gd[3] = {64, 64, cuuint64_t(fp / (64 * 128))};
            cuuint64_t gs[2] = {128, 64 * 128};
            cuuint32_t box[3] = {64, 64, cuuint32_t(box_rows / 64)};
            enc_tiled(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, x, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        const int loads = static_cast<int>((size_t(32) << 20) / box_bytes);  // 32 MB per CTA
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            l2_stream<<<ctas, 256, kRingBytes + 1024>>>(m, mode, loads, box_rows, kind == 1 ? nboxes - 64 : nboxes, slots,
                                                        nprod, kind);
            cudaEventRecord(e1);
            if (cudaDeviceSynchronize() != cudaSuccess) {
                printf("error: %s\n", cudaGetErrorString(cudaGetLastError()));
                exit(1);
            }
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep > 0 && ms < best) best = ms;
        }
        const double bytes = double(ctas) * loads * box_bytes;
        const double gbs = bytes / (best * 1e-3) / 1e9;
        printf("| %s | %zu MB | %d KB | %d | %d | %d | %s | %.0f | %.1f | %.0f |\n", kinds[kind], fp_mb, box_bytes / 1024,
               slots, nprod, ctas, names[mode], gbs, gbs / ctas / 1.965, box_bytes / (gbs / ctas / 1.965));
    };
    // 1. per-operation cost: box size x producers x CTAs (L2-resident footprint, distinct boxes)
    for (int kind = 0; kind < 3; ++kind)
        for (int box_rows : {32, 64, 128, 256, 512})
            for (int nprod : {1, 2, 4})
                for (int ctas : {sms, sms / 2}) {
                    if (kind == 1 && box_rows > 256) continue;
                    if (kind == 2 && box_rows < 64) continue;
                    if (kind == 0 && box_rows > 256) continue;
                    run(kind, 48, box_rows, 192, nprod, ctas, 0);
                }
    // 1b. the same from a per-CTA 512 KB window (no TLB misses in the TMA unit)
    for (int kind = 0; kind < 2; ++kind)
        for (int box_rows : {32, 128, 256})
            for (int nprod : {1, 2, 4}) run(kind, 128, box_rows, 192, nprod, sms, 4);
    // 2. ring depth
    for (int ring_kb : {32, 64, 96, 128, 192}) run(0, 48, 128, ring_kb, 2, sms, 0);
    // 3. sharing pattern and footprint (16 KB and 32 KB boxes)
    for (size_t fp_mb : {16, 48, 96, 2048})
        for (int box_rows : {128, 256})
            for (int mode : {0, 1, 3}) run(0, fp_mb, box_rows, 192, 4, sms, mode);
    return 0;
}
