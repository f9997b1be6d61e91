// store_bench.cu -- output-stream throughput of the epilogue's store path:
// 148 CTAs (one per SM) write a (M x K) bf16 row-major tensor (NHWC output of
// a 1x1 layer) as 128-row x 128-byte tiles, either with TMA stores from
// `nbuf` smem staging tiles kept in flight, or with coalesced st.global.v4
// from registers.  Prints TB/s for each variant.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2110_03901_b200/csrc \
//        tools/store_bench.cu -o tools/store_bench -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include "ptx.cuh"

using namespace imconv;

constexpr int kTile = 128 * 128;  // bytes of one staging tile

// mode 0: TMA store, one issuing thread, `nbuf` tiles in flight (wait_group.read nbuf-1)
// mode 1: st.global.v4 by 128 threads (each thread one 16-byte piece per row step)
__global__ void __launch_bounds__(128, 1) store_stream(const __grid_constant__ CUtensorMap m, int mode, int nbuf,
                                                      long long m_rows, int k_cols, uint8_t *y) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int col_chunks = k_cols / 64;  // 64 bf16 = 128 bytes
    const long long tiles = (m_rows / 128) * col_chunks;
    // fill the staging tiles once (contents are irrelevant)
    for (int i = threadIdx.x; i < nbuf * kTile / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(i, i + 1, i + 2, i + 3);
    ptx::fence_proxy_async_smem();
    __syncthreads();
    if (mode == 0) {
        if (threadIdx.x == 0) {
            int it = 0;
            for (long long t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
                const int c = static_cast<int>(t % col_chunks);
                const long long r = t / col_chunks;
                ptx::tma_store_2d(&m, smem + (it % nbuf) * kTile, c * 64, static_cast<int>(r * 128));
                ptx::tma_store_commit();
                switch (nbuf) {
                    case 1: ptx::tma_store_wait_read<0>(); break;
                    case 2: ptx::tma_store_wait_read<1>(); break;
                    case 4: ptx::tma_store_wait_read<3>(); break;
                    default: ptx::tma_store_wait_read<7>(); break;
                }
            }
            ptx::tma_store_wait<0>();
        }
    } else {
        // each tile: 128 rows x 128 bytes = 1024 x 16 B; 128 threads x 8 iterations,
        // 8 consecutive threads cover one row's 128 bytes
        const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
        for (long long t = blockIdx.x; t < tiles; t += gridDim.x) {
            const int c = static_cast<int>(t % col_chunks);
            const long long r = t / col_chunks;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int piece = i * 128 + threadIdx.x;
                const long long row = r * 128 + (piece >> 3);
                uint4 *dst = reinterpret_cast<uint4 *>(y + (row * k_cols + c * 64) * 2) + (piece & 7);
                *dst = v;
            }
        }
    }
}

int main() {
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    const long long M = 50176;  // 256 x 14 x 14 output pixels (s4 1x1b)
    const int K = 1024;
    uint8_t *y;
    cudaMalloc(&y, M * K * 2);
    CUtensorMap tm;
    cuuint64_t gdim[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(M)};
    cuuint64_t gstride[1] = {static_cast<cuuint64_t>(K * 2)};
    cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, y, gdim, gstride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(store_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 9 * kTile);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    // an L2-sized scrub buffer so each run starts with the output not resident
    uint8_t *scrub;
    const size_t scrub_bytes = 256ull << 20;
    cudaMalloc(&scrub, scrub_bytes);
    struct V { int mode, nbuf; const char *name; } vs[] = {
        {0, 1, "TMA store, 1 tile in flight"}, {0, 2, "TMA store, 2 tiles in flight"},
        {0, 4, "TMA store, 4 tiles in flight"}, {0, 8, "TMA store, 8 tiles in flight"},
        {1, 1, "st.global.v4 coalesced (128 thr)"}};
    for (const V &v : vs) {
        float best = 1e9f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaMemsetAsync(scrub, rep, scrub_bytes);
            cudaEventRecord(e0);
            store_stream<<<148, 128, 9 * kTile>>>(tm, v.mode, v.nbuf, M, K, y);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep > 0 && ms < best) best = ms;
        }
        const double bytes = static_cast<double>(M) * K * 2;
        printf("%-36s %8.2f us  %6.2f TB/s\n", v.name, best * 1e3, bytes / (best * 1e-3) / 1e12);
    }
    // per-SM ceiling: the same TMA store stream (2 tiles in flight) from fewer CTAs
    for (int nb : {2, 0})
    for (int ctas : {37, 56, 74, 148}) {
        float best = 1e9f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaMemsetAsync(scrub, rep, scrub_bytes);
            cudaEventRecord(e0);
            store_stream<<<ctas, 128, 9 * kTile>>>(tm, nb ? 0 : 1, nb ? nb : 1, M, K, y);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep > 0 && ms < best) best = ms;
        }
        const double bytes = static_cast<double>(M) * K * 2;
        printf("%s %d, %3d CTAs     %8.2f us  %6.2f TB/s  %5.1f GB/s per SM\n", nb ? "TMA store, in flight" : "st.global.v4 (128 thr)", nb, ctas, best * 1e3,
               bytes / (best * 1e-3) / 1e12, bytes / (best * 1e-3) / 1e9 / ctas);
    }
    cudaError_t err = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(err));
    return 0;
}
