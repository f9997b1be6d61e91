// m64_probe.cu -- the stem's transposed formulation on tcgen05:
//   D^T (64 output channels x 256 pixels) = W^T (64 x K) * X^T (K x 256 pixels)
// A = the HWCN filter rows as an MN-major SW128 operand (M = 64 channels = one
// 128-byte row per k), B = 16-byte pixels as a K-major no-swizzle operand
// whose rows (pixels) start at a 16-byte-aligned plane offset (the row-band
// kernel's taps).  Checks the result (and reports which TMEM lanes hold the
// 64 accumulator rows), then times back-to-back MMAs of this shape against
// the current 128 x 64 x 16 form.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2110_03901_b200/csrc \
//        tools/m64_probe.cu -o tools/m64_probe
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "conv_kernel.cuh"

using namespace imconv;

template <int M, int N>
__device__ __forceinline__ uint32_t idesc_t(bool a_mn, bool b_mn) {
    uint32_t d = 0;
    d |= 1u << 4;   // F32 accumulate
    d |= 1u << 7;   // A bf16
    d |= 1u << 10;  // B bf16
    d |= (a_mn ? 1u : 0u) << 15;
    d |= (b_mn ? 1u : 0u) << 16;
    d |= static_cast<uint32_t>(N >> 3) << 17;
    d |= static_cast<uint32_t>(M >> 4) << 24;
    return d;
}

// pixels: (kPix + 16) x 16 B (8 bf16 channels) = one plane; filter: K=16 x 64 channels
constexpr int kPix = 256;

__global__ void __launch_bounds__(128, 1) probe(const __nv_bfloat16 *pix, const __nv_bfloat16 *filt, int shift,
                                               float *out, int iters, long long *cycles, int mode) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sa = smem;              // filter: 16 k-rows x 128 B (MN-major SW128), 2 KB
    uint8_t *sb = smem + 4096;       // plane: (kPix + 16) pixels x 16 B
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 16 * 8; i += blockDim.x) {  // filter k-row k, chunk c (8 channels)
        const int k = i / 8, c = i % 8;
        *reinterpret_cast<uint4 *>(sa + k * 128 + ((c ^ (k & 7)) << 4)) =
            *reinterpret_cast<const uint4 *>(filt + k * 64 + c * 8);
    }
    for (int i = threadIdx.x; i < kPix + 16; i += blockDim.x)
        *reinterpret_cast<uint4 *>(sb + i * 16) = *reinterpret_cast<const uint4 *>(pix + i * 8);
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 0) ptx::tmem_alloc<256>(&tslot);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tslot;
    if (warp == 0) {
        long long t0 = clock64();
        if (mode == 0) {
            // transposed: M = 64 (channels), N = 256 (pixels), K = 16 = 2 taps of 8 channels
            // B rows (pixels) are 16 B, core matrix = 8 rows x 16 B; second K half = next tap (+16 B: next pixel)
            const uint32_t idesc = idesc_t<64, 256>(true, false);
            const uint64_t adesc = ptx::smem_desc(ptx::smem_u32(sa), 1024 /*unused*/, 1024, ptx::LAYOUT_SW128);
            const uint64_t bdesc = ptx::smem_desc(ptx::smem_u32(sb) + shift * 16, 16, 128, ptx::LAYOUT_NONE);
            for (int it = 0; it < iters; ++it) ptx::mma_f16_elect(tmem, adesc, bdesc, idesc, it > 0 ? 1u : 0u);
        } else if (mode >= 2) {
            // the stem's issue pattern: 4 tap pairs (LBO 16 / 2144 / 16 / 16, starts 0 / 32 / 2192 / 2224 B),
            // B rows advancing per pair, 4 accumulators (output rows j) -- mode 3: commit every 16 MMAs
            const uint32_t idesc = idesc_t<128, 64>(false, true);
            const uint32_t base = ptx::smem_u32(sb);
            const uint64_t ad[4] = {ptx::smem_desc(base + 0, 16, 128, ptx::LAYOUT_NONE),
                                    ptx::smem_desc(base + 32, 2144, 128, ptx::LAYOUT_NONE),
                                    ptx::smem_desc(base + 2192 % 2048, 16, 128, ptx::LAYOUT_NONE),
                                    ptx::smem_desc(base + 2224 % 2048, 16, 128, ptx::LAYOUT_NONE)};
            const uint64_t bdesc = ptx::smem_desc(ptx::smem_u32(sa), 8192, 1024, ptx::LAYOUT_SW128);
            for (int it = 0; it < iters; it += 16) {
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int pr = 0; pr < 4; ++pr)
                        ptx::mma_f16_elect(tmem + j * 64, ad[pr], bdesc + (pr * 128 >> 4), idesc, 1u);
                if (mode == 3) {
                    ptx::mma_commit_elect(&bar);
                }
            }
        } else {
            // current form: M = 128 pixels, N = 64 channels (B = filter MN-major SW128)
            const uint32_t idesc = idesc_t<128, 64>(false, true);
            const uint64_t adesc = ptx::smem_desc(ptx::smem_u32(sb) + shift * 16, 16, 128, ptx::LAYOUT_NONE);
            const uint64_t bdesc = ptx::smem_desc(ptx::smem_u32(sa), 8192, 1024, ptx::LAYOUT_SW128);
            for (int it = 0; it < iters; ++it) ptx::mma_f16_elect(tmem, adesc, bdesc, idesc, it > 0 ? 1u : 0u);
        }
        ptx::mma_commit_elect(&bar);
        ptx::mbar_wait(&bar, 0);
        if (lane == 0) cycles[blockIdx.x] = clock64() - t0;
    }
    if (mode == 3) {
        // (warp 0 committed iters/16 + 1 times; wait for the final phase)
    }
    ptx::mbar_wait(&bar, mode == 3 ? static_cast<uint32_t>((iters / 16) & 1) : 0u);
    ptx::tc_fence_after();
    if (blockIdx.x == 0) {
        // dump all 128 lanes x 256 columns (only the first iteration's shape matters for the check)
        uint32_t v[32];
        for (int h = 0; h < 8; ++h) {
            ptx::tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + h * 32, v);
            ptx::tmem_ld_wait();
            for (int j = 0; j < 32; ++j) out[(warp * 32 + lane) * 256 + h * 32 + j] = __uint_as_float(v[j]);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc<256>(tmem);
}

int main() {
    std::vector<__nv_bfloat16> hp((kPix + 16) * 8), hf(16 * 64);
    std::vector<float> fp((kPix + 16) * 8), ff(16 * 64);
    uint32_t seed = 7;
    auto rnd = [&]() { seed = seed * 1664525u + 1013904223u; return static_cast<int>((seed >> 16) % 7) - 3; };
    for (size_t i = 0; i < hp.size(); ++i) { fp[i] = rnd(); hp[i] = __float2bfloat16(fp[i]); }
    for (size_t i = 0; i < hf.size(); ++i) { ff[i] = rnd(); hf[i] = __float2bfloat16(ff[i]); }
    __nv_bfloat16 *dp, *df;
    float *dout;
    long long *dcyc;
    cudaMalloc(&dp, hp.size() * 2);
    cudaMalloc(&df, hf.size() * 2);
    cudaMalloc(&dout, 128 * 256 * 4);
    cudaMalloc(&dcyc, 148 * 8);
    cudaMemcpy(dp, hp.data(), hp.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(df, hf.data(), hf.size() * 2, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 1024);
    std::vector<float> out(128 * 256);
    // correctness, transposed form, shift 1 (misaligned)
    for (int shift : {0, 1, 3}) {
        probe<<<1, 128, 16 * 1024>>>(dp, df, shift, dout, 1, dcyc, 0);
        if (cudaDeviceSynchronize() != cudaSuccess) { printf("launch failed\n"); return 1; }
        cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
        // D^T[m = channel][n = pixel] = sum_k W^T[m][k] X^T[k][n], k = half*8 + c:
        //   half 0: pixel n (+shift), half 1: pixel n+1 (+shift)
        int found_lanes[64];
        double maxerr = 0;
        for (int m = 0; m < 64; ++m) {
            found_lanes[m] = -1;
            for (int lane = 0; lane < 128 && found_lanes[m] < 0; ++lane) {
                double err = 0;
                for (int n = 0; n < 256; ++n) {
                    double ref = 0;
                    for (int k = 0; k < 16; ++k) {
                        const int pixel = n + shift + (k >> 3), c = k & 7;
                        ref += ff[k * 64 + m] * fp[pixel * 8 + c];
                    }
                    err = std::fmax(err, std::fabs(ref - out[lane * 256 + n]));
                }
                if (err == 0) found_lanes[m] = lane;
            }
            if (found_lanes[m] < 0) maxerr = 1;
        }
        printf("transposed M=64 N=256, shift %d: %s; lanes of rows 0,1,15,16,31,32,63 = %d %d %d %d %d %d %d\n", shift,
               maxerr == 0 ? "EXACT" : "WRONG", found_lanes[0], found_lanes[1], found_lanes[15], found_lanes[16],
               found_lanes[31], found_lanes[32], found_lanes[63]);
    }
    // throughput: 148 CTAs, 4096 MMAs each
    for (int mode : {0, 1, 2})
        for (int shift : {0, 1}) {
            const int iters = 4096;
            probe<<<148, 128, 16 * 1024>>>(dp, df, shift, dout, iters, dcyc, mode);
            cudaDeviceSynchronize();
            std::vector<long long> cyc(148);
            cudaMemcpy(cyc.data(), dcyc, 148 * 8, cudaMemcpyDeviceToHost);
            double avg = 0;
            for (long long c : cyc) avg += c;
            avg /= 148;
            const double macs = mode == 0 ? 64.0 * 256 * 16 : 128.0 * 64 * 16;
            printf("%s shift %d: %.1f cycles/MMA, %.0f MAC/clk/SM\n",
                   mode == 0 ? "M=64  N=256 (transposed)" : mode == 1 ? "M=128 N=64  (current)  " : "stem pattern (4 pairs x 4 acc)", shift, avg / iters,
                   macs / (avg / iters));
        }
    return 0;
}
