// desc_probe.cu -- can a tcgen05 K-major SW128 A operand start at a row that is
// not a multiple of the 8-row (1024 B) swizzle atom?  (Needed for "halo"
// tiles: a 3x3 tap <r,s> = the loaded input rows shifted by s pixels = s
// 128-byte rows.)  Writes a 136 x 64 bf16 A tile in the TMA SW128 layout
// (16-byte chunk c of row r at ((c ^ (r & 7)) << 4), rows 1024-aligned), a
// 64 x 64 MN-major SW128 B tile, then for shift s computes
// D = A[s : s+128, :] @ B with the descriptor start moved by s*128 bytes and
// the descriptor's base-offset field (bits 49-51) set per variant; compares
// with the host product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2110_03901_b200/csrc \
//        tools/desc_probe.cu -o tools/desc_probe
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "conv_kernel.cuh"

using namespace imconv;

constexpr int kARows = 136;

__global__ void __launch_bounds__(128, 1) probe(const __nv_bfloat16 *a, const __nv_bfloat16 *b, int shift,
                                               int variant, float *out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sa = smem;               // 136 rows x 128 B (17 KB, padded to 18 KB)
    uint8_t *sb = smem + 18 * 1024;   // 64 k-rows x 128 B
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // A: row r, 16-byte chunk c (8 bf16 channels) -> SW128 position
    for (int i = threadIdx.x; i < kARows * 8; i += blockDim.x) {
        const int r = i / 8, c = i % 8;
        uint4 v = *reinterpret_cast<const uint4 *>(a + r * 64 + c * 8);
        *reinterpret_cast<uint4 *>(sa + r * 128 + ((c ^ (r & 7)) << 4)) = v;
    }
    // B (MN-major): k-row k holds 64 n values (128 B), SW128 by k-row
    for (int i = threadIdx.x; i < 64 * 8; i += blockDim.x) {
        const int k = i / 8, c = i % 8;
        uint4 v = *reinterpret_cast<const uint4 *>(b + k * 64 + c * 8);
        *reinterpret_cast<uint4 *>(sb + k * 128 + ((c ^ (k & 7)) << 4)) = v;
    }
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 0) ptx::tmem_alloc<64>(&tslot);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tslot;
    if (warp == 0) {
        const uint32_t idesc = make_idesc<ELEM_BF16, 64>();
        const uint32_t a_addr = ptx::smem_u32(sa) + shift * 128;
        uint64_t adesc = ptx::smem_desc(variant == 2 ? (a_addr & ~1023u) : a_addr, 16, 1024, ptx::LAYOUT_SW128);
        if (variant == 1) adesc |= static_cast<uint64_t>(shift & 7) << 49;
        if (variant == 2) {
            // start rounded down to the atom, phase in the base-offset field
            adesc = ptx::smem_desc(a_addr, 16, 1024, ptx::LAYOUT_SW128) | (static_cast<uint64_t>(shift & 7) << 49);
        }
        const uint64_t bdesc = ptx::smem_desc(ptx::smem_u32(sb), 8192, 1024, ptx::LAYOUT_SW128);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
            ptx::mma_f16_elect(tmem, adesc + (kk * 32 >> 4), bdesc + (kk * 2048 >> 4), idesc, kk > 0);
        ptx::mma_commit_elect(&bar);
    }
    ptx::mbar_wait(&bar, 0);
    ptx::tc_fence_after();
    uint32_t v[32];
    for (int h = 0; h < 2; ++h) {
        ptx::tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + h * 32, v);
        ptx::tmem_ld_wait();
        for (int j = 0; j < 32; ++j) out[(warp * 32 + lane) * 64 + h * 32 + j] = __uint_as_float(v[j]);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc<64>(tmem);
}

int main() {
    std::vector<__nv_bfloat16> ha(kARows * 64), hb(64 * 64);
    std::vector<float> fa(kARows * 64), fb(64 * 64);
    uint32_t seed = 12345;
    auto rnd = [&]() { seed = seed * 1664525u + 1013904223u; return static_cast<int>((seed >> 16) % 9) - 4; };
    for (int i = 0; i < kARows * 64; ++i) { fa[i] = static_cast<float>(rnd()); ha[i] = __float2bfloat16(fa[i]); }
    for (int i = 0; i < 64 * 64; ++i) { fb[i] = static_cast<float>(rnd()); hb[i] = __float2bfloat16(fb[i]); }
    __nv_bfloat16 *da, *db;
    float *dout;
    cudaMalloc(&da, ha.size() * 2);
    cudaMalloc(&db, hb.size() * 2);
    cudaMalloc(&dout, 128 * 64 * 4);
    cudaMemcpy(da, ha.data(), ha.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(db, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
    std::vector<float> hout(128 * 64);
    const char *names[3] = {"start+s*128, base_offset 0", "start+s*128, base_offset s&7", "start+s*128 | bo (dup)"};
    for (int variant = 0; variant < 2; ++variant) {
        for (int shift : {0, 1, 2, 3, 5, 7, 8}) {
            probe<<<1, 128, 40 * 1024>>>(da, db, shift, variant, dout);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            cudaMemcpy(hout.data(), dout, hout.size() * 4, cudaMemcpyDeviceToHost);
            double maxerr = 0;
            for (int m = 0; m < 128; ++m)
                for (int n = 0; n < 64; ++n) {
                    double ref = 0;
                    for (int k = 0; k < 64; ++k) ref += fa[(m + shift) * 64 + k] * fb[k * 64 + n];
                    maxerr = std::fmax(maxerr, std::fabs(ref - hout[m * 64 + n]));
                }
            printf("%-32s shift %d: max |err| = %g %s\n", names[variant], shift, maxerr, maxerr == 0 ? "EXACT" : "WRONG");
        }
    }
    return 0;
}
