// mma_bench.cu -- microbenchmark of tcgen05.mma issue throughput on one SM
// (all 148 SMs run the same loop).  Operands are static shared memory; no
// global traffic.  Prints cycles per MMA for M = 128 (cta_group::1), bf16,
// K = 16, over N and operand layouts.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2110_03901_b200/csrc tools/mma_bench.cu -o mma_bench
#include <cstdio>
#include <string>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace imconv;

// FLAGS: 1 = commit every 4 MMAs, 2 = rotate over 4 accumulators, 4 = random operand data,
//        8 = first MMA of every 28 overwrites (accumulate = 0)
template <int N, int A_MODE, int FLAGS = 0>  // A_MODE: 0 = SW128 K-major, 1 = no-swizzle K-major, 2 = A in TMEM
__global__ void __launch_bounds__(128, 1) mma_loop(int iters, long long *out_cycles) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sa = smem;              // 16 KB
    uint8_t *sb = smem + 16384;      // 32 KB
    __shared__ uint64_t bar, bar2[4];
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (16384 + 32768) / 16; i += blockDim.x) {
        uint32_t v = (FLAGS & 4) ? (uint32_t(i) * 2654435761u) & 0x3F7F3F7Fu : 0u;  // finite bf16 pairs
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(v, v ^ 0x00010001u, v ^ 0x00020002u, v ^ 0x00030003u);
    }
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        for (int i = 0; i < 4; ++i) ptx::mbar_init(&bar2[i], 1);
        ptx::fence_barrier_init();
    }
    if (warp == 0) ptx::tmem_alloc<512>(&tslot);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tbase = tslot;
    if (threadIdx.x == 0) {
        uint32_t idesc = 0;
        idesc |= 1u << 4;           // F32 accumulate
        idesc |= 1u << 7;           // A bf16
        idesc |= 1u << 10;          // B bf16
        idesc |= 1u << 16;          // B MN-major
        idesc |= (uint32_t)(N >> 3) << 17;
        idesc |= (uint32_t)(128 >> 4) << 24;
        const uint32_t a0 = ptx::smem_u32(sa), b0 = ptx::smem_u32(sb);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const int kk = it & 3;
            const uint64_t bdesc = ptx::smem_desc(b0 + kk * 2048, 8192, 1024, ptx::LAYOUT_SW128);
            if constexpr (A_MODE == 2) {
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tbase),
                    "r"(tbase + 256 + kk * 8), "l"(bdesc), "r"(idesc), "r"(1)
                    : "memory");
            } else {
                uint64_t adesc;
                if (A_MODE == 0)
                    adesc = ptx::smem_desc(a0 + kk * 32, 16, 1024, ptx::LAYOUT_SW128);
                else if (A_MODE == 1)
                    adesc = ptx::smem_desc(a0 + kk * 4096, 16, 128, ptx::LAYOUT_NONE);
                else if (A_MODE == 3)  // misaligned start, overlapping K columns (row-band pattern)
                    adesc = ptx::smem_desc(a0 + (it & 7) * 16, 16, 128, ptx::LAYOUT_NONE);
                else if (A_MODE == 4)  // 128-aligned start, LBO = 16 (overlapping K columns)
                    adesc = ptx::smem_desc(a0 + kk * 1024, 16, 128, ptx::LAYOUT_NONE);
                else if (A_MODE == 5)  // misaligned start, LBO = 2048
                    adesc = ptx::smem_desc(a0 + (it & 7) * 16, 2048, 128, ptx::LAYOUT_NONE);
                else                   // 128-aligned start, LBO = 2048
                    adesc = ptx::smem_desc(a0 + kk * 128, 2048, 128, ptx::LAYOUT_NONE);
                const uint32_t d = (FLAGS & 2) ? tbase + ((it >> 2) & 3) * 64 : tbase;
                const uint32_t accf = (FLAGS & 8) ? ((it % 28) != 0) : 1u;
                ptx::mma_f16(d, adesc, bdesc, idesc, accf);
            }
            if ((FLAGS & 1) && kk == 3) ptx::mma_commit(&bar2[(it >> 2) & 3]);
        }
        ptx::mma_commit(&bar);
        ptx::mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (blockIdx.x == 0) *out_cycles = t1 - t0;
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tbase);
    }
}

// Replays the stem row-band MMA stream: 4 output rows x 4 tap pairs per stage,
// A = no-swizzle planes (pair offsets / LBOs of the 7x7/2 stem), B = resident
// filter (SBO 1024, LBO = 57344), 24-stage ring, commit per stage.
__global__ void __launch_bounds__(256, 1) rowband_replay(int stages, long long *out_cycles, int bmode) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar[24];
    __shared__ uint64_t done;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (200 * 1024) / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
    if (threadIdx.x == 0) {
        for (int i = 0; i < 24; ++i) ptx::mbar_init(&bar[i], 1);
        ptx::mbar_init(&done, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 0) ptx::tmem_alloc<512>(&tslot);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tbase = tslot;
    if (warp >= 1 && (bmode & 2)) ptx::mbar_wait(&done, 0);  // spinning bystanders
    if (threadIdx.x == 0) {
        uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | (8u << 17) | (8u << 24);
        const uint32_t b0 = ptx::smem_u32(smem);
        const uint32_t a0 = b0 + 57344 + 16384;
        const int off[4] = {16, 48, 2192, 2224}, lbo[4] = {16, 2128, 16, 16};
        long long t0 = clock64();
        for (int st = 0; st < stages; ++st) {
            const uint32_t a_st = a0 + (st % 24) * 4352;
            for (int j = 0; j < 4; ++j) {
                const int rr = (st + j) % 7;
                for (int pr = 0; pr < 4; ++pr) {
                    const uint64_t adesc = ptx::smem_desc(a_st + off[pr], lbo[pr], 128, ptx::LAYOUT_NONE);
                    const uint64_t bdesc = (bmode & 1) == 0
                        ? ptx::smem_desc(b0 + ((rr * 4 + pr) * 2) * 1024, 57344, 1024, ptx::LAYOUT_SW128)
                        : ptx::smem_desc(b0 + ((rr * 4 + pr) * 2) * 1024, 8192, 1024, ptx::LAYOUT_SW128);
                    ptx::mma_f16(tbase + ((st & 1) * 256) + j * 64, adesc, bdesc, idesc, 1);
                }
            }
            ptx::mma_commit(&bar[st % 24]);
        }
        ptx::mma_commit(&bar[0]);
        long long t1 = clock64();
        if (blockIdx.x == 0) *out_cycles = t1 - t0;
        ptx::mbar_arrive(&done);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tbase);
    }
}

void run_replay(int bmode) {
    long long *d;
    cudaMalloc(&d, sizeof(long long));
    cudaFuncSetAttribute(rowband_replay, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    const int stages = 2048;
    rowband_replay<<<148, 256, 210 * 1024>>>(stages, d, bmode);
    rowband_replay<<<148, 256, 210 * 1024>>>(stages, d, bmode);
    cudaError_t e = cudaDeviceSynchronize();
    long long c = 0;
    cudaMemcpy(&c, d, sizeof(c), cudaMemcpyDeviceToHost);
    printf("rowband replay bmode=%d: %.1f cyc/stage (16 MMAs), %.1f cyc/MMA (%s)\n", bmode, double(c) / stages,
           double(c) / stages / 16, cudaGetErrorString(e));
    cudaFree(d);
}

// Pipeline replay: a producer warp (warp 1) and the MMA thread (warp 0) run
// the row-band handshake on a ring of `nst` stages: producer waits empty[s],
// (optionally) fences to the async proxy, arrives full[s] (lagged by `lag`
// stages); the MMA thread waits full[s], fences, issues `mps` MMAs, commits
// empty[s].  No data movement.
// variant bits: 1 = skip tcgen05.fence::after_thread_sync, 2 = only lane 0 waits, 4 = skip __syncwarp,
//               8 = lane 0 runs the whole loop alone (no warp convergence at all)
__global__ void __launch_bounds__(256, 1) pipe_replay(int stages, int mps, int lag, int use_fence,
                                                      long long *out_cycles, int variant, int nn) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int nst = 24;
    __shared__ uint64_t full[nst], empty[nst];
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < (200 * 1024) / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; ++i) {
            ptx::mbar_init(&full[i], 32);
            ptx::mbar_init(&empty[i], 1);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 0) ptx::tmem_alloc<512>(&tslot);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tbase = tslot;
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(nn >> 3) << 17) | (8u << 24);
    const uint32_t b0 = ptx::smem_u32(smem);
    const uint32_t a0 = b0 + 57344 + 16384;
    if (warp == 1) {
        int pend[32];
        int np = 0;
        for (int st = 0; st < stages; ++st) {
            const int s = st % nst;
            if (variant & 32) {
                // no handshake: full barriers are completed without waiting for empty
            } else if (variant & 16) {
                const uint32_t a = ptx::smem_u32(&empty[s]);
                while (!ptx::mbar_try_wait(a, ((st / nst) & 1) ^ 1)) __nanosleep(256);
            } else {
                ptx::mbar_wait(&empty[s], ((st / nst) & 1) ^ 1);
            }
            pend[np++] = s;
            if (np > lag) {
                if (use_fence) ptx::fence_proxy_async_smem();
                ptx::mbar_arrive(&full[pend[0]]);
                for (int u = 0; u < lag; ++u) pend[u] = pend[u + 1];
                --np;
            }
        }
        for (int u = 0; u < np; ++u) ptx::mbar_arrive(&full[pend[u]]);
    } else if (warp == 0 && (!(variant & 8) || lane == 0)) {
        // (variant 256: the a0 region holds 4 SW128 A tiles of 16 KB for the uniform issuer)
        long long t0 = clock64();
        long long tw = 0;
        bool ready = false;  // variant 512: stage st's full barrier already seen complete (look-ahead)
        for (int st = 0; st < stages; ++st) {
            const int s = st % nst;
            const long long ta = clock64();
            if (!(variant & 64) && (!(variant & 2) || lane == 0) && !ready) ptx::mbar_wait(&full[s], (st / nst) & 1);
            tw += clock64() - ta;
            if (variant & 512) {
                const uint32_t a_u = __shfl_sync(0xffffffffu, a0, 0), b_u = __shfl_sync(0xffffffffu, b0, 0);
                const uint32_t t_u = __shfl_sync(0xffffffffu, tbase, 0);
                const uint64_t ad0 = ptx::smem_desc(a_u + (s % 4) * 16384, 16, 1024, ptx::LAYOUT_SW128);
                const uint64_t bd0 = ptx::smem_desc(b_u, 8192, 1024, ptx::LAYOUT_SW128);
                ptx::tc_fence_after();
                for (int k = 0; k < mps; ++k) {
                    ptx::mma_f16_elect(t_u, ad0 + static_cast<uint64_t>((k & 3) * 2), bd0 + static_cast<uint64_t>((k & 3) * 128),
                                       idesc, 1);
                    if (k == mps / 2 - 1) {
                        const int sn = (st + 1) % nst;
                        if (variant & 4096) {  // blocking wait for the next stage, hidden behind this stage's last MMAs
                            if (st + 1 < stages) ptx::mbar_wait(&full[sn], ((st + 1) / nst) & 1);
                            ready = true;
                        } else {
                            ready = st + 1 < stages && ptx::mbar_test_wait(ptx::smem_u32(&full[sn]), ((st + 1) / nst) & 1);
                        }
                    }
                }
                ptx::mma_commit_elect(&empty[s]);
                continue;
            }
            if (!(variant & 1)) ptx::tc_fence_after();
            if (variant & 256) {
                // the production issuer: whole warp, warp-uniform descriptors (uniform datapath)
                const uint32_t a_u = __shfl_sync(0xffffffffu, a0, 0), b_u = __shfl_sync(0xffffffffu, b0, 0);
                const uint32_t t_u = __shfl_sync(0xffffffffu, tbase, 0);
                const uint64_t ad0 = ptx::smem_desc(a_u + (s % 4) * 16384, 16, 1024, ptx::LAYOUT_SW128);
                const uint64_t bd0 = ptx::smem_desc(b_u, 8192, 1024, ptx::LAYOUT_SW128);
                for (int k = 0; k < mps; ++k)
                    ptx::mma_f16_elect(t_u, ad0 + static_cast<uint64_t>((k & 3) * 2), bd0 + static_cast<uint64_t>((k & 3) * 128),
                                       idesc, 1);
                if (variant & 1024) {
                    // one commit per pair of stages (arrives on both stages' empty barriers in turn)
                    if (st & 1) {
                        ptx::mma_commit_elect(&empty[(st - 1) % nst]);
                        ptx::mma_commit_elect(&empty[s]);
                    }
                } else if (variant & 2048) {
                    // no commit at all in the loop (producer never waits: lag large) -- lower bound
                } else {
                    ptx::mma_commit_elect(&empty[s]);
                }
            } else if (variant & 128) {
                const uint32_t a_st = a0 + s * 4352;
                for (int k = 0; k < mps; ++k) {
                    const uint64_t adesc = ptx::smem_desc(a_st + 16 + (k & 3) * 32, 16, 128, ptx::LAYOUT_NONE);
                    const uint64_t bdesc = ptx::smem_desc(b0 + (k & 7) * 2048, 57344, 1024, ptx::LAYOUT_SW128);
                    ptx::mma_f16_elect(tbase + (nn == 64 ? (k & 3) * 64 : 0), adesc, bdesc, idesc, 1);
                }
                ptx::mma_commit_elect(&empty[s]);
            } else if (lane == 0) {
                const uint32_t a_st = a0 + s * 4352;
                for (int k = 0; k < mps; ++k) {
                    const uint64_t adesc = ptx::smem_desc(a_st + 16 + (k & 3) * 32, 16, 128, ptx::LAYOUT_NONE);
                    const uint64_t bdesc = ptx::smem_desc(b0 + (k & 7) * 2048, 57344, 1024, ptx::LAYOUT_SW128);
                    ptx::mma_f16(tbase + (nn == 64 ? (k & 3) * 64 : 0), adesc, bdesc, idesc, 1);
                }
                ptx::mma_commit(&empty[s]);
            }
            if (!(variant & 12)) __syncwarp();
        }
        long long t1 = clock64();
        if (blockIdx.x == 0 && lane == 0) {
            out_cycles[0] = t1 - t0;
            out_cycles[1] = tw;
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tbase);
    }
}

void run_pipe(int mps, int lag, int fence, int variant = 0, int nn = 64) {
    long long *d;
    cudaMalloc(&d, 2 * sizeof(long long));
    cudaFuncSetAttribute(pipe_replay, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    const int stages = 4096;
    pipe_replay<<<148, 256, 210 * 1024>>>(stages, mps, lag, fence, d, variant, nn);
    pipe_replay<<<148, 256, 210 * 1024>>>(stages, mps, lag, fence, d, variant, nn);
    cudaError_t e = cudaDeviceSynchronize();
    long long cc[2] = {0, 0};
    cudaMemcpy(cc, d, sizeof(cc), cudaMemcpyDeviceToHost);
    const long long c = cc[0];
    printf("pipe replay N=%3d mps=%2d lag=%d fence=%d var=%3d: %7.1f cyc/stage %6.1f cyc/MMA  wait %.1f cyc/stage (%s)\n",
           nn, mps, lag, fence, variant, double(c) / stages, double(c) / stages / mps, double(cc[1]) / stages,
           cudaGetErrorString(e));
    cudaFree(d);
}

template <int N, int A_MODE, int FLAGS = 0>
void run(const char *name) {
    long long *d;
    cudaMalloc(&d, sizeof(long long));
    auto k = mma_loop<N, A_MODE, FLAGS>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    const int iters = 4096;
    k<<<148, 128, 64 * 1024>>>(iters, d);
    k<<<148, 128, 64 * 1024>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long c = 0;
    cudaMemcpy(&c, d, sizeof(c), cudaMemcpyDeviceToHost);
    const double macs = 128.0 * N * 16;
    printf("%-28s N=%3d  %7.1f cyc/MMA  %6.0f MAC/clk/SM  (%s)\n", name, N, double(c) / iters, macs * iters / c,
           cudaGetErrorString(e));
    cudaFree(d);
}

int main(int argc, char **argv) {
    if (argc > 1 && std::string(argv[1]) == "align") {
        // no-swizzle K-major A with plane-like LBO (2 KB): 128-B aligned starts vs starts moving by
        // 16 B (the row-band stem's tap runs)
        run<64, 6>("SS  none aligned LBO2048");
        run<64, 5>("SS  none misaligned LBO2048");
        run<128, 6>("SS  none aligned LBO2048");
        run<128, 5>("SS  none misaligned LBO2048");
        run<256, 6>("SS  none aligned LBO2048");
        run<256, 5>("SS  none misaligned LBO2048");
        run<64, 0>("SS  A=SW128");
        run<128, 0>("SS  A=SW128");
        return 0;
    }
    // pipe replay of the production issuer (variant 256: uniform datapath), N = 256:
    //   +64 = no full-barrier wait, +1 = no tcgen05 fence -> which part of the per-stage handshake costs
    for (int mps : {4, 8, 16})
        for (int v : {256, 256 + 64, 256 + 64 + 2048 + 32}) run_pipe(mps, 4, 1, v, 256);
    return 0;
    run_replay(0);
    for (int v : {0, 128}) run_pipe(4, 4, 1, v, 256);
    for (int v : {0, 128}) run_pipe(8, 4, 1, v, 256);
    for (int v : {0, 128}) run_pipe(4, 4, 1, v, 128);
    run<64, 0>("SS  A=SW128");
    run<128, 0>("SS  A=SW128");
    run<256, 0>("SS  A=SW128");
    run<64, 1>("SS  A=no-swizzle");
    run<128, 1>("SS  A=no-swizzle");
    run<256, 1>("SS  A=no-swizzle");
    run<64, 3>("SS  none misaligned LBO16");
    run<64, 4>("SS  none aligned LBO16");
    run<64, 5>("SS  none misaligned LBO2048");
    run<64, 6>("SS  none aligned LBO2048");
    run<128, 3>("SS  none misaligned LBO16");
    run<128, 6>("SS  none aligned LBO2048");
    run<64, 3, 1>("misal + commit/4");
    run<64, 3, 2>("misal + 4 accumulators");
    run<64, 3, 4>("misal + random data");
    run<64, 3, 8>("misal + overwrite/28");
    run<64, 3, 15>("misal + all");
    run<256, 0, 15>("SW128 + all");
    run<64, 2>("TS  A=TMEM");
    run<128, 2>("TS  A=TMEM");
    run<256, 2>("TS  A=TMEM");
    return 0;
}
