// The layer GEMM's per-chunk MMA sequence in isolation (one CTA per SM on
// all SMs): per chunk of KC = 40 (5 K steps), A (128 x 40, two buffers) and
// W (256 x 40, two stages) from shared memory, either
//   variant 0: per step one M128 N256 (A_hi x [W_hi|W_lo]) + one M128 N128 (A_lo x W_hi)
//   variant 1: per step two M128 N256
//   variant 2: per step three M128 N128
// with a tcgen05.commit per chunk; modes: no commits, commit/wait round
// trip, 512 threads of scattered shared stores / random 16 B global gathers
// / proxy fences next to the MMAs, and the kernel's two-stage
// full/free mbarrier handshake with 512 producer threads doing no work.
// Prints cycles per chunk.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2512_15742_b200/csrc tools/mb_chunk.cu -o tools/bin/mb_chunk
#include <cuda_runtime.h>

#include <cstdio>

#include "skan_tc.cuh"

using namespace skan;

__global__ void __launch_bounds__(544, 1) k_chunks(int chunks, int variant, long long* out, const uint4* gbuf) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ __align__(8) uint64_t fullb[2];
    __shared__ uint32_t s_tmem;
    const int KC = 40;
    const uint32_t tile_a = 128 * KC * 4, tile_w = 256 * KC * 4;  // 20 KB, 40 KB
    unsigned char* A = smem;                   // 2 buffers x (A_hi | A_lo) = 80 KB
    unsigned char* W = smem + 4 * tile_a;      // 2 stages = 80 KB
    for (int q = threadIdx.x * 16; q < 4 * tile_a + 2 * tile_w; q += 544 * 16) {
        uint32_t h = q * 2654435761u;
        *reinterpret_cast<float4*>(smem + q) = make_float4(__uint_as_float((h & 0x3FFFFFFF) | 0x3F000000), 0.5f, -0.25f, 1.f);
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc::smem_addr(&bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc::smem_addr(&bar[1])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc::smem_addr(&fullb[0])), "r"(512));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc::smem_addr(&fullb[1])), "r"(512));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __shared__ volatile int s_stop;
    if (threadIdx.x == 0) s_stop = 0;
    if (threadIdx.x < 32) tc::tmem_alloc<256>(&s_tmem);
    tc::fence_proxy_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = s_tmem;
    auto waitp = [](uint64_t* b, unsigned par) {
        uint32_t ok = 0;
        while (!ok)
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                : "=r"(ok)
                : "r"(tc::smem_addr(b)), "r"(par)
                : "memory");
    };
    if ((variant & 512) && threadIdx.x >= 32) {
        // the kernel's handshake with no work: wait for chunk c-2's MMAs, fence, arrive
        for (int c = 0; c < chunks; ++c) {
            if (c >= 2) waitp(&bar[c & 1], ((c - 2) >> 1) & 1);
            tc::fence_proxy_async();
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_addr(&fullb[c & 1])) : "memory");
        }
    } else if (threadIdx.x >= 32) {
        // producer-like traffic next to the MMAs: noise bit 64 = scattered
        // 4-byte shared stores, bit 128 = 16-byte random global gathers
        const int noise = variant & (64 | 128 | 256);
        unsigned char* scratch = smem + 4 * tile_a + 2 * tile_w;  // 16 KB past the operands
        uint32_t h = threadIdx.x * 2654435761u + blockIdx.x;
        uint4 acc = make_uint4(0, 0, 0, 0);
        while (noise && !s_stop) {
#pragma unroll 4
            for (int u = 0; u < 8; ++u) {
                h = h * 1664525u + 1013904223u;
                if (noise & 64)
                    *reinterpret_cast<float*>(scratch + ((threadIdx.x * 16 + u * 4) & 0x3FFC)) = __uint_as_float(h);
                if (noise & 128) {
                    const uint4 v = __ldg(gbuf + (h >> 16));  // 65536 x 16 B = 1 MB
                    acc.x ^= v.x;
                }
                if ((variant & 256) && u == 7) tc::fence_proxy_async();  // the producers' per-chunk proxy fence
            }
        }
        if (acc.x == 0x12345678u) out[7] = acc.y;
    }
    if (threadIdx.x < 32) {
        const uint32_t lboA = 16 * 128, lboW = 32 * 128;
        const uint64_t da0 = tc::make_desc(tc::smem_addr(A), lboA, 128);
        const uint64_t dw0 = tc::make_desc(tc::smem_addr(W), lboW, 128);
        const uint32_t i2 = tc::idesc_tf32(128, 256), i1 = tc::idesc_tf32(128, 128);
        const uint64_t sA = (2 * lboA) >> 4, sW = (2 * lboW) >> 4;
        const int v = variant & 3;
        const long long t0 = clock64();
        for (int c = 0; c < chunks; ++c) {
            if (variant & 512) {
                waitp(&fullb[c & 1], (c >> 1) & 1);
                tc::fence_after_sync();
            }
            const uint64_t da = da0 + (c & 1) * ((2 * tile_a) >> 4), dw = dw0 + (c & 1) * (tile_w >> 4);
#pragma unroll
            for (int s = 0; s < 5; ++s) {
                if (v == 0) {
                    tc::mma_tf32_ss_warp(tmem, da + s * sA, dw + s * sW, i2, (c | s) != 0);
                    tc::mma_tf32_ss_warp(tmem, da + (tile_a >> 4) + s * sA, dw + s * sW, i1, 1u);
                } else if (v == 1) {
                    tc::mma_tf32_ss_warp(tmem, da + s * sA, dw + s * sW, i2, (c | s) != 0);
                    tc::mma_tf32_ss_warp(tmem, da + (tile_a >> 4) + s * sA, dw + s * sW, i2, 1u);
                } else {
                    tc::mma_tf32_ss_warp(tmem, da + s * sA, dw + s * sW, i1, (c | s) != 0);
                    tc::mma_tf32_ss_warp(tmem + 128, da + s * sA, dw + (2048 >> 4) + s * sW, i1, (c | s) != 0);
                    tc::mma_tf32_ss_warp(tmem, da + (tile_a >> 4) + s * sA, dw + s * sW, i1, 1u);
                }
            }
            if (!(variant & 16)) tc::mma_commit_warp(&bar[c & 1]);
            if (variant & 32) {  // round trip: wait for this chunk's commit before the next
                uint32_t ok = 0;
                while (!ok)
                    asm volatile(
                        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                        : "=r"(ok)
                        : "r"(tc::smem_addr(&bar[c & 1])), "r"((c >> 1) & 1)
                        : "memory");
            }
        }
        tc::mma_commit_warp(&bar[0]);
        // wait for everything: the last commit on bar[0]
        uint32_t done = 0;
        const unsigned par = (variant & 16) ? 0u : (((chunks + 1) / 2) & 1);  // same count in round-trip mode
        if (variant & 32) {  // bar[0] has completed ceil(chunks/2) phases; one more arrive from the final commit
            // (wait parity for the final commit's phase)
        }
        while (!done)
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(tc::smem_addr(&bar[0])), "r"(par)
                : "memory");
        const long long t1 = clock64();
        if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
        if (threadIdx.x == 0) s_stop = 1;
    }
    tc::fence_before_sync();
    __syncthreads();
    if (threadIdx.x < 32) tc::tmem_free<256>(tmem);
}

int main() {
    long long* d;
    cudaMalloc(&d, 64);
    const int smem = 4 * 128 * 40 * 4 + 2 * 256 * 40 * 4 + 16384;
    uint4* gbuf;
    cudaMalloc(&gbuf, 1 << 20);
    cudaMemset(gbuf, 1, 1 << 20);
    cudaFuncSetAttribute(k_chunks, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int chunks = 400;
    const char* names[] = {"N256+N128 (kernel)", "2 x N256", "3 x N128"};
    const int flag_list[] = {0, 16, 32, 64, 128, 192, 256 | 64, 256 | 192, 512};
    const char* flag_names[] = {"commit/chunk", "no commits  ", "round trip  ", "+smem stores", "+gathers    ", "+both       ",
                                "+stores+fence", "+all+fence  ", "2-stage handshake"};
    for (int nc = 0; nc < 9; ++nc)
        for (int v = 0; v < 3; ++v) {
            long long h = 0;
            const int flags = flag_list[nc];
            k_chunks<<<148, 544, smem>>>(chunks, v | flags, d, gbuf);
            k_chunks<<<148, 544, smem>>>(chunks, v | flags, d, gbuf);
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            printf("%-20s %s: %7.1f clk/chunk  %s\n", names[v], flag_names[nc],
                   static_cast<double>(h) / chunks, e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    return 0;
}
