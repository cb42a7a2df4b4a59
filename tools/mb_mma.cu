// tcgen05.mma throughput (cycles per instruction, one CTA per SM on all
// SMs, descriptors precomputed, 8 MMAs unrolled per loop trip) for the
// shapes the layer GEMM can use: A and B from shared memory (SS), A from
// TMEM (TS), tcgen05.cp of the A block into TMEM (+ TS MMA); zero or
// random operands; alone and while 512 threads stream shared-memory
// loads/stores next to it (noise=3: the producers' traffic pattern).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2512_15742_b200/csrc tools/mb_mma.cu -o tools/bin/mb_mma
#include <cuda_runtime.h>

#include <cstdio>

#include "skan_tc.cuh"

using namespace skan;

constexpr int kT = 544;

__device__ __forceinline__ void mma_any(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, int kind) {
    if (kind == 3 || kind == 4) {  // cp of a 128x32B A block into TMEM (+ TS MMA for kind 3)
        asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(d + 320u), "l"(b) : "memory");
        if (kind == 4) return;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
            "r"(static_cast<uint32_t>(a)), "l"(b), "r"(idesc)
            : "memory");
    } else if (kind == 2) {  // tf32, A from TMEM (a = tmem address)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
            "r"(static_cast<uint32_t>(a)), "l"(b), "r"(idesc)
            : "memory");
    } else if (kind == 0) {
        tc::mma_tf32(d, a, b, idesc, true);
    } else {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
            "l"(a), "l"(b), "r"(idesc)
            : "memory");
    }
}

// kind 0: tf32 (K = 8 per MMA), kind 1: bf16 (K = 16 per MMA); noise: 0 none,
// 1 = 512 threads storing, 2 = loading, 3 = load + 2 stores (producer mix)
__device__ __forceinline__ uint4 lds_v(const void* p) {
    uint4 v;
    asm volatile("ld.volatile.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(tc::smem_addr(p)));
    return v;
}

__global__ void __launch_bounds__(kT, 1) k_mma(int M, int N, int kind, int reps, int noise, int swz, long long* out,
                                                int data_kind) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t s_tmem;
    __shared__ volatile int s_stop;
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t lboA = (M / 8) * 128, lboB = (N / 8) * 128;
    // A: M x 64 tf32 (or M x 128 bf16) = M * 256 B; B: N * 256 B
    unsigned char* A = smem;
    unsigned char* B = smem + M * 256;
    unsigned char* scratch = B + N * 256;  // noise region (64 KB)
    for (int q = tid * 16; q < (M + N) * 256; q += kT * 16) {
        // non-zero operands (pseudo-random f32 in [-1, 1]): the tensor pipe's rate with real data
        uint32_t h = (q * 2654435761u) ^ 0x9E3779B9u;
        float f[4];
        for (int u = 0; u < 4; ++u) {
            h = h * 1664525u + 1013904223u;
            f[u] = data_kind ? (static_cast<float>(h >> 8) * (2.0f / 16777216.0f) - 1.0f) : 0.f;
        }
        *reinterpret_cast<float4*>(smem + q) = make_float4(f[0], f[1], f[2], f[3]);
    }
    if (tid == 0) {
        s_stop = 0;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc::smem_addr(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tc::tmem_alloc<512>(&s_tmem);
    tc::fence_proxy_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = s_tmem;
    if (warp == kT / 32 - 1) {
        if ((tid & 31) == 0) {
            const uint32_t idesc = kind != 1 ? tc::idesc_tf32(M, N)
                                             : ((1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
                                                (static_cast<uint32_t>(M >> 4) << 24));
            const uint32_t a0 = tc::smem_addr(A), b0 = tc::smem_addr(B);
            uint64_t da[8], db[8];
#pragma unroll
            for (int s = 0; s < 8; ++s) {
                if (swz == 0) {
                    da[s] = tc::make_desc(a0 + s * 2 * lboA, lboA, 128);
                    db[s] = tc::make_desc(b0 + s * 2 * lboB, lboB, 128);
                } else {
                    // rows of swz bytes, 8-row atoms (SBO = 8 * swz), K blocks of swz bytes per row
                    const int per = swz / 32, kb = s / per, ks = s % per;
                    const uint64_t lt = swz == 128 ? 2ull : (swz == 64 ? 4ull : 6ull);
                    da[s] = tc::make_desc(a0 + kb * M * swz + ks * 32, 16, 8 * swz) | (lt << 61);
                    db[s] = tc::make_desc(b0 + kb * N * swz + ks * 32, 16, 8 * swz) | (lt << 61);
                }
            }
            if (kind >= 2)
#pragma unroll
                for (int s = 0; s < 8; ++s) da[s] = tmem + 256 + 8 * s;
            const long long t0 = clock64();
#pragma unroll 1
            for (int r = 0; r < reps; r += 8) {
#pragma unroll
                for (int s = 0; s < 8; ++s) mma_any(tmem, da[s], db[s], idesc, kind);
            }
            tc::mma_commit(&bar);
            uint32_t done = 0;
            while (!done) {
                asm volatile(
                    "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                    : "=r"(done)
                    : "r"(tc::smem_addr(&bar))
                    : "memory");
            }
            const long long t1 = clock64();
            s_stop = 1;
            if (blockIdx.x == 0) out[0] = t1 - t0;
        }
    } else if (noise) {
        long long ops = 0;
        uint4 acc = make_uint4(tid, 0, 0, 0);
        while (!s_stop) {
#pragma unroll 4
            for (int u = 0; u < 16; ++u) {
                const uint32_t o = ((tid + u * 512) * 16) & 0xFFFF;
                uint4* p = reinterpret_cast<uint4*>(scratch + o);
                if (noise == 1) {
                    *p = acc;
                } else if (noise == 2) {
                    const uint4 v = lds_v(p);
                    acc.x ^= v.x;
                } else {
                    const uint4 v = lds_v(p);
                    acc.y += v.y;
                    *reinterpret_cast<uint4*>(scratch + (o ^ 0x8000)) = acc;
                    *reinterpret_cast<uint4*>(scratch + (o ^ 0x4000)) = acc;
                }
            }
            ops += 16;
        }
        if (blockIdx.x == 0 && tid == 0) out[1] = ops;
        if (acc.x == 0xFFFFFFFF) out[2] = acc.y;
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_free<512>(tmem);
}

int main() {
    long long* d;
    cudaMalloc(&d, 64);
    const int smem = 200 * 1024;
    cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    struct S { int M, N, kind; } shapes[] = {{64, 128, 0}, {128, 128, 0}, {64, 256, 0}, {128, 256, 0}, {128, 128, 1}, {128, 256, 1}, {128, 128, 2}, {128, 256, 2}, {64, 256, 2}, {128, 128, 3}, {128, 128, 4}};
    const int reps = 4096;
    for (int dk : {0, 1})
    for (int swz : {0})
    for (auto sh : shapes) {
        for (int noise = 0; noise < 4; noise += 3) {
            long long h[2] = {0, 0};
            cudaMemset(d, 0, 64);
            k_mma<<<148, kT, smem>>>(sh.M, sh.N, sh.kind, reps, noise, swz, d, dk);
            k_mma<<<148, kT, smem>>>(sh.M, sh.N, sh.kind, reps, noise, swz, d, dk);
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            const double cpm = static_cast<double>(h[0]) / reps;
            const int kk = sh.kind == 1 ? 16 : 8;
            const double flop_clk = 2.0 * sh.M * sh.N * kk / cpm;
            printf("data%d swz%3d %s M=%3d N=%3d noise=%d: %6.1f clk/mma  %7.0f flop/clk/SM  operand B/clk %5.1f  noise ops/thread %lld %s\n",
                   dk, swz, sh.kind == 1 ? "bf16" : (sh.kind == 2 ? "tf32-TS" : (sh.kind == 3 ? "cp+TS" : (sh.kind == 4 ? "cp-only" : "tf32"))), sh.M, sh.N, noise, cpm, flop_clk, (sh.M + sh.N) * 32.0 / cpm, h[1],
                   e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    }
    return 0;
}
