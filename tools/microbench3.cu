// Grid-barrier variants for the persistent batch-1 kernel, 148 CTAs x 256
// threads, cooperative launch; CTA 0 clock64 per barrier (median of 10
// barriers inside one launch, warm).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/microbench3.cu -o tools/microbench3.bin
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

// A: single counter + generation, one polling thread per CTA
__device__ void bar_counter(unsigned* b) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* vgen = b + 32;
        const unsigned gen = *vgen;
        __threadfence();
        if (atomicAdd(b, 1u) == gridDim.x - 1) {
            b[0] = 0;
            __threadfence();
            atomicAdd(b + 32, 1u);
        } else {
            while (*vgen == gen) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// B: 16 group counters on separate 128-B lines, top counter, gen; one poller per CTA
__device__ void bar_tree(unsigned* b) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* vgen = b + 32;
        const unsigned gen = *vgen;
        const int g = blockIdx.x & 15;
        const unsigned members = (gridDim.x - g + 15) / 16;
        __threadfence();
        bool rel = false;
        if (atomicAdd(b + 64 + 32 * g, 1u) == members - 1) {
            b[64 + 32 * g] = 0;
            if (atomicAdd(b, 1u) == 15) {
                b[0] = 0;
                rel = true;
            }
        }
        if (rel) {
            __threadfence();
            atomicAdd(b + 32, 1u);
        } else {
            while (*vgen == gen) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// C: per-CTA flags, but only CTA-local warp 0 polls 32 flags at a time...
// (each CTA: 148 flags read by 148 threads -> hot spot) -- reference variant
__device__ void bar_flags(unsigned* f, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f + blockIdx.x * 32), "r"(target));
    if (threadIdx.x < gridDim.x) {
        unsigned v;
        do {
            asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f + threadIdx.x * 32));
        } while (static_cast<int>(v - target) < 0);
    }
    __syncthreads();
    if (threadIdx.x == 0) __threadfence();
    __syncthreads();
}

__global__ void k(unsigned* bars, unsigned* flags, unsigned epoch, long long* out) {
    cg::grid_group grid = cg::this_grid();
    long long t0, acc[4] = {0, 0, 0, 0};
    for (int rep = 0; rep < 10; ++rep) {
        __syncthreads();
        t0 = clock64();
        grid.sync();
        acc[0] += clock64() - t0;
        __syncthreads();
        t0 = clock64();
        bar_counter(bars);
        acc[1] += clock64() - t0;
        __syncthreads();
        t0 = clock64();
        bar_tree(bars + 1024);
        acc[2] += clock64() - t0;
        __syncthreads();
        t0 = clock64();
        bar_flags(flags, epoch + rep + 1);
        acc[3] += clock64() - t0;
    }
    if (threadIdx.x == 0 && blockIdx.x == 0)
        for (int i = 0; i < 4; ++i) out[i] = acc[i] / 10;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned *bars, *flags;
    long long* out;
    cudaMalloc(&bars, 64 * 1024);
    cudaMalloc(&flags, 64 * 1024);
    cudaMalloc(&out, 64);
    cudaMemset(bars, 0, 64 * 1024);
    cudaMemset(flags, 0, 64 * 1024);
    unsigned epoch = 0;
    for (int rep = 0; rep < 50; ++rep, epoch += 16) {
        void* args[] = {&bars, &flags, &epoch, &out};
        cudaLaunchCooperativeKernel((void*)k, sms, 256, args, 0, 0);
    }
    cudaDeviceSynchronize();
    long long h[4];
    cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
    printf("cg grid.sync %lld | counter %lld | tree %lld | flags(spread, relaxed poll) %lld cycles; err %s\n", h[0],
           h[1], h[2], h[3], cudaGetErrorString(cudaGetLastError()));
    return 0;
}
