// Skeleton of the persistent batch-1 kernel's fixed costs: 148 CTAs x 256
// threads, (1) stage 2048 doubles + locate + smem histogram, (2) two flag
// grid barriers, (3) an L2 round trip; CTA 0's clock64 deltas (warm caches,
// 200 back-to-back launches so clocks are up).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Iinclude tools/microbench2.cu -o tools/microbench2.bin
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2512_15742_b200/csrc/skan_device.cuh"

using namespace skan::dev;

__device__ __forceinline__ void flag_sync(unsigned* flags, unsigned target, bool sleep) {
    __syncthreads();
    if (threadIdx.x == 0)
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x), "r"(target) : "memory");
    if (threadIdx.x < gridDim.x) {
        unsigned v;
        while (true) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + threadIdx.x) : "memory");
            if (static_cast<int>(v - target) >= 0) break;
            if (sleep) __nanosleep(8);
        }
    }
    __syncthreads();
}

__device__ __forceinline__ void flag_sync_relaxed(unsigned* flags, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        *(volatile unsigned*)(flags + blockIdx.x) = target;
    }
    if (threadIdx.x < gridDim.x) {
        while (static_cast<int>(*(volatile unsigned*)(flags + threadIdx.x) - target) < 0) {
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void k(const double* x, const long long* gkey, const double* gnode, unsigned* flags, unsigned epoch,
                  long long* out, int* err, float* sink, const float* part) {
    __shared__ long long skey[10];
    __shared__ double snode[10];
    __shared__ double s_x[2048];
    __shared__ float s_t[2048];
    __shared__ unsigned char s_bm[2048];
    __shared__ int s_h[8][32];
    long long t[12];
    int n = 0;
    __syncthreads();
    t[n++] = clock64();
    if (threadIdx.x < 10) {
        skey[threadIdx.x] = gkey[threadIdx.x];
        snode[threadIdx.x] = gnode[threadIdx.x];
    }
#pragma unroll 4
    for (int i = threadIdx.x; i < 2048; i += 256) s_x[i] = x[i];
    s_h[threadIdx.x >> 5][threadIdx.x & 31] = 0;
    __syncthreads();
    t[n++] = clock64();
#pragma unroll 1
    for (int i = threadIdx.x; i < 2048; i += 256) {
        int m;
        fast_locate_tab(skey, snode, 10, -1.0, 4.5, 4.5f, s_x[i], err, m, s_t[i]);
        s_bm[i] = static_cast<unsigned char>(m);
        atomicAdd(&s_h[threadIdx.x >> 5][m], 1);
    }
    __syncthreads();
    t[n++] = clock64();
    flag_sync(flags, epoch + 1, true);
    t[n++] = clock64();
    flag_sync(flags, epoch + 2, false);
    t[n++] = clock64();
    flag_sync_relaxed(flags, epoch + 3);
    t[n++] = clock64();
    // one L2 round trip (partials written by others)
    float v = __ldcg(part + (blockIdx.x * 256 + threadIdx.x) % 4096);
    __syncthreads();
    t[n++] = clock64();
    sink[blockIdx.x * 256 + threadIdx.x] = v + s_t[threadIdx.x] + s_bm[threadIdx.x] + s_h[0][threadIdx.x & 31];
    if (threadIdx.x == 0 && blockIdx.x == 0)
        for (int i = 1; i < n; ++i) out[i - 1] = t[i] - t[i - 1];
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *x, *node;
    long long *key, *out;
    unsigned* flags;
    int* err;
    float *sink, *part;
    cudaMalloc(&x, 2048 * 8);
    cudaMalloc(&key, 80);
    cudaMalloc(&node, 80);
    cudaMalloc(&flags, 4096);
    cudaMalloc(&out, 128);
    cudaMalloc(&err, 4);
    cudaMalloc(&sink, sms * 256 * 4);
    cudaMalloc(&part, 4096 * 4);
    cudaMemset(flags, 0, 4096);
    cudaMemset(part, 0, 4096 * 4);
    double hx[2048], hn[10];
    long long hk[10];
    for (int i = 0; i < 2048; ++i) hx[i] = -1.4 + 2.8 * (i * 7919 % 2048) / 2047.0;
    for (int i = 0; i < 10; ++i) {
        hn[i] = i == 0 ? -1.0 : (i == 9 ? 1.0 : -1.0 + i * (2.0 / 9.0));
        long long b;
        memcpy(&b, &hn[i], 8);
        hk[i] = b ^ ((b >> 63) & 0x7FFFFFFFFFFFFFFFLL);
    }
    cudaMemcpy(x, hx, sizeof hx, cudaMemcpyHostToDevice);
    cudaMemcpy(node, hn, sizeof hn, cudaMemcpyHostToDevice);
    cudaMemcpy(key, hk, sizeof hk, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    unsigned epoch = 0;
    for (int rep = 0; rep < 200; ++rep, epoch += 4) {
        void* args[] = {&x, &key, &node, &flags, &epoch, &out, &err, &sink, &part};
        cudaLaunchCooperativeKernel((void*)k, sms, 256, args, 0, 0);
    }
    cudaEventRecord(a);
    const int reps = 100;
    for (int rep = 0; rep < reps; ++rep, epoch += 4) {
        void* args[] = {&x, &key, &node, &flags, &epoch, &out, &err, &sink, &part};
        cudaLaunchCooperativeKernel((void*)k, sms, 256, args, 0, 0);
    }
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    long long h[12];
    cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
    const char* names[] = {"stage x + tables", "locate+hist 2048", "flag barrier (sleep)", "flag barrier (spin)",
                           "volatile barrier", "L2 round trip"};
    for (int i = 0; i < 6; ++i) printf("%-24s %7lld cycles\n", names[i], h[i]);
    printf("launch-to-launch %.2f us per kernel; err %s\n", ms * 1000 / reps, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
