// Microbenchmarks of the batch-1 kernel's primitives, CTA-wide (256 threads,
// clock64 between __syncthreads), one CTA per SM on all SMs:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Iinclude tools/microbench.cu -o tools/microbench.bin
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2512_15742_b200/csrc/skan_device.cuh"

using namespace skan::dev;

__device__ long long tick() {
    __syncthreads();
    return clock64();
}

__global__ void k(const double* x, const long long* gkey, const double* gnode, unsigned* bar, long long* out,
                  int* err, float* sink) {
    __shared__ long long skey[10];
    __shared__ double snode[10];
    __shared__ int cnt[32];
    __shared__ __align__(8) uint64_t mbar;
    long long t[16];
    int n = 0;
    t[n++] = tick();
    // 0: mbarrier init + fence
    if (threadIdx.x == 0) mbar_init(&mbar, 1);
    t[n++] = tick();
    // 1: node tables to smem (L2 warm)
    if (threadIdx.x < 10) {
        skey[threadIdx.x] = gkey[threadIdx.x];
        snode[threadIdx.x] = gnode[threadIdx.x];
    }
    t[n++] = tick();
    // 2: 8 x loads per thread (L2 warm)
    double xv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) xv[q] = x[threadIdx.x * 8 + q];
    float acc = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) acc += static_cast<float>(xv[q]);
    t[n++] = tick();
    // 3: 8 fast_locate_tab per thread from smem tables
    int mm[8];
    float tt[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) fast_locate_tab(skey, snode, 10, -1.0f, 4.5f, xv[q], err, mm[q], tt[q]);
#pragma unroll
    for (int q = 0; q < 8; ++q) acc += tt[q] + mm[q];
    t[n++] = tick();
    // 4: 8 F2F.F32.F64 + 8 DADD only
#pragma unroll
    for (int q = 0; q < 8; ++q) acc += __double2float_rn(xv[q] - 0.25);
    t[n++] = tick();
    // 5: ballot histogram (8 x 9)
    int w = 0;
    for (int q = 0; q < 8; ++q)
        for (int b = 0; b < 9; ++b) {
            const int c = __popc(__ballot_sync(0xFFFFFFFFu, mm[q] == b));
            if ((threadIdx.x & 31) == b) w += c;
        }
    if (threadIdx.x < 32) cnt[threadIdx.x] = w;
    t[n++] = tick();
    // 6: grid barrier (all CTAs)
    if (threadIdx.x == 0) {
        volatile unsigned* vgen = bar + 1;
        const unsigned gen = *vgen;
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            bar[0] = 0;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*vgen == gen) __nanosleep(16);
        }
        __threadfence();
    }
    t[n++] = tick();
    // 7: second barrier
    if (threadIdx.x == 0) {
        volatile unsigned* vgen = bar + 1;
        const unsigned gen = *vgen;
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            bar[0] = 0;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*vgen == gen) __nanosleep(16);
        }
        __threadfence();
    }
    t[n++] = tick();
    // 8: 16 DADD chain per thread
    double d = xv[0];
#pragma unroll
    for (int q = 0; q < 16; ++q) d += xv[q & 7];
    acc += static_cast<float>(d);
    t[n++] = tick();
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc + cnt[threadIdx.x & 31];
    if (threadIdx.x == 0 && blockIdx.x == 0)
        for (int i = 1; i < n; ++i) out[i - 1] = t[i] - t[i - 1];
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* x;
    long long* key;
    double* node;
    unsigned* bar;
    long long* out;
    int* err;
    float* sink;
    cudaMalloc(&x, 2048 * sizeof(double));
    cudaMalloc(&key, 10 * sizeof(long long));
    cudaMalloc(&node, 10 * sizeof(double));
    cudaMalloc(&bar, 64);
    cudaMalloc(&out, 16 * sizeof(long long));
    cudaMalloc(&err, sizeof(int));
    cudaMalloc(&sink, sms * 256 * sizeof(float));
    cudaMemset(bar, 0, 64);
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
    for (int rep = 0; rep < 20; ++rep) k<<<sms, 256>>>(x, key, node, bar, out, err, sink);
    cudaDeviceSynchronize();
    long long h[16];
    cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
    const char* names[] = {"mbar_init+fence", "node tables->smem", "8 x loads", "8 fast_locate",
                           "8 F2F+DADD", "ballot hist 8x9", "grid barrier", "grid barrier 2", "16 DADD chain"};
    for (int i = 0; i < 9; ++i) printf("%-20s %8lld cycles\n", names[i], h[i]);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
