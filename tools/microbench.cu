// Microbenchmarks of the batch-1 kernel's primitives (SM cycles via clock64):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I.. tools/microbench.cu -o /tmp/mb && /tmp/mb
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2512_15742_b200/csrc/skan_device.cuh"

using namespace skan::dev;

__global__ void k(const double* x, long long* out, int* err) {
    long long t0, t1;
    double acc = 0.0;
    // 1. DDIV latency chain
    double v = x[threadIdx.x];
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 16; ++i) v = __ddiv_rn(v + 1.0, 1.0000001);
    t1 = clock64();
    acc += v;
    if (threadIdx.x == 0) out[0] = (t1 - t0) / 16;
    // 2. DFMA latency chain
    v = x[threadIdx.x];
    t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 64; ++i) v = fma(v, 1.0000001, 0.5);
    t1 = clock64();
    acc += v;
    if (threadIdx.x == 0) out[1] = (t1 - t0) / 64;
    // 3. locate_many<8>
    double xs[8], tt[8];
    bool ok[8];
    int mm[8];
    for (int q = 0; q < 8; ++q) {
        xs[q] = x[(threadIdx.x * 8 + q) & 255];
        ok[q] = true;
    }
    __syncthreads();
    t0 = clock64();
    locate_many<8>(-1.0, 1.0, 10, 2.0 / 9.0, xs, ok, mm, tt, err);
    for (int q = 0; q < 8; ++q) acc += tt[q] + mm[q];
    t1 = clock64();
    if (threadIdx.x == 0) out[2] = t1 - t0;
    // 4. 72 ballots
    __syncthreads();
    t0 = clock64();
    int w = 0;
    for (int q = 0; q < 8; ++q)
        for (int b = 0; b < 9; ++b) {
            const int c = __popc(__ballot_sync(0xFFFFFFFFu, mm[q] == b));
            if ((threadIdx.x & 31) == b) w += c;
        }
    t1 = clock64();
    acc += w;
    if (threadIdx.x == 0) out[3] = t1 - t0;
    // 5. globaltimer read cost
    t0 = clock64();
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    t1 = clock64();
    acc += static_cast<double>(g & 1);
    if (threadIdx.x == 0) out[4] = t1 - t0;
    // 6. __syncthreads
    t0 = clock64();
    __syncthreads();
    t1 = clock64();
    if (threadIdx.x == 0) out[5] = t1 - t0;
    if (acc == 12345.0) out[6] = 1;
}

int main() {
    double* x;
    long long* out;
    int* err;
    cudaMalloc(&x, 256 * sizeof(double));
    cudaMalloc(&out, 8 * sizeof(long long));
    cudaMalloc(&err, sizeof(int));
    double hx[256];
    for (int i = 0; i < 256; ++i) hx[i] = -1.4 + 2.8 * i / 255.0;
    cudaMemcpy(x, hx, sizeof hx, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 3; ++rep) {
        k<<<1, 256>>>(x, out, err);
        cudaDeviceSynchronize();
    }
    long long h[8];
    cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("ddiv latency %lld cyc, dfma latency %lld cyc, locate_many<8> %lld cyc, 72 ballots %lld cyc, "
           "globaltimer read %lld cyc, syncthreads %lld cyc (clock rate attr %d kHz) err=%s\n",
           h[0], h[1], h[2], h[3], h[4], h[5], clk, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
