// Cost of the batch-1 kernel's small phases measured in isolation, inside a
// 148 x 384 cooperative launch like k_head_b1 (clock64 in CTA 0 between
// __syncthreads; median of 50 launches), with a small and a 218 KB dynamic
// shared-memory footprint:
//   A one L2 round trip (ld.global.cg of data written by another SM)
//   B the final reduction of 148 x 20 partials (12 warps, 2 outputs each)
//   C a cooperative-groups grid barrier
//   D 8 independent fp64 locates per thread
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mb_phase.cu -o tools/bin/mb_phase
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

constexpr int kT = 384;

__device__ __forceinline__ long long tick() {
    __syncthreads();
    return clock64();
}

__global__ void __launch_bounds__(kT, 1) k_phase(float* part, double* y, long long* out, const double* xs) {
    extern __shared__ unsigned char smem[];
    const int P = gridDim.x;
    // every CTA writes 20 partials
    if (threadIdx.x < 20) part[blockIdx.x * 20 + threadIdx.x] = 1.0f + blockIdx.x;
    __threadfence();
    long long t[8];
    int n = 0;
    t[n++] = tick();
    cooperative_groups::this_grid().sync();  // C
    t[n++] = tick();
    // A: one dependent L2 round trip per warp (lane 0)
    float a = 0.f;
    if ((threadIdx.x & 31) == 0) a = __ldcg(part + ((blockIdx.x + 37) % P) * 20);
    if (a == -1.f) smem[0] = 1;
    t[n++] = tick();
    // B: final reduction
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int j = warp; j < 20; j += kT / 32) {
        float buf[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int z = lane + 32 * u;
            buf[u] = z < P ? __ldcg(part + z * 20 + j) : 0.f;
        }
        double v = 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) v += static_cast<double>(buf[u]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
        if (lane == 0) y[blockIdx.x * 20 + j] = v;
    }
    t[n++] = tick();
    // D: 8 fp64 "locates" per thread
    double acc = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const double x = xs[(threadIdx.x + q * kT) & 2047];
        const double qq = (x + 1.0) * 4.5;
        const int i = __double2int_rd(qq);
        const double f = qq - i;
        acc += static_cast<double>(__double2float_rn(f)) + i;
    }
    if (acc == -1.0) smem[1] = 1;
    t[n++] = tick();
    if (blockIdx.x == 0 && threadIdx.x == 0)
        for (int k = 1; k < n; ++k) out[k - 1] = t[k] - t[k - 1];
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* part;
    double *y, *xs;
    long long* out;
    cudaMalloc(&part, 256 * 20 * 4);
    cudaMalloc(&y, 256 * 20 * 8);
    cudaMalloc(&xs, 2048 * 8);
    cudaMemset(xs, 0, 2048 * 8);
    cudaMallocManaged(&out, 16 * 8);
    float* flush;
    cudaMalloc(&flush, 256u << 20);
    cudaFuncSetAttribute(k_phase, cudaFuncAttributeMaxDynamicSharedMemorySize, 218 * 1024);
    const char* names[] = {"C grid.sync", "A L2 round trip", "B final reduce", "D 8 fp64 locates"};
    for (size_t smem : {size_t(0), size_t(218 * 1024)}) {
        std::vector<std::vector<long long>> v(4);
        for (int r = 0; r < 60; ++r) {
            cudaMemsetAsync(flush, r, 256u << 20);
            void* args[] = {&part, &y, &out, &xs};
            cudaLaunchCooperativeKernel((void*)k_phase, sms, kT, args, smem, 0);
            cudaDeviceSynchronize();
            if (r >= 10)
                for (int k = 0; k < 4; ++k) v[k].push_back(out[k]);
        }
        printf("dynamic smem %zu KB\n", smem / 1024);
        for (int k = 0; k < 4; ++k) {
            std::sort(v[k].begin(), v[k].end());
            printf("  %-18s median %6lld cycles\n", names[k], v[k][v[k].size() / 2]);
        }
    }
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
