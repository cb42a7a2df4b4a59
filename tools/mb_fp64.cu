// Dependent-chain latency (cycles per op, one warp) and throughput (ops per
// cycle per SM, 32 warps) of the arithmetic the batch-1 path leans on:
// DADD, DMUL, F2I.F64.FLOOR, double->float, double shuffles, MUFU.EX2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mb_fp64.cu -o tools/bin/mb_fp64
#include <cuda_runtime.h>

#include <cstdio>

constexpr int N = 4096;

template <int OP>
__global__ void k_lat(double* out, double a, long long* cyc) {
    double v = a + threadIdx.x * 1e-9;
    float f = static_cast<float>(v);
    int iv = 0;
    const long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) {
        if constexpr (OP == 0) v = v + 1.0000001;
        if constexpr (OP == 1) v = v * 1.0000001;
        if constexpr (OP == 2) { iv = __double2int_rd(v + iv); }
        if constexpr (OP == 3) { f = __double2float_rn(v + f); }
        if constexpr (OP == 4) v = __shfl_xor_sync(0xFFFFFFFFu, v, 1) + 1.0;
        if constexpr (OP == 5) f = exp2f(f * 0.999f);
        if constexpr (OP == 6) f = f * 1.0001f + 0.5f;
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[OP] = t1 - t0;
    if (v + f + iv == 123.0) out[threadIdx.x] = v;
}

template <int OP>
__global__ void k_tput(double* out, double a, long long* cyc) {
    double v0 = a + threadIdx.x, v1 = v0 + 1, v2 = v0 + 2, v3 = v0 + 3, v4 = v0 + 4, v5 = v0 + 5, v6 = v0 + 6,
           v7 = v0 + 7;
    __syncthreads();
    const long long t0 = clock64();
#pragma unroll 4
    for (int i = 0; i < N / 8; ++i) {
        if constexpr (OP == 0) {
            v0 += 1.0000001; v1 += 1.0000001; v2 += 1.0000001; v3 += 1.0000001;
            v4 += 1.0000001; v5 += 1.0000001; v6 += 1.0000001; v7 += 1.0000001;
        } else {
            v0 *= 1.0000001; v1 *= 1.0000001; v2 *= 1.0000001; v3 *= 1.0000001;
            v4 *= 1.0000001; v5 *= 1.0000001; v6 *= 1.0000001; v7 *= 1.0000001;
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[8 + OP] = t1 - t0;
    if (v0 + v1 + v2 + v3 + v4 + v5 + v6 + v7 == 123.0) out[threadIdx.x] = v0;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 1 << 16);
    cudaMallocManaged(&cyc, 16 * sizeof(long long));
    const char* names[] = {"DADD", "DMUL", "F2I.F64.FLOOR(+DADD)", "F2F.F32.F64(+DADD)", "SHFL.64+DADD", "MUFU.EX2+FMUL",
                           "FFMA"};
    for (int rep = 0; rep < 2; ++rep) {
        k_lat<0><<<1, 32>>>(out, 1.0, cyc);
        k_lat<1><<<1, 32>>>(out, 1.0, cyc);
        k_lat<2><<<1, 32>>>(out, 1.0, cyc);
        k_lat<3><<<1, 32>>>(out, 1.0, cyc);
        k_lat<4><<<1, 32>>>(out, 1.0, cyc);
        k_lat<5><<<1, 32>>>(out, 1.0, cyc);
        k_lat<6><<<1, 32>>>(out, 1.0, cyc);
        k_tput<0><<<1, 1024>>>(out, 1.0, cyc);
        k_tput<1><<<1, 1024>>>(out, 1.0, cyc);
        cudaDeviceSynchronize();
    }
    for (int i = 0; i < 7; ++i) printf("latency %-22s %6.1f cycles/op\n", names[i], double(cyc[i]) / N);
    printf("throughput DADD %6.1f lane-ops/cycle/SM\n", 1024.0 * N / double(cyc[8]));
    printf("throughput DMUL %6.1f lane-ops/cycle/SM\n", 1024.0 * N / double(cyc[9]));
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
