// Cost of handing data from one SM to others across a grid barrier, shaped
// like the batch-1 head kernel's layer boundary: 148 CTAs x 384 threads
// (cooperative), each CTA writes a row of W floats (float4 stores), grid
// barrier, then each CTA reads its slice of ~W/148 columns from all 148 rows
// and sums them (clock64 in thread 0 around the read phase; median over
// CTAs and launches).  Variants:
//   A  read the rows written in this launch (the kernel's pattern)
//   B  read rows written by the PREVIOUS launch (no fresh write -> read)
//   C  as A, stores with st.global.cg (L2 only)
//   D  as A, a second grid barrier before reading
//   E  as A, the reads are st/ld .release/.acquire at gpu scope (fence pattern)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mb_handoff.cu -o tools/bin/mb_handoff
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

constexpr int kT = 384;

template <int MODE>
__global__ void __launch_bounds__(kT, 1) k_handoff(float* part, float* part_old, int W, long long* out, float* sink) {
    const int P = gridDim.x, c = blockIdx.x, tid = threadIdx.x;
    // write my row
    float4* row = reinterpret_cast<float4*>(part + static_cast<size_t>(c) * W);
    for (int j = tid; j < W / 4; j += kT) {
        const float4 v = make_float4(c + j, 1.f, 2.f, 3.f);
        if (MODE == 2) __stcg(row + j, v);
        else row[j] = v;
    }
    cooperative_groups::this_grid().sync();
    if (MODE == 3) cooperative_groups::this_grid().sync();
    __syncthreads();
    const long long t0 = clock64();
    const float* src = MODE == 1 ? part_old : part;
    const int r0 = W * c / P, r1 = W * (c + 1) / P, nr = r1 - r0;
    const int warp = tid >> 5, lane = tid & 31;
    float acc = 0.f;
    if (MODE == 4) {  // v1 pattern: for each z, nr contiguous floats
        const int total = P * nr;
        float v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = tid + u * kT, z = e / (nr > 0 ? nr : 1);
            v[u] = e < total ? __ldcg(src + static_cast<size_t>(z) * W + r0 + (e - z * nr)) : 0.f;
        }
        acc = v[0] + v[1] + v[2] + v[3];
    } else if (MODE == 5) {  // consumer-contiguous block: P * 10 floats at c * P * 10
        const float4* blk = reinterpret_cast<const float4*>(src + static_cast<size_t>(c) * P * 10);
        if (tid < P * 10 / 4) {
            const float4 q = __ldcg(blk + tid);
            acc = q.x + q.y + q.z + q.w;
        }
    } else if (MODE == 6) {  // one float per thread: latency only
        acc = __ldcg(src + static_cast<size_t>((c * 7 + 3) % P) * W + tid);
    } else if (warp < nr) {
        float a[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int z = lane + 32 * u;
            a[u] = z < P ? __ldcg(src + static_cast<size_t>(z) * W + r0 + warp) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += a[u];
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
    __syncthreads();
    const long long t1 = clock64();
    if (tid == 0) out[c] = t1 - t0;
    if (acc == 123456.f) sink[c] = acc;
}

static float* g_flush;
static size_t g_flush_n = (256u << 20) / 4;

template <int MODE>
void run(const char* name, float* part, float* old, int W, long long* d_out, float* sink, int sms, bool flush) {
    std::vector<long long> all;
    for (int r = 0; r < 30; ++r) {
        if (flush) cudaMemsetAsync(g_flush, r & 0xFF, g_flush_n * 4);
        void* args[] = {&part, &old, &W, &d_out, &sink};
        cudaLaunchCooperativeKernel((void*)k_handoff<MODE>, sms, kT, args, 0, 0);
        std::vector<long long> h(sms);
        cudaMemcpy(h.data(), d_out, sms * 8, cudaMemcpyDeviceToHost);
        if (r >= 5) all.insert(all.end(), h.begin(), h.end());
    }
    std::sort(all.begin(), all.end());
    printf("%-48s flush=%d  median %6lld  p90 %6lld cycles\n", name, flush, all[all.size() / 2], all[all.size() * 9 / 10]);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaMalloc(&g_flush, g_flush_n * 4);
    const int W = 1408;
    float *part, *old, *sink;
    long long* d_out;
    cudaMalloc(&part, sizeof(float) * sms * W);
    cudaMalloc(&old, sizeof(float) * sms * W);
    cudaMemset(old, 0, sizeof(float) * sms * W);
    cudaMalloc(&sink, 4096);
    cudaMalloc(&d_out, 8 * sms);
    for (int f = 0; f < 2; ++f) {
        run<0>("A fresh rows (this launch)", part, old, W, d_out, sink, sms, f);
        run<1>("B rows of an earlier launch", part, old, W, d_out, sink, sms, f);
        run<2>("C fresh rows, st.global.cg", part, old, W, d_out, sink, sms, f);
        run<3>("D fresh rows, two grid barriers", part, old, W, d_out, sink, sms, f);
        run<4>("E v1 pattern: z-runs of nr contiguous", part, old, W, d_out, sink, sms, f);
        run<5>("F consumer-contiguous block (LDG.128)", part, old, W, d_out, sink, sms, f);
        run<6>("G one float per thread", part, old, W, d_out, sink, sms, f);
    }
    printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
