// Fixed costs that bound the batch-1 latency path, measured with CUDA events
// (median of 200 launches, each preceded by a 256 MiB L2-flushing memset or
// not), one CTA of 256 threads per SM:
//   A  empty kernel: plain / cooperative / 200 KB dynamic shared memory
//   B  straight-line code of N instructions executed once per warp (cold
//      instruction cache): how much does code size cost per launch?
//   C  a chain of R dependent L2 round trips in one warp (latency per hop)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mb_launch.cu -o /tmp/mb_launch
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

__global__ void k_empty(int* p) {
    if (p && threadIdx.x == 0 && blockIdx.x == 100000) *p = 1;
}

__global__ void k_empty_smem(int* p) {
    extern __shared__ int s[];
    if (p && threadIdx.x == 0 && blockIdx.x == 100000) *p = s[0];
}

__global__ void k_coop(int* p) {
    cooperative_groups::this_grid().sync();
    if (p && threadIdx.x == 0 && blockIdx.x == 100000) *p = 1;
}

template <int N>
__global__ void k_code(float* out, float a) {
    float v0 = a + threadIdx.x, v1 = v0 * 1.5f, v2 = v0 * 0.5f, v3 = v0 + 2.f;
#pragma unroll
    for (int i = 0; i < N / 4; ++i) {
        v0 = v0 * 1.000001f + 0.5f;
        v1 = v1 * 0.999999f + 0.25f;
        v2 = v2 * 1.000002f - 0.5f;
        v3 = v3 * 0.999998f - 0.25f;
    }
    if (v0 + v1 + v2 + v3 == 12345.f) out[threadIdx.x] = v0;
}

__global__ void k_chain(const unsigned* next, int hops, unsigned* out) {
    if (threadIdx.x != 0) return;
    unsigned p = blockIdx.x * 32;
    for (int h = 0; h < hops; ++h) p = __ldcg(next + p);
    if (p == 0xFFFFFFFFu) out[blockIdx.x] = p;
}

static float* g_flush;
static size_t g_flush_n = (256u << 20) / 4;

template <class F>
float time_it(F launch, bool flush, int reps = 200) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    std::vector<float> t;
    for (int r = 0; r < reps + 10; ++r) {
        if (flush) cudaMemsetAsync(g_flush, r & 0xFF, g_flush_n * 4);
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r >= 10) t.push_back(ms * 1e3f);
    }
    std::sort(t.begin(), t.end());
    return t[t.size() / 2];
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaMalloc(&g_flush, g_flush_n * 4);
    float* out;
    cudaMalloc(&out, 4096);
    unsigned* next;
    const int n_next = 1 << 22;
    cudaMalloc(&next, n_next * 4);
    {
        std::vector<unsigned> h(n_next);
        unsigned s = 12345;
        for (int i = 0; i < n_next; ++i) {
            s = s * 1664525u + 1013904223u;
            h[i] = (s >> 4) % n_next;
        }
        cudaMemcpy(next, h.data(), n_next * 4, cudaMemcpyHostToDevice);
    }
    const int smem = 200 * 1024;
    cudaFuncSetAttribute(k_empty_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    // warm the clocks
    for (int i = 0; i < 2000; ++i) cudaMemsetAsync(g_flush, 0, g_flush_n * 4);
    cudaDeviceSynchronize();
    for (int fl = 0; fl < 2; ++fl) {
        const bool f = fl == 1;
        printf("--- flush=%d\n", fl);
        printf("A empty plain          %7.2f us\n", time_it([&] { k_empty<<<sms, 256>>>(nullptr); }, f));
        printf("A empty 200KB smem     %7.2f us\n", time_it([&] { k_empty_smem<<<sms, 256, smem>>>(nullptr); }, f));
        printf("A coop + 1 grid.sync   %7.2f us\n", time_it([&] {
                   void* args[] = {nullptr};
                   int* np = nullptr;
                   args[0] = &np;
                   cudaLaunchCooperativeKernel((void*)k_coop, sms, 256, args, 0, 0);
               }, f));
        printf("B code    256 instr    %7.2f us\n", time_it([&] { k_code<256><<<sms, 256>>>(out, 1.f); }, f));
        printf("B code   1024 instr    %7.2f us\n", time_it([&] { k_code<1024><<<sms, 256>>>(out, 1.f); }, f));
        printf("B code   4096 instr    %7.2f us\n", time_it([&] { k_code<4096><<<sms, 256>>>(out, 1.f); }, f));
        printf("B code  16384 instr    %7.2f us\n", time_it([&] { k_code<16384><<<sms, 256>>>(out, 1.f); }, f));
        for (int hops : {1, 8, 32})
            printf("C chain %2d L2/DRAM hops %7.2f us\n", hops,
                   time_it([&] { k_chain<<<sms, 32>>>(next, hops, (unsigned*)out); }, f));
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
