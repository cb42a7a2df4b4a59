// Launch-overhead variants of a kernel shaped like the batch-1 head kernel
// (148 CTAs x 256 threads): parameter-block size, cooperative attribute,
// 205 KB dynamic shared memory, PDL; CUDA-event median of 200 launches,
// after a 256 MiB memset (flush) or back to back.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mb_launch2.cu -o tools/bin/mb_launch2
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

struct Big {
    char pad[2100];
    int* p;
};
struct Small {
    int* p;
};

template <class A>
__global__ void k_empty(A a) {
    extern __shared__ int s[];
    if (a.p && threadIdx.x == 0 && blockIdx.x == 100000) *a.p = s[0];
}

template <class A>
__global__ void k_sync(A a) {
    cooperative_groups::this_grid().sync();
    if (a.p && threadIdx.x == 0 && blockIdx.x == 100000) *a.p = 1;
}

static float* g_flush;
static size_t g_flush_n = (256u << 20) / 4;
static bool g_kernel_flush = false;

__global__ void k_fill(float* p, size_t n, float v) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) p[i] = v;
}

template <class F>
float time_it(F launch, bool flush, int reps = 200) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    std::vector<float> t;
    for (int r = 0; r < reps + 10; ++r) {
        if (flush) {
            if (g_kernel_flush) k_fill<<<148 * 8, 256, 0, s>>>(g_flush, g_flush_n, float(r));
            else cudaMemsetAsync(g_flush, r & 0xFF, g_flush_n * 4, s);
        }
        cudaEventRecord(a, s);
        launch(s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r >= 10) t.push_back(ms * 1e3f);
    }
    double sum = 0;
    for (float v : t) sum += v;
    std::sort(t.begin(), t.end());
    cudaStreamDestroy(s);
    printf("[mean %6.2f] ", sum / t.size());
    return t[t.size() / 2];
}

template <class K, class A>
void launch_ex(K k, A a, int grid, size_t smem, bool coop, cudaStream_t s) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(384);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = coop ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k, a);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaMalloc(&g_flush, g_flush_n * 4);
    const size_t big_smem = 218 * 1024;
    cudaFuncSetAttribute(k_empty<Small>, cudaFuncAttributeMaxDynamicSharedMemorySize, big_smem);
    cudaFuncSetAttribute(k_empty<Big>, cudaFuncAttributeMaxDynamicSharedMemorySize, big_smem);
    cudaFuncSetAttribute(k_sync<Big>, cudaFuncAttributeMaxDynamicSharedMemorySize, big_smem);
    for (int i = 0; i < 2000; ++i) cudaMemsetAsync(g_flush, 0, g_flush_n * 4);
    cudaDeviceSynchronize();
    Small sm{nullptr};
    Big bg{};
    bg.p = nullptr;
    for (int fl = 0; fl < 3; ++fl) {
        const bool f = fl >= 1;
        g_kernel_flush = fl == 2;
        printf("--- flush=%s\n", fl == 0 ? "none" : (fl == 1 ? "memset" : "fill kernel"));
        printf("small params, 0 smem          %7.2f us\n", time_it([&](cudaStream_t s) { launch_ex(k_empty<Small>, sm, sms, 0, false, s); }, f));
        printf("1.8 KB params, 0 smem         %7.2f us\n", time_it([&](cudaStream_t s) { launch_ex(k_empty<Big>, bg, sms, 0, false, s); }, f));
        printf("1.8 KB params, 205 KB smem    %7.2f us\n", time_it([&](cudaStream_t s) { launch_ex(k_empty<Big>, bg, sms, big_smem, false, s); }, f));
        printf("  + cooperative attr          %7.2f us\n", time_it([&](cudaStream_t s) { launch_ex(k_empty<Big>, bg, sms, big_smem, true, s); }, f));
        printf("  + cooperative + grid.sync   %7.2f us\n", time_it([&](cudaStream_t s) { launch_ex(k_sync<Big>, bg, sms, big_smem, true, s); }, f));
        printf("  two launches back to back   %7.2f us\n", time_it([&](cudaStream_t s) {
                   launch_ex(k_empty<Big>, bg, sms, big_smem, false, s);
                   launch_ex(k_empty<Big>, bg, sms, big_smem, false, s);
               }, f));
        // the same kernel as a one-node CUDA graph (instantiated once)
        {
            cudaStream_t cs;
            cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
            cudaGraph_t g;
            cudaGraphExec_t ge;
            cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
            launch_ex(k_empty<Big>, bg, sms, big_smem, false, cs);
            cudaStreamEndCapture(cs, &g);
            cudaGraphInstantiate(&ge, g, 0);
            cudaGraphUpload(ge, cs);
            printf("  graph of 1 kernel (205 KB) %7.2f us\n", time_it([&](cudaStream_t s) { cudaGraphLaunch(ge, s); }, f));
            cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
            launch_ex(k_empty<Big>, bg, sms, big_smem, false, cs);
            launch_ex(k_empty<Big>, bg, sms, big_smem, false, cs);
            cudaStreamEndCapture(cs, &g);
            cudaGraphInstantiate(&ge, g, 0);
            cudaGraphUpload(ge, cs);
            printf("  graph of 2 kernels          %7.2f us\n", time_it([&](cudaStream_t s) { cudaGraphLaunch(ge, s); }, f));
        }
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
