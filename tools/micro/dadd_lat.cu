// Dependent-add latency of FP64 (DADD) vs FP32 (FADD) on one thread, clock64.
#include <cstdio>
__global__ void k(double* o, float* of, long long* t, int n, double x, float xf) {
    double a = x; float b = xf;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { a = __dadd_rn(a, x); a = __dadd_rn(a, -x); }
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) { b = __fadd_rn(b, xf); b = __fadd_rn(b, -xf); }
    long long t2 = clock64();
    o[0] = a; of[0] = b; t[0] = t1 - t0; t[1] = t2 - t1;
}
int main() {
    double* o; float* of; long long* t; cudaMallocManaged(&o, 8); cudaMallocManaged(&of, 4); cudaMallocManaged(&t, 16);
    const int n = 1 << 16;
    k<<<1, 1>>>(o, of, t, n, 1.0, 1.0f); cudaDeviceSynchronize();
    k<<<1, 1>>>(o, of, t, n, 1.0, 1.0f); cudaDeviceSynchronize();
    printf("DADD dependent: %.2f clk/add   FADD: %.2f clk/add\n", double(t[0]) / (2.0 * n), double(t[1]) / (2.0 * n));
}
