// sm_100a kernels for the LUTHAM forward (SHARe-KAN compressed KAN heads).
//
//   K1  k_locate_input   knot-interval selection, bit-exact with
//                        holoquant::locate (kan.cpp:28-58)
//   K2  k_gather_fast    fused decode + gather + interpolate + accumulate,
//                        fp32 math, per-split partials (no atomics)
//       k_combine        fixed-order split reduction in double + bias sums,
//                        fused with the next layer's K1
//   K2x k_gather_exact   fp64, reference operation order, sequential i:
//                        bitwise equal to compressed_forward (lutham.cpp:793-814)
//   K5  k_unpack_indices SKAN v1 LSB-first index unpack (lutham.cpp:114-137)
//       k_pli_lookup     batched single-edge primitive (lutham.cpp:730-739)
#include <cuda_runtime.h>

#include <cstdint>

#include "skan_internal.hpp"

namespace skan {
namespace {

constexpr int kThreads = 128;  // threads per gather CTA
constexpr int kIC = 64;        // inputs whose brackets are staged per smem pass

// ---------------------------------------------------------------------------
// Knot selection.  Every double operation is an explicit round-to-nearest
// intrinsic so nvcc can neither contract lo + i*dx (kan.cpp:25) nor
// (x - lo)/dx into an FMA: the bracket and t are bitwise the reference's.

__device__ __forceinline__ double node_pos(double lo, double hi, int G, int i, double dx) {
    if (i == 0) return lo;
    if (i == G - 1) return hi;
    return __dadd_rn(lo, __dmul_rn(static_cast<double>(i), dx));  // kan.cpp:21-26
}

__device__ __forceinline__ bool locate_dev(double lo, double hi, int G, double dx, double x,
                                           int& idx, double& t) {
    bool clamped = false;
    if (x < lo) {
        x = lo;
        clamped = true;
    } else if (x > hi) {
        x = hi;
        clamped = true;
    }
    int i = static_cast<int>(floor(__ddiv_rn(__dsub_rn(x, lo), dx)));
    if (i < 0) i = 0;
    if (i > G - 2) i = G - 2;
    if (i < G - 2 && x >= node_pos(lo, hi, G, i + 1, dx)) {
        ++i;
    } else if (i > 0 && x < node_pos(lo, hi, G, i, dx)) {
        --i;
    }
    double tt;
    if (x >= node_pos(lo, hi, G, i + 1, dx)) {
        tt = 1.0;
    } else {
        tt = __ddiv_rn(__dsub_rn(x, node_pos(lo, hi, G, i, dx)), dx);
        if (tt < 0.0) tt = 0.0;
        if (tt > 1.0) tt = 1.0;
    }
    idx = i;
    t = tt;
    return clamped;
}

__global__ void k_locate_input(const double* __restrict__ x, long long n, double lo, double hi,
                               int G, double dx, int* __restrict__ bm, float* __restrict__ btf,
                               double* __restrict__ btd, int* __restrict__ err) {
    for (long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; p < n;
         p += static_cast<long long>(gridDim.x) * blockDim.x) {
        const double v = x[p];
        int m = 0;
        double t = 0.0;
        if (!isfinite(v)) {
            *err = 1;  // ValueError("spline evaluated at non-finite x"), kan.cpp:29
        } else {
            locate_dev(lo, hi, G, dx, v, m, t);
        }
        bm[p] = m;
        btf[p] = static_cast<float>(t);
        btd[p] = t;
    }
}

// ---------------------------------------------------------------------------
// Edge decode policies.  Each returns, for edge e, what the per-sample loop
// needs: the codebook row base and the gain (fast: float incl. codebook
// scale; exact: double gain + double bias, as RuntimeLayer::gain/bias).

template <int FMT>
struct Edge;

template <>
struct Edge<FMT_I8_R32> {
    const int8_t* row;
    uint32_t r;
    __device__ __forceinline__ void load(const DevLayer& L, size_t e) {
        r = __ldg(L.rec + e);
        row = L.cb8 + static_cast<size_t>(r & 0xFFFFu) * L.G;
    }
    __device__ __forceinline__ int gcode() const { return (r >> 16) & 0xFF; }
    __device__ __forceinline__ int bcode() const { return static_cast<int8_t>(r >> 24); }
};

template <>
struct Edge<FMT_I8_WIDE> {
    const int8_t* row;
    uint32_t gbv;
    __device__ __forceinline__ void load(const DevLayer& L, size_t e) {
        const uint32_t k = L.idx ? __ldg(L.idx + e) : 0u;
        gbv = __ldg(L.gb + e);
        row = L.cb8 + static_cast<size_t>(k) * L.G;
    }
    __device__ __forceinline__ int gcode() const { return gbv & 0xFF; }
    __device__ __forceinline__ int bcode() const { return static_cast<int8_t>(gbv >> 8); }
};

template <>
struct Edge<FMT_F32> {
    const float* row;
    float g, b;
    __device__ __forceinline__ void load(const DevLayer& L, size_t e) {
        const uint32_t k = L.idx ? __ldg(L.idx + e) : 0u;
        g = __ldg(L.gain + e);
        b = __ldg(L.bias + e);
        row = L.cb32 + static_cast<size_t>(k) * L.G;
    }
};

template <>
struct Edge<FMT_DENSE> {
    const float* row;
    __device__ __forceinline__ void load(const DevLayer& L, size_t e) {
        row = L.cb32 + e * static_cast<size_t>(L.G);
    }
};

// Stage brackets (index, t) of samples [sbase, sbase+SC) x inputs
// [ic, ic+n) into shared memory; padding samples get (0, 0).
template <int SC, typename T>
__device__ __forceinline__ void stage_brackets(int (*s_m)[kIC], T (*s_t)[kIC], const int* bm,
                                               const T* bt, int B, int in, int sbase, int ic,
                                               int n) {
    for (int q = threadIdx.x; q < SC * kIC; q += kThreads) {
        const int sl = q / kIC, il = q % kIC, s = sbase + sl;
        int m = 0;
        T t = T(0);
        if (s < B && il < n) {
            const size_t p = static_cast<size_t>(s) * in + ic + il;
            m = bm[p];
            t = bt[p];
        }
        s_m[sl][il] = m;
        s_t[sl][il] = t;
    }
}

// ---------------------------------------------------------------------------
// K2 fast: CTA = TJ outputs x (kThreads/TJ)*SPT samples x one i-split.
// Thread (jl, sg) owns output j and SPT consecutive samples; it streams the
// edges (i, j) of its split in ascending i (coalesced along j), decodes each
// edge once and evaluates it for its SPT samples.  Partials go to
// partial[z][s][j]; k_combine reduces them in fixed z order.
template <int FMT, int TJ, int SPT>
__global__ void __launch_bounds__(kThreads)
    k_gather_fast(DevLayer L, int B, int ichunk, const int* __restrict__ bm,
                  const float* __restrict__ btf, float* __restrict__ partial) {
    constexpr int SG = kThreads / TJ;
    constexpr int SC = SG * SPT;
    __shared__ int s_m[SC][kIC];
    __shared__ float s_t[SC][kIC];
    __shared__ float s_lut[256];
    if (FMT == FMT_I8_R32 || FMT == FMT_I8_WIDE) {
        for (int q = threadIdx.x; q < 256; q += kThreads) s_lut[q] = L.lutf[q];
    }
    const int jl = threadIdx.x % TJ, sg = threadIdx.x / TJ;
    const int j = blockIdx.x * TJ + jl;
    const int sbase = blockIdx.y * SC;
    const int z = blockIdx.z;
    const int ibeg = z * ichunk, iend = min(L.in, ibeg + ichunk);
    const bool jok = j < L.out;
    float acc[SPT];
#pragma unroll
    for (int r = 0; r < SPT; ++r) acc[r] = 0.f;

    for (int ic = ibeg; ic < iend; ic += kIC) {
        const int n = min(kIC, iend - ic);
        __syncthreads();
        stage_brackets<SC, float>(s_m, s_t, bm, btf, B, L.in, sbase, ic, n);
        __syncthreads();
        if (!jok) continue;
        for (int il = 0; il < n; ++il) {
            const size_t e = static_cast<size_t>(ic + il) * L.out + j;
            Edge<FMT> ed;
            ed.load(L, e);
            float g = 1.f;
            if constexpr (FMT == FMT_I8_R32 || FMT == FMT_I8_WIDE) g = s_lut[ed.gcode()];
            if constexpr (FMT == FMT_F32) g = ed.g;
#pragma unroll
            for (int r = 0; r < SPT; ++r) {
                const int sl = sg * SPT + r;
                const int m = s_m[sl][il];
                const float t = s_t[sl][il];
                float c0, c1;
                if constexpr (FMT == FMT_I8_R32 || FMT == FMT_I8_WIDE) {
                    c0 = static_cast<float>(__ldg(ed.row + m));
                    c1 = static_cast<float>(__ldg(ed.row + m + 1));
                } else {
                    c0 = __ldg(ed.row + m);
                    c1 = __ldg(ed.row + m + 1);
                }
                const float v = fmaf(t, c1 - c0, c0);
                if constexpr (FMT == FMT_DENSE) {
                    acc[r] += v;
                } else {
                    acc[r] = fmaf(g, v, acc[r]);
                }
            }
        }
    }
    if (jok) {
#pragma unroll
        for (int r = 0; r < SPT; ++r) {
            const int s = sbase + sg * SPT + r;
            if (s < B) partial[(static_cast<size_t>(z) * B + s) * L.out + j] = acc[r];
        }
    }
}

// Fixed-order split reduction (z ascending) in double, plus the per-output
// bias sum; then the next layer's knot selection on the finished value.
__global__ void k_combine(DevLayer L, int B, int nsplit, const float* __restrict__ partial,
                          double* __restrict__ y, int has_next, double nlo, double nhi, int nG,
                          double ndx, int* __restrict__ bm, float* __restrict__ btf,
                          double* __restrict__ btd, int* __restrict__ err) {
    const long long n = static_cast<long long>(B) * L.out;
    for (long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; p < n;
         p += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int j = static_cast<int>(p % L.out);
        double v = L.bias_sum ? L.bias_sum[j] : 0.0;
        for (int z = 0; z < nsplit; ++z) v += static_cast<double>(partial[static_cast<size_t>(z) * n + p]);
        y[p] = v;
        if (has_next) {
            int m = 0;
            double t = 0.0;
            if (!isfinite(v)) {
                *err = 1;
            } else {
                locate_dev(nlo, nhi, nG, ndx, v, m, t);
            }
            bm[p] = m;
            btf[p] = static_cast<float>(t);
            btd[p] = t;
        }
    }
}

// ---------------------------------------------------------------------------
// K2 exact: same tiling, one split (ascending i), every double op in the
// reference's order with explicit _rn intrinsics (no FMA):
//   compressed: y += (g*c0 + b)*w0 + (g*c1 + b)*t      lutham.cpp:810
//   dense:      y += c0*w0 + c1*t                      lutham.cpp:787-788
template <int FMT, int TJ, int SPT>
__global__ void __launch_bounds__(kThreads)
    k_gather_exact(DevLayer L, int B, const int* __restrict__ bm, const double* __restrict__ btd,
                   double* __restrict__ y) {
    constexpr int SG = kThreads / TJ;
    constexpr int SC = SG * SPT;
    __shared__ int s_m[SC][kIC];
    __shared__ double s_t[SC][kIC];
    const int jl = threadIdx.x % TJ, sg = threadIdx.x / TJ;
    const int j = blockIdx.x * TJ + jl;
    const int sbase = blockIdx.y * SC;
    const bool jok = j < L.out;
    double acc[SPT];
#pragma unroll
    for (int r = 0; r < SPT; ++r) acc[r] = 0.0;

    for (int ic = 0; ic < L.in; ic += kIC) {
        const int n = min(kIC, L.in - ic);
        __syncthreads();
        stage_brackets<SC, double>(s_m, s_t, bm, btd, B, L.in, sbase, ic, n);
        __syncthreads();
        if (!jok) continue;
        for (int il = 0; il < n; ++il) {
            const size_t e = static_cast<size_t>(ic + il) * L.out + j;
            Edge<FMT> ed;
            ed.load(L, e);
            double g = 0.0, b = 0.0;
            if constexpr (FMT == FMT_I8_R32 || FMT == FMT_I8_WIDE) {
                g = __ldg(L.lutd + ed.gcode());
                b = __dmul_rn(static_cast<double>(ed.bcode()), L.bs);
            }
            if constexpr (FMT == FMT_F32) {
                g = static_cast<double>(ed.g);
                b = static_cast<double>(ed.b);
            }
#pragma unroll
            for (int r = 0; r < SPT; ++r) {
                const int sl = sg * SPT + r;
                const int m = s_m[sl][il];
                const double t = s_t[sl][il];
                const double w0 = __dsub_rn(1.0, t);
                double c0, c1, term;
                if constexpr (FMT == FMT_I8_R32 || FMT == FMT_I8_WIDE) {
                    c0 = __dmul_rn(static_cast<double>(__ldg(ed.row + m)), L.cs);
                    c1 = __dmul_rn(static_cast<double>(__ldg(ed.row + m + 1)), L.cs);
                } else {
                    c0 = static_cast<double>(__ldg(ed.row + m));
                    c1 = static_cast<double>(__ldg(ed.row + m + 1));
                }
                if constexpr (FMT == FMT_DENSE) {
                    term = __dadd_rn(__dmul_rn(c0, w0), __dmul_rn(c1, t));
                } else {
                    term = __dadd_rn(__dmul_rn(__dadd_rn(__dmul_rn(g, c0), b), w0),
                                     __dmul_rn(__dadd_rn(__dmul_rn(g, c1), b), t));
                }
                acc[r] = __dadd_rn(acc[r], term);
            }
        }
    }
    if (jok) {
#pragma unroll
        for (int r = 0; r < SPT; ++r) {
            const int s = sbase + sg * SPT + r;
            if (s < B) y[static_cast<size_t>(s) * L.out + j] = acc[r];
        }
    }
}

// ---------------------------------------------------------------------------

__global__ void k_locate_raw(const double* __restrict__ x, int n, double lo, double hi, int G,
                             double dx, int* __restrict__ idx, double* __restrict__ t,
                             uint8_t* __restrict__ clamped, int* __restrict__ err) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        const double v = x[p];
        if (!isfinite(v)) {
            *err = 1;
            continue;
        }
        int m;
        double tt;
        const bool c = locate_dev(lo, hi, G, dx, v, m, tt);
        idx[p] = m;
        t[p] = tt;
        if (clamped) clamped[p] = c ? 1 : 0;
    }
}

// pli_lookup (lutham.cpp:730-739): g * (c0*(1-t) + c1*t) + b
__global__ void k_pli_lookup(const double* __restrict__ cb, int k, int G, double dx,
                             const int* __restrict__ rows, const double* __restrict__ g,
                             const double* __restrict__ b, const double* __restrict__ x, double lo,
                             double hi, int n, double* __restrict__ y, int* __restrict__ err) {
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        const int r = rows[p];
        if (r < 0 || r >= k) {
            atomicOr(err, 2);  // ShapeError("codebook row out of range")
            continue;
        }
        const double xv = x[p];
        if (!isfinite(xv)) {
            atomicOr(err, 1);
            continue;
        }
        int m;
        double t;
        locate_dev(lo, hi, G, dx, xv, m, t);
        const double* row = cb + static_cast<size_t>(r) * G;
        const double v = __dadd_rn(__dmul_rn(row[m], __dsub_rn(1.0, t)), __dmul_rn(row[m + 1], t));
        y[p] = __dadd_rn(__dmul_rn(g[p], v), b[p]);
    }
}

// K5: out[n] = bits [n*bits, (n+1)*bits) of the LSB-first stream.  The caller
// guarantees the buffer holds ceil(count*bits/8) bytes (lutham.cpp:121-123).
__global__ void k_unpack_indices(const uint8_t* __restrict__ bytes, uint64_t count, int bits,
                                 uint32_t* __restrict__ out) {
    const uint64_t nbytes = (count * static_cast<uint64_t>(bits) + 7) / 8;
    const uint64_t mask = (static_cast<uint64_t>(1) << bits) - 1;
    for (uint64_t n = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; n < count;
         n += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t bit = n * static_cast<uint64_t>(bits);
        const uint64_t byte0 = bit >> 3;
        const int shift = static_cast<int>(bit & 7);
        uint64_t acc = 0;
        const int need = (shift + bits + 7) / 8;  // <= 5
        for (int q = 0; q < need; ++q) {
            const uint64_t at = byte0 + q;
            if (at < nbytes) acc |= static_cast<uint64_t>(bytes[at]) << (8 * q);
        }
        out[n] = static_cast<uint32_t>((acc >> shift) & mask);
    }
}

int grid_for(long long n, int threads) {
    long long b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > 65535LL * 16) b = 65535LL * 16;
    return static_cast<int>(b);
}

template <int FMT, int TJ>
void dispatch_fast_spt(const DevLayer& L, const LaunchCfg& c, int B, const int* bm,
                       const float* btf, float* partial, cudaStream_t s) {
    dim3 grid(c.jt, c.st, c.nsplit);
    switch (c.spt) {
        case 1: k_gather_fast<FMT, TJ, 1><<<grid, kThreads, 0, s>>>(L, B, c.ichunk, bm, btf, partial); break;
        case 2: k_gather_fast<FMT, TJ, 2><<<grid, kThreads, 0, s>>>(L, B, c.ichunk, bm, btf, partial); break;
        case 4: k_gather_fast<FMT, TJ, 4><<<grid, kThreads, 0, s>>>(L, B, c.ichunk, bm, btf, partial); break;
        default: k_gather_fast<FMT, TJ, 8><<<grid, kThreads, 0, s>>>(L, B, c.ichunk, bm, btf, partial); break;
    }
}

template <int FMT>
void dispatch_fast_tj(const DevLayer& L, const LaunchCfg& c, int B, const int* bm,
                      const float* btf, float* partial, cudaStream_t s) {
    switch (c.tj) {
        case 32: dispatch_fast_spt<FMT, 32>(L, c, B, bm, btf, partial, s); break;
        case 64: dispatch_fast_spt<FMT, 64>(L, c, B, bm, btf, partial, s); break;
        default: dispatch_fast_spt<FMT, 128>(L, c, B, bm, btf, partial, s); break;
    }
}

template <int FMT, int TJ>
void dispatch_exact_spt(const DevLayer& L, const LaunchCfg& c, int B, const int* bm,
                        const double* btd, double* y, cudaStream_t s) {
    dim3 grid(c.jt, c.st, 1);
    switch (c.spt) {
        case 1: k_gather_exact<FMT, TJ, 1><<<grid, kThreads, 0, s>>>(L, B, bm, btd, y); break;
        case 2: k_gather_exact<FMT, TJ, 2><<<grid, kThreads, 0, s>>>(L, B, bm, btd, y); break;
        case 4: k_gather_exact<FMT, TJ, 4><<<grid, kThreads, 0, s>>>(L, B, bm, btd, y); break;
        default: k_gather_exact<FMT, TJ, 8><<<grid, kThreads, 0, s>>>(L, B, bm, btd, y); break;
    }
}

template <int FMT>
void dispatch_exact_tj(const DevLayer& L, const LaunchCfg& c, int B, const int* bm,
                       const double* btd, double* y, cudaStream_t s) {
    switch (c.tj) {
        case 32: dispatch_exact_spt<FMT, 32>(L, c, B, bm, btd, y, s); break;
        case 64: dispatch_exact_spt<FMT, 64>(L, c, B, bm, btd, y, s); break;
        default: dispatch_exact_spt<FMT, 128>(L, c, B, bm, btd, y, s); break;
    }
}

}  // namespace

// ---------------------------------------------------------------------------

LaunchCfg choose_cfg(const DevLayer& L, int B, bool exact, int num_sms) {
    LaunchCfg c{};
    c.tj = L.out <= 32 ? 32 : (L.out <= 64 ? 64 : 128);
    c.spt = B >= 8 ? 8 : (B >= 4 ? 4 : (B >= 2 ? 2 : 1));
    const int sc = (kThreads / c.tj) * c.spt;
    c.jt = (L.out + c.tj - 1) / c.tj;
    c.st = (B + sc - 1) / sc;
    if (exact) {
        c.nsplit = 1;
        c.ichunk = L.in;
        return c;
    }
    const long long base = static_cast<long long>(c.jt) * c.st;
    const long long target = 4LL * (num_sms > 0 ? num_sms : 148);
    long long ns = (target + base - 1) / base;
    const long long maxns = L.in / 16 > 1 ? L.in / 16 : 1;
    if (ns > maxns) ns = maxns;
    if (ns < 1) ns = 1;
    c.ichunk = static_cast<int>((L.in + ns - 1) / ns);
    c.nsplit = (L.in + c.ichunk - 1) / c.ichunk;
    return c;
}

void launch_locate_input(const double* x, int n_rows, int width, const DevLayer& L, int* bm,
                         float* btf, double* btd, int* err, cudaStream_t s) {
    const long long n = static_cast<long long>(n_rows) * width;
    if (n == 0) return;
    k_locate_input<<<grid_for(n, 256), 256, 0, s>>>(x, n, L.lo, L.hi, L.G, L.dx, bm, btf, btd, err);
}

void launch_gather_fast(const DevLayer& L, const LaunchCfg& c, int B, const int* bm,
                        const float* btf, float* partial, cudaStream_t s) {
    switch (L.fmt) {
        case FMT_I8_R32: dispatch_fast_tj<FMT_I8_R32>(L, c, B, bm, btf, partial, s); break;
        case FMT_I8_WIDE: dispatch_fast_tj<FMT_I8_WIDE>(L, c, B, bm, btf, partial, s); break;
        case FMT_F32: dispatch_fast_tj<FMT_F32>(L, c, B, bm, btf, partial, s); break;
        default: dispatch_fast_tj<FMT_DENSE>(L, c, B, bm, btf, partial, s); break;
    }
}

void launch_combine(const DevLayer& L, const LaunchCfg& c, int B, const float* partial,
                    double* y, const DevLayer* next, int* bm, float* btf, double* btd, int* err,
                    cudaStream_t s) {
    const long long n = static_cast<long long>(B) * L.out;
    if (n == 0) return;
    k_combine<<<grid_for(n, 256), 256, 0, s>>>(
        L, B, c.nsplit, partial, y, next != nullptr, next ? next->lo : 0.0, next ? next->hi : 0.0,
        next ? next->G : 2, next ? next->dx : 1.0, bm, btf, btd, err);
}

void launch_gather_exact(const DevLayer& L, const LaunchCfg& c, int B, const int* bm,
                         const double* btd, double* y, cudaStream_t s) {
    switch (L.fmt) {
        case FMT_I8_R32: dispatch_exact_tj<FMT_I8_R32>(L, c, B, bm, btd, y, s); break;
        case FMT_I8_WIDE: dispatch_exact_tj<FMT_I8_WIDE>(L, c, B, bm, btd, y, s); break;
        case FMT_F32: dispatch_exact_tj<FMT_F32>(L, c, B, bm, btd, y, s); break;
        default: dispatch_exact_tj<FMT_DENSE>(L, c, B, bm, btd, y, s); break;
    }
}

void launch_locate_raw(const double* x, int n, double lo, double hi, int G, int* idx, double* t,
                       uint8_t* clamped, int* err, cudaStream_t s) {
    if (n <= 0) return;
    const double dx = (hi - lo) / static_cast<double>(G - 1);
    k_locate_raw<<<grid_for(n, 256), 256, 0, s>>>(x, n, lo, hi, G, dx, idx, t, clamped, err);
}

void launch_pli_lookup(const double* cb, int k, int G, const int* rows, const double* g,
                       const double* b, const double* x, double lo, double hi, int n, double* y,
                       int* err, cudaStream_t s) {
    if (n <= 0) return;
    const double dx = (hi - lo) / static_cast<double>(G - 1);
    k_pli_lookup<<<grid_for(n, 256), 256, 0, s>>>(cb, k, G, dx, rows, g, b, x, lo, hi, n, y, err);
}

void launch_unpack_indices(const uint8_t* bytes, uint64_t count, int bits, uint32_t* out,
                           cudaStream_t s) {
    if (count == 0) return;
    k_unpack_indices<<<grid_for(static_cast<long long>(count), 256), 256, 0, s>>>(bytes, count, bits, out);
}

}  // namespace skan
