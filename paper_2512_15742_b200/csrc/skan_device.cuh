// Device helpers shared by the sm_100a kernel translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "skan_internal.hpp"

namespace skan {
namespace dev {

__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------------------
// Knot selection.  Every double operation is an explicit round-to-nearest
// intrinsic so nvcc can neither contract lo + i*dx (kan.cpp:25) nor
// (x - lo)/dx into an FMA: the bracket and t are bitwise the reference's.

__device__ __forceinline__ double node_pos(double lo, double hi, int G, int i, double dx) {
    if (i == 0) return lo;
    if (i == G - 1) return hi;
    return __dadd_rn(lo, __dmul_rn(static_cast<double>(i), dx));  // kan.cpp:21-26
}

// kan.cpp:28-58
__device__ __forceinline__ bool locate_dev(double lo, double hi, int G, double dx, double x, int& idx,
                                           double& t) {
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

// ---------------------------------------------------------------------------
// Division-free knot selection for the fast path.  locate()'s floor-then-
// correct sequence always ends at the unique i in [0, G-2] with
// node(i) <= x < node(i+1) over the reference's own node positions
// (pinned by tests/test_oracle.py::test_bracket_is_the_node_search_the_fast_path_uses),
// so the bracket index is found with an fp32 estimate and exact comparisons
// against precomputed node keys -- integer compares, no FP64 division (the
// FP64 pipe is narrow: one exact locate costs ~2 dependent 160-cycle
// divisions).  t is then computed as float(x - node(i)) * (1/dx) in fp32,
// within an ulp of float(locate().t) -- inside the fast path's tolerance;
// the exact path keeps locate_dev.

// Order-preserving int64 key of a non-NaN double; +0 and -0 share key 0
// (they compare equal as doubles).
__device__ __forceinline__ long long dkey(double d) {
    long long b = __double_as_longlong(d);
    if (b == static_cast<long long>(0x8000000000000000ULL)) b = 0;
    return b ^ ((b >> 63) & 0x7FFFFFFFFFFFFFFFLL);
}

__device__ __forceinline__ bool finite_bits(double d) {
    return ((__double_as_longlong(d) >> 52) & 0x7FF) != 0x7FF;
}

// key[G] node keys and node[G] node positions (global or shared memory).
// Branch-free (no per-lane loops, which diverge and serialise the warp):
// the estimate floor(float((x-lo)*inv_dx)) is within one bracket of the
// answer, one select-based step corrects it, and a loop runs only in the
// (uniform-checked) case that it did not.
__device__ __forceinline__ void fast_locate_tab(const long long* key, const double* node, int G, double lo,
                                                double inv_dx, float inv_dx_f, double x, int* err, int& m,
                                                float& t, double q_eps = -1.0) {
    if (!finite_bits(x)) {
        *err = 1;  // ValueError("spline evaluated at non-finite x"), kan.cpp:29
        x = node[0];
    }
    if (q_eps >= 0.0) {
        // common path: q = (x-lo)*inv_dx is within q_eps (host-derived bound
        // on the rounding of q and of the node positions) of the exact
        // position, so away from integers floor(q) IS the bracket and
        // q - floor(q) is t to far below a float ulp; no table loads.
        const double q = __dmul_rn(__dsub_rn(x, lo), inv_dx);
        const int i = __double2int_rd(q);
        const double f = __dsub_rn(q, static_cast<double>(i));
        if (i >= 0 && i <= G - 2 && f > q_eps && f < 1.0 - q_eps) {
            m = i;
            t = __double2float_rn(f);
            return;
        }
    }
    long long kx = dkey(x);
    const long long klo = key[0], khi = key[G - 1];
    const bool below = kx < klo, above = kx > khi;
    kx = below ? klo : (above ? khi : kx);
    x = below ? node[0] : (above ? node[G - 1] : x);
    int i = __float2int_rd(__double2float_rn(__dsub_rn(x, lo) * inv_dx));
    i = min(max(i, 0), G - 2);
    const bool up = i < G - 2 && kx >= key[i + 1];
    const bool down = !up && i > 0 && kx < key[i];
    i += up ? 1 : (down ? -1 : 0);
    const bool ok = (i == G - 2 || kx < key[i + 1]) && (i == 0 || kx >= key[i]);
    if (__builtin_expect(!ok, 0)) {  // estimate was off by more than one bracket
        while (i < G - 2 && kx >= key[i + 1]) ++i;
        while (i > 0 && kx < key[i]) --i;
    }
    const bool full = kx >= key[i + 1];  // at or past the upper node: t = 1 exactly
    float tt = __double2float_rn(x - node[i]) * inv_dx_f;
    tt = fminf(fmaxf(tt, 0.f), 1.f);
    m = i;
    t = full ? 1.f : tt;
}

__device__ __forceinline__ void fast_locate(const DevLayer& L, double x, int* err, int& m, float& t) {
    fast_locate_tab(L.nkey, L.node, L.G, L.lo, L.inv_dx, L.inv_dx_f, x, err, m, t, L.q_eps);
}

// int8 codebook pair p = c0 | c1 << 8  ->  (c0, c1 - c0) as floats without
// the quarter-rate I2F pipe: 0x4B000000 | (u ^ 0x80) is the float
// 2^23 + u^0x80, so subtracting 2^23 + 128 yields the signed value; the
// difference of two such floats is exact.
__device__ __forceinline__ void pair_to_f(uint32_t p, float& c0, float& dc) {
    const float f0 = __int_as_float(static_cast<int>((p & 0xFFu) ^ 0x4B000080u));
    const float f1 = __int_as_float(static_cast<int>(((p >> 8) & 0xFFu) ^ 0x4B000080u));
    c0 = f0 - 8388736.0f;
    dc = f1 - f0;
}

// locate() for N independent inputs in lock step: the same operations as
// locate_dev, restructured so the N division chains interleave (ILP)
// instead of running back to back.  Bitwise identical results.
template <int N>
__device__ __forceinline__ void locate_many(double lo, double hi, int G, double dx, const double* xin,
                                            const bool* valid, int* idx, double* t, int* err) {
    double x[N], q[N];
    int i[N];
#pragma unroll
    for (int n = 0; n < N; ++n) {
        double v = valid[n] ? xin[n] : lo;
        if (valid[n] && !isfinite(v)) {
            *err = 1;
            v = lo;
        }
        v = v < lo ? lo : (v > hi ? hi : v);
        x[n] = v;
        q[n] = __ddiv_rn(__dsub_rn(v, lo), dx);
    }
#pragma unroll
    for (int n = 0; n < N; ++n) {
        int k = static_cast<int>(floor(q[n]));
        k = k < 0 ? 0 : (k > G - 2 ? G - 2 : k);
        const double up = node_pos(lo, hi, G, k + 1, dx), here = node_pos(lo, hi, G, k, dx);
        if (k < G - 2 && x[n] >= up) {
            ++k;
        } else if (k > 0 && x[n] < here) {
            --k;
        }
        i[n] = k;
    }
#pragma unroll
    for (int n = 0; n < N; ++n) q[n] = __ddiv_rn(__dsub_rn(x[n], node_pos(lo, hi, G, i[n], dx)), dx);
#pragma unroll
    for (int n = 0; n < N; ++n) {
        double tt = q[n];
        if (x[n] >= node_pos(lo, hi, G, i[n] + 1, dx)) {
            tt = 1.0;
        } else {
            tt = tt < 0.0 ? 0.0 : (tt > 1.0 ? 1.0 : tt);
        }
        idx[n] = i[n];
        t[n] = tt;
    }
}

// locate with the non-finite check (ValueError, kan.cpp:29) folded into err
__device__ __forceinline__ void bracket_of(double lo, double hi, int G, double dx, double v, int* err, int& m,
                                           double& t) {
    m = 0;
    t = 0.0;
    if (!isfinite(v)) {
        *err = 1;
    } else {
        locate_dev(lo, hi, G, dx, v, m, t);
    }
}

__device__ __forceinline__ float i8lo(uint32_t p) { return static_cast<float>(static_cast<int8_t>(p & 0xFFu)); }
__device__ __forceinline__ float i8hi(uint32_t p) {
    return static_cast<float>(static_cast<int8_t>((p >> 8) & 0xFFu));
}

// TMA 1-D bulk copy global -> shared, completing on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}

}  // namespace dev
}  // namespace skan
