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

// The node search for inputs the cheap paths cannot settle (within q_eps of
// a knot, or pathological domains): locate()'s floor-then-correct sequence
// ends at the unique i in [0, G-2] with node(i) <= x < node(i+1) over the
// reference's own node positions (pinned by
// tests/test_oracle.py::test_bracket_is_the_node_search_the_fast_path_uses),
// so step from the estimate floor((x-lo)*inv_dx) with exact comparisons
// against node positions computed exactly as kan.cpp:21-26 does.  Returns
// (bracket, float t bits) packed in registers.  Out of line: it is rare, and
// inlining it at every call site multiplies the code a cold instruction
// cache must fetch.
static __device__ __noinline__ unsigned long long locate_search(double lo, double hi, int G, double dx,
                                                                double inv_dx, float inv_dx_f, double x) {
    int i;
    float t;
    if (!(x > lo)) {  // clamped to lo (also NaN, flagged by the caller)
        i = 0;
        t = 0.f;
    } else if (!(x < hi)) {  // clamped to hi: at the last node, t = 1
        i = G - 2;
        t = 1.f;
    } else {
        i = static_cast<int>(floor(__dmul_rn(__dsub_rn(x, lo), inv_dx)));
        i = min(max(i, 0), G - 2);
        while (i < G - 2 && x >= node_pos(lo, hi, G, i + 1, dx)) ++i;
        while (i > 0 && x < node_pos(lo, hi, G, i, dx)) --i;
        if (x >= node_pos(lo, hi, G, i + 1, dx)) {
            t = 1.f;
        } else {
            t = __double2float_rn(__dsub_rn(x, node_pos(lo, hi, G, i, dx))) * inv_dx_f;
            t = fminf(fmaxf(t, 0.f), 1.f);
        }
    }
    return static_cast<unsigned>(i) | (static_cast<unsigned long long>(__float_as_uint(t)) << 32);
}

// Clamped inputs settle without the node tables: x <= lo is clamped to lo
// (kan.cpp:31-37) -> bracket 0, t = 0 exactly; x >= hi -> bracket G-2,
// t = 1 exactly (x >= node(G-1) = hi, kan.cpp:49-50).  In-domain inputs
// whose q = (x-lo)/dx lies more than q_eps (a host-derived bound on the
// rounding of q and of the node positions) from an integer take
// floor(q) as the bracket and q - floor(q) as t.  Returns false for the
// rest (locate_search settles them).  Non-finite x raises the ValueError
// flag (kan.cpp:29).  Straight-line code: callers locate several inputs
// with full ILP, then search the rare unsettled ones.
__device__ __forceinline__ bool locate_easy(double lo, double hi, int G, double inv_dx, double q_eps, double x,
                                            int* err, int& m, float& t) {
    if (!finite_bits(x)) *err = 1;  // ValueError("spline evaluated at non-finite x"), kan.cpp:29
    const bool below = !(x > lo);   // also NaN: any bracket will do once err is set
    const bool above = !below && !(x < hi);
    const double q = __dmul_rn(__dsub_rn(x, lo), inv_dx);
    const int i = __double2int_rd(q);
    const double f = __dsub_rn(q, static_cast<double>(i));
    const bool easy = q_eps >= 0.0 && i >= 0 && i <= G - 2 && f > q_eps && f < 1.0 - q_eps;
    m = below ? 0 : (above ? G - 2 : i);
    t = below ? 0.f : (above ? 1.f : __double2float_rn(f));
    return below || above || easy;
}

// Bracket only, in fp32 (one double->float conversion, no fp64 pipe work):
// x < lo and x > hi follow exactly from float(x) < float(lo) and
// float(x) > float(hi) (rounding is monotone); in-domain inputs take
// floor(q) when q's fraction is more than qf_eps from an integer.  Returns
// false when undecided (near a knot, at the domain ends, non-finite):
// callers fall back to the exact fp64 path.
__device__ __forceinline__ bool bracket_f32(const DevLayer& L, double x, int& m) {
    // branch-free (callers unroll several inputs for ILP)
    const float xf = __double2float_rn(x);
    const bool below = xf < L.lo_f, above = xf > L.hi_f;
    const float q = (xf - L.lo_f) * L.inv_dx_f;
    const float r = q + 12582912.0f;  // 1.5 * 2^23: rounds q to the nearest integer
    const int n = __float_as_int(r) - 0x4B400000;
    const float fr = q - (r - 12582912.0f);  // exact, in [-0.5, 0.5]
    const int i = fr < 0.f ? n - 1 : n;
    const float f = fr < 0.f ? fr + 1.f : fr;
    const bool inside = i >= 0 && i <= L.G - 2 && f > L.qf_eps && f < 1.f - L.qf_eps;
    m = below ? 0 : (above ? L.G - 2 : i);
    return finite_bits(x) && L.qf_eps >= 0.f && (below || above || inside);
}

__device__ __forceinline__ void fast_locate(const DevLayer& L, double x, int* err, int& m, float& t) {
    if (!locate_easy(L.lo, L.hi, L.G, L.inv_dx, L.q_eps, x, err, m, t)) {
        const unsigned long long r = locate_search(L.lo, L.hi, L.G, L.dx, L.inv_dx, L.inv_dx_f, x);
        m = static_cast<int>(r & 0xFFFFFFFFu);
        t = __uint_as_float(static_cast<unsigned>(r >> 32));
    }
}

// Element (i, j, m) of a dense layer's grid.  Layers the tensor-core GEMM
// takes keep ONLY the GEMM's pre-tiled layout (DevLayer::wt: 128-output x
// IC-input tiles, K-major within a tile, k = m * IC + input, IC = 4 for even
// G, 8 for odd); the others keep the natural [in][out][G] layout (cb32).
__device__ __forceinline__ float dense_at(const DevLayer& L, int i, int j, int m) {
    if (L.wt) {
        const int IC = (L.G & 1) ? 8 : 4;
        const int ch = i / IC, il = i - ch * IC, jt = j >> 7, r = j & 127, k = m * IC + il;
        const size_t off = (static_cast<size_t>(jt) * L.wt_nch + ch) * (128 * IC * L.G) +
                           static_cast<size_t>((k >> 2) * 512 + (r >> 3) * 32 + (r & 7) * 4 + (k & 3));
        return __ldg(L.wt + off);
    }
    return __ldg(L.cb32 + (static_cast<size_t>(i) * L.out + j) * L.G + m);
}

// int8 codebook pair p = c0 | c1 << 8  ->  (c0, c1 - c0) as floats without
// the quarter-rate I2F pipe: 0x4B000000 | (u ^ 0x80) is the float
// 2^23 + u^0x80, so subtracting 2^23 + 128 yields the signed value; the
// difference of two such floats is exact.
__device__ __forceinline__ void pair_to_f(uint32_t p, float& c0, float& dc) {
    const uint32_t q = p ^ 0x8080u;
    const float f0 = __int_as_float(static_cast<int>(__byte_perm(q, 0x4B000000u, 0x7440)));
    const float f1 = __int_as_float(static_cast<int>(__byte_perm(q, 0x4B000000u, 0x7441)));
    c0 = f0 - 8388736.0f;
    dc = f1 - f0;
}

// 2^x on the SFU, no range fix-up (arguments here are far from the
// denormal range or produce a gain that is zeroed anyway)
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
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
// Slice c of P of [base, base+bytes) prefetched into L2 (no shared memory,
// no completion tracking).  Slices are 16-byte granular.
__device__ __forceinline__ void prefetch_l2_slice(const void* base, size_t bytes, int c, int P) {
    const size_t chunk = ((bytes + P - 1) / P + 15) & ~static_cast<size_t>(15);
    const size_t off = chunk * c;
    if (off >= bytes) return;
    const size_t n = (bytes - off < chunk ? bytes - off : chunk) & ~static_cast<size_t>(15);
    if (n == 0) return;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(static_cast<const char*>(base) + off),
                 "r"(static_cast<uint32_t>(n))
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
