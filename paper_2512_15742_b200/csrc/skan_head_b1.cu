// Batch-1 latency path: the whole head in ONE persistent, cooperative kernel.
//
// At batch 1 the head is a chain of dependent memory round trips and every
// CTA executes each phase's code once from a cold instruction cache, so the
// design minimises phases, round trips and code, not bytes:
//   * one CTA per SM (148), 384 threads;
//   * layer 0 (the wide one, e.g. 2048 -> 1408): every edge of input row i
//     uses the same bracket m_i, so rows are bucketed by bracket and each CTA
//     serves a share of ONE bucket, with that bucket's codebook pair plane
//     P_m[k] = (c[k][m], c[k][m+1]) (K x 2 bytes) and its rows' records
//     staged in shared memory by TMA bulk copies.  x itself arrives by one
//     bulk copy.  Thread t owns outputs 4t..4t+3 and walks the CTA's rows in
//     ascending order: no cross-warp reduction, one float4 partial per thread;
//   * the int8 gain is computed (exp2 of the log code, code 127 -> 0) rather
//     than looked up, keeping the LSU free for the random plane gathers;
//   * later layers are split by input rows across CTAs; each CTA reduces
//     exactly the previous-layer outputs it consumes (fixed order, double),
//     adds their bias sums and locates them; its records were bulk-copied
//     at kernel start;
//   * one grid barrier per layer boundary; the last layer ends with an
//     arrival counter instead: the last CTA to arrive reduces y.
// All summation orders are fixed functions of the launch shape and the
// bracket histogram: results are bitwise reproducible run to run.
// int8 tables with <= 65536-row codebooks (FMT_I8_R32); other heads use the
// multi-kernel path.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "skan_device.cuh"
#include "skan_internal.hpp"

namespace skan {
namespace {

using namespace dev;

constexpr int kT = 384;  // threads per CTA: 4 outputs each covers out <= 1536
constexpr int kW = kT / 32;
constexpr int kMaxPer = 8;       // layer-0 inputs per thread (in <= kT * kMaxPer)
constexpr int kMaxRows = 128;    // layer-0 rows per CTA
constexpr size_t kPrefetchBytes = 16 * 1024;  // row-split records prefetched at kernel start

// Optional phase timeline (profiling hook): thread 0 of each CTA stamps
// %globaltimer (ns) at fixed phase ids.
__device__ __forceinline__ void stamp(const HeadB1Args& h, int phase) {
    if (h.timeline && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        h.timeline[blockIdx.x * 16 + phase] = t;
        h.timeline[(gridDim.x + blockIdx.x) * 16 + phase] = clock64();
    }
}

// SM clock at kernel start / end (slots 14, 15): timeline ns vs cycles
__device__ __forceinline__ void stamp_clock(const HeadB1Args& h, int slot) {
    if (h.timeline && threadIdx.x == 0) h.timeline[blockIdx.x * 16 + slot] = clock64();
}

__device__ __forceinline__ void grid_sync() { cooperative_groups::this_grid().sync(); }

// Grid barrier on a monotonic counter (the launch is cooperative, so all
// CTAs are co-resident): one release add and an acquire poll by thread 0,
// block barriers either side.  `target` = the counter's value at launch + P.
__device__ __forceinline__ void grid_barrier(unsigned* ctr, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
        } while (static_cast<int>(v - target) < 0);
    }
    __syncthreads();
}

// Last-arriver test on a monotonic counter: acq_rel add (the CTA's writes,
// ordered before by the block barrier, are released; the last arriver
// acquires everyone else's).
__device__ __forceinline__ unsigned arrive_acq_rel(unsigned* ctr) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
    return old;
}

// float(gain(code) * codebook_scale) for the fast path (see DevLayer::g_base);
// the record's gain code is byte 2
__device__ __forceinline__ float gain_of_rec(const DevLayer& L, uint32_t r) {
    // signed value of the int8 code, exact, without the quarter-rate I2F
    const uint32_t u = __byte_perm(r, 0u, 0x4442) ^ 0x4B000080u;
    const float c = __int_as_float(static_cast<int>(u)) - 8388736.0f;
    const float g = ex2_approx(fmaf(c, L.g_step, L.g_base));
    return u == (0x4B000080u ^ 127u) ? 0.f : g;
}

__device__ __forceinline__ void rows_of(const DevLayer& L, int c, int P, int& r0, int& r1) {
    r0 = L.in * c / P;  // 32-bit: in <= 16384, c <= P <= 256
    r1 = L.in * (c + 1) / P;
}

// Reduce rows [r0, r1) of the previous layer's per-CTA partials
// prev[z*width + i] (z < nz): the nz x n block is loaded coalesced into
// s_red, then C lanes per row sum it in ascending z per lane and a fixed
// butterfly combines them (fixed order: bitwise reproducible); + the
// previous layer's bias sums of these rows (bias_rows[q]); then locate with
// layer L's grid.
__device__ void reduce_rows(const float* prev, int width, int nz, const double* bias_rows, const DevLayer& L,
                            int r0, int r1, int* s_m, float* s_t, float* s_red, int* err) {
    const int n = r1 - r0;
    const int total = nz * n;
#pragma unroll 1
    for (int e0 = threadIdx.x; e0 < total; e0 += 4 * kT) {
        float v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = e0 + u * kT, z = e / n;
            v[u] = e < total ? __ldcg(prev + static_cast<size_t>(z) * width + r0 + (e - z * n)) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (e0 + u * kT < total) s_red[e0 + u * kT] = v[u];
    }
    __syncthreads();
    int C = 1;
    while (C < 32 && (C * 2) * n <= kT) C <<= 1;
    const int c = threadIdx.x & (C - 1), groups = kT / C;
    for (int pass = 0; pass < n; pass += groups) {
        const int q = pass + threadIdx.x / C;
        const int i = min(q, n - 1);
        double v = 0.0;
#pragma unroll 4
        for (int z = c; z < nz; z += C) v += static_cast<double>(s_red[z * n + i]);
        for (int o = C >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
        if (c == 0 && q < n) {
            int m;
            float t;
            fast_locate(L, v + (bias_rows ? bias_rows[q] : 0.0), err, m, t);
            s_m[q] = m;
            s_t[q] = t;
        }
    }
}

// Row-split layer: this CTA's rows [r0, r1) (brackets in s_m/s_t), all
// outputs.  Warp w takes rows w, w+kW, ...; lane l outputs l, l+32, ...;
// records from shared memory when prefetched (s_rec != nullptr); per-warp
// accumulators in shared memory; fixed-order sum over warps.
__device__ void rowsplit_layer(const DevLayer& L, int r0, int r1, const int* s_m, const float* s_t,
                               const uint32_t* s_rec, float* s_acc, float* part_out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int q = threadIdx.x; q < kW * L.out; q += kT) s_acc[q] = 0.f;
    __syncthreads();
    float* acc = s_acc + warp * L.out;
#pragma unroll 1
    for (int rl = warp; rl < r1 - r0; rl += kW) {
        const int m = s_m[rl];
        const float t = s_t[rl];
        const uint32_t* rec = s_rec ? s_rec + static_cast<size_t>(rl) * L.out
                                    : L.rec + static_cast<size_t>(r0 + rl) * L.out;
        const uint16_t* plane = L.pair8 + static_cast<size_t>(m) * L.K;
#pragma unroll 1
        for (int j = lane; j < L.out; j += 64) {  // 2 independent edges per lane per step
            const bool two = j + 32 < L.out;
            const uint32_t ra = rec[j], rb = two ? rec[j + 32] : 0u;
            const uint32_t pa = __ldg(plane + (ra & 0xFFFFu)), pb = two ? __ldg(plane + (rb & 0xFFFFu)) : 0u;
            float c0, dc;
            pair_to_f(pa, c0, dc);
            acc[j] = fmaf(gain_of_rec(L, ra), fmaf(t, dc, c0), acc[j]);
            if (two) {
                pair_to_f(pb, c0, dc);
                acc[j + 32] = fmaf(gain_of_rec(L, rb), fmaf(t, dc, c0), acc[j + 32]);
            }
        }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < L.out; j += kT) {
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < kW; ++w) s += s_acc[w * L.out + j];
        part_out[static_cast<size_t>(blockIdx.x) * L.out + j] = s;
    }
}

// floor(a / b) for 0 <= a < 2^24, 1 <= b < 2^24: fp32 reciprocal estimate
// (off by at most one), one integer fix-up each way (no division sequence)
__device__ __forceinline__ int idiv_small(int a, int b) {
    int q = static_cast<int>(static_cast<float>(a) * __frcp_rn(static_cast<float>(b)));
    if ((q + 1) * b <= a) ++q;
    if (q * b > a) --q;
    return q;
}

// Exact bracket of an in-domain (or clamped) x from a bracket estimate
// within one of the answer, by double comparisons against the reference's
// node positions (kan.cpp:21-58: the unique i with node(i) <= x < node(i+1)).
__device__ __forceinline__ int bracket_exact(const double* node, const DevLayer& L, double x, int est) {
    if (!(x > L.lo)) return 0;
    if (!(x < L.hi)) return L.G - 2;
    int i = min(max(est, 0), L.G - 2);
    if (x < node[i]) --i;
    else if (x >= node[i + 1]) ++i;
    return i;
}

// Pair-plane layer 0.  Shared memory: [plane K*2 B][records rec_cap rows x
// out x 4 B]; x, t and brackets of all inputs are staged in the record
// region first (free until the records land).  Rows beyond rec_cap (only
// for very skewed shapes) read their records from global memory.
__device__ void planes_layer0(const HeadB1Args& h, unsigned char* smem, uint64_t* bar_x, uint64_t* bar,
                              float* part_out) {
    const DevLayer& L = h.L[0];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int GP = L.G - 1;
    __shared__ int s_cnt[32];
    __shared__ int s_scan[kW];
    __shared__ int s_bucket, s_lo, s_hi;
    __shared__ int s_rows[kMaxRows];
    __shared__ float s_trow[kMaxRows];
    uint16_t* s_plane = reinterpret_cast<uint16_t*>(smem);
    const uint32_t plane_bytes = static_cast<uint32_t>(L.K) * 2u;
    uint32_t* s_rec = reinterpret_cast<uint32_t*>(smem + ((plane_bytes + 127u) & ~127u));
    const uint32_t row_bytes = static_cast<uint32_t>(L.out) * 4u;
    double* s_x = reinterpret_cast<double*>(s_rec);
    uint8_t* s_bm = reinterpret_cast<uint8_t*>(s_x + L.in);  // brackets, padded to whole words with 0xFF
    const uint32_t* s_bw = reinterpret_cast<const uint32_t*>(s_bm);
    const int nwords = (L.in + 3) / 4;

    if (h.x_tma) {
        mbar_wait(bar_x, 0);
    } else {
        for (int i = tid; i < L.in; i += kT) s_x[i] = h.x[i];
        __syncthreads();
    }
    stamp(h, 2);
    // 1. brackets of all inputs, input i by thread i % kT: fp32 estimate; the
    //    undecided (near a knot, at the domain ends) settle by exact double
    //    comparisons against the node table; t comes later, for this CTA's
    //    rows only
    {
        int m[kMaxPer];
        unsigned hard = 0;
#pragma unroll
        for (int q = 0; q < kMaxPer; ++q) {
            const int i = tid + q * kT;
            m[q] = -1;
            if (i < L.in && !bracket_f32(L, s_x[i], m[q])) hard |= 1u << q;
        }
#pragma unroll 1
        for (; hard; hard &= hard - 1) {
            const int q = __ffs(hard) - 1;
            int est = -1;
#pragma unroll
            for (int u = 0; u < kMaxPer; ++u)
                if (u == q) est = m[u];
            const double x = s_x[tid + q * kT];
            int mm;
            if (!finite_bits(x) || !(L.qf_eps >= 0.f)) {
                float tt;
                fast_locate(L, x, h.err, mm, tt);
            } else {
                mm = bracket_exact(h.node0, L, x, est);
            }
#pragma unroll
            for (int u = 0; u < kMaxPer; ++u)
                if (u == q) m[u] = mm;
        }
#pragma unroll
        for (int q = 0; q < kMaxPer; ++q) {
            const int i = tid + q * kT;
            if (i < L.in) s_bm[i] = static_cast<uint8_t>(m[q]);
        }
        if (tid < 4 * nwords - L.in) s_bm[L.in + tid] = 0xFF;
    }
    __syncthreads();
    // 2. histogram: warp w counts buckets w, w+kW, ... over the bracket bytes
    //    four at a time (integer counts: order-free, deterministic)
#pragma unroll 1
    for (int b = warp; b < GP; b += kW) {
        const uint32_t pat = static_cast<uint32_t>(b) * 0x01010101u;
        int n = 0;
#pragma unroll 4
        for (int w4 = lane; w4 < nwords; w4 += 32) n += __popc(__vcmpeq4(s_bw[w4], pat) & 0x01010101u);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xFFFFFFFFu, n, o);
        if (lane == 0) s_cnt[b] = n;
    }
    __syncthreads();
    stamp(h, 3);
    // 3. CTA -> bucket (warp 0, lane b = bucket b): each non-empty bucket
    //    gets 1 + floor((P - nonempty) * n_b / in) CTAs; CTA c serves the
    //    bucket whose CTA range contains c and an even share of its rows.
    //    The plane (largest transfer) is requested first.
    if (warp == 0) {
        const int P = gridDim.x;
        const int n = lane < GP ? s_cnt[lane] : 0;
        const int nonempty = __popc(__ballot_sync(0xFFFFFFFFu, n > 0));
        const int alloc = n > 0 ? 1 + idiv_small((P - nonempty) * n, L.in) : 0;
        int incl = alloc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += y;
        }
        const int c = blockIdx.x;
        const bool mine = c >= incl - alloc && c < incl;
        if (mine) {  // at most one lane
            const int q = c - (incl - alloc);
            const int lo = idiv_small(n * q, alloc), hi = idiv_small(n * (q + 1), alloc);
            s_bucket = lane;
            s_lo = lo;
            s_hi = hi;
            const int rec_rows = min(min(hi - lo, kMaxRows), h.rec_cap);
            mbar_expect_tx(bar, plane_bytes + static_cast<uint32_t>(rec_rows) * row_bytes);
            bulk_g2s(smem, L.pair8 + static_cast<size_t>(lane) * L.K, plane_bytes, bar);  // the whole plane
        }
        if (__ballot_sync(0xFFFFFFFFu, mine) == 0 && lane == 0) {  // spare CTA: no rows
            s_bucket = GP;
            s_lo = s_hi = 0;
        }
    }
    // 4. my rows: thread t scans bracket words [2t, 2t+2), rank = exclusive
    //    scan of the match counts, rows ascending in i
    __syncthreads();
    const int bucket = s_bucket, lo = s_lo, hi = s_hi;
    const int nrows = min(hi - lo, kMaxRows);
    const int rec_rows = min(nrows, h.rec_cap);
    const uint32_t pat = static_cast<uint32_t>(bucket) * 0x01010101u;
    const int wpt = (nwords + kT - 1) / kT;
    uint32_t hits[4];
    int cnt = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int w4 = tid * wpt + u;
        hits[u] = (u < wpt && w4 < nwords) ? (__vcmpeq4(s_bw[w4], pat) & 0x01010101u) : 0u;
        cnt += __popc(hits[u]);
    }
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_scan[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int v = lane < kW ? s_scan[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xFFFFFFFFu, v, o);
            if (lane >= o) v += y;
        }
        if (lane < kW) s_scan[lane] = v;  // inclusive prefix over warps
    }
    __syncthreads();
    int rank = incl - cnt + (warp > 0 ? s_scan[warp - 1] : 0) - lo;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll 1
        for (uint32_t mk = hits[u]; mk; mk &= mk - 1) {
            const int i = (tid * wpt + u) * 4 + (__ffs(mk) - 1) / 8;
            if (rank >= 0 && rank < nrows) {
                // t of this row (fast path: float(x - node(m)) / dx, t = 1 at or past the upper node)
                const double x = s_x[i];
                float t;
                if (!(x > L.lo)) t = 0.f;
                else if (!(x < L.hi) || x >= h.node0[bucket + 1]) t = 1.f;
                else t = fminf(fmaxf(__double2float_rn(__dsub_rn(x, h.node0[bucket])) * L.inv_dx_f, 0.f), 1.f);
                s_rows[rank] = i;
                s_trow[rank] = t;
            }
            ++rank;
        }
    }
    __syncthreads();  // staging area free: records may land now
    if (tid < rec_rows)
        bulk_g2s(s_rec + static_cast<size_t>(tid) * L.out, L.rec + static_cast<size_t>(s_rows[tid]) * L.out,
                 row_bytes, bar);
    stamp(h, 4);
    if (bucket < GP) mbar_wait(bar, 0);
    stamp(h, 5);
    // 5. thread t: outputs 4t..4t+3 over all of this CTA's rows, ascending
    //    (records from shared memory; rows past rec_cap from global memory)
    const int j = tid * 4;
    if (j < L.out) {
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
        auto edge4 = [&](const uint4& r, float t) {
            float c0, dc;
            pair_to_f(s_plane[r.x & 0xFFFFu], c0, dc);
            a0 = fmaf(gain_of_rec(L, r.x), fmaf(t, dc, c0), a0);
            pair_to_f(s_plane[r.y & 0xFFFFu], c0, dc);
            a1 = fmaf(gain_of_rec(L, r.y), fmaf(t, dc, c0), a1);
            pair_to_f(s_plane[r.z & 0xFFFFu], c0, dc);
            a2 = fmaf(gain_of_rec(L, r.z), fmaf(t, dc, c0), a2);
            pair_to_f(s_plane[r.w & 0xFFFFu], c0, dc);
            a3 = fmaf(gain_of_rec(L, r.w), fmaf(t, dc, c0), a3);
        };
        const uint4* srec = reinterpret_cast<const uint4*>(s_rec + j);
        const int rstride = L.out / 4;
#pragma unroll 2
        for (int rr = 0; rr < rec_rows; ++rr) edge4(srec[rr * rstride], s_trow[rr]);
#pragma unroll 1
        for (int rr = rec_rows; rr < nrows; ++rr)
            edge4(__ldg(reinterpret_cast<const uint4*>(L.rec + static_cast<size_t>(s_rows[rr]) * L.out + j)), s_trow[rr]);
        *reinterpret_cast<float4*>(part_out + static_cast<size_t>(blockIdx.x) * L.out + j) = make_float4(a0, a1, a2, a3);
    }
}

__global__ void __launch_bounds__(kT, 1) k_head_b1(const __grid_constant__ HeadB1Args hp) {
    extern __shared__ __align__(128) unsigned char smem[];
    const HeadB1Args& h = hp;  // parameters straight from the constant bank
    // bias sums: layer 0's of this CTA's layer-1 rows, later the last layer's
    __shared__ double s_bias[kT];
    __shared__ __align__(8) uint64_t s_bar[3];  // [0] layer-0 plane+records, [1] row-split prefetch, [2] x
    __shared__ int s_last;
    const int P = gridDim.x, c = blockIdx.x;
    stamp(hp, 0);
    stamp_clock(hp, 14);
    unsigned char* s_pref = smem + hp.pref_offset;
    if (threadIdx.x == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        mbar_init(&s_bar[2], 1);
        // x (layer-0 pair planes) and this CTA's row-split records (contiguous
        // rows) are bulk-copied now
        if (hp.planes0 && hp.x_tma) {
            const uint32_t xb = static_cast<uint32_t>(hp.L[0].in) * 8u;
            const uint32_t plane_bytes = static_cast<uint32_t>(hp.L[0].K) * 2u;
            unsigned char* dst = smem + ((plane_bytes + 127u) & ~127u);
            mbar_expect_tx(&s_bar[2], xb);
            for (uint32_t off = 0; off < xb; off += 32768u)
                bulk_g2s(dst + off, reinterpret_cast<const char*>(hp.x) + off, min(32768u, xb - off), &s_bar[2]);
        }
        if (hp.pref_mask) {
            uint32_t total = 0;
#pragma unroll 1
            for (int l = 0; l < hp.nl; ++l) {
                if (!(hp.pref_mask >> l & 1)) continue;
                int r0, r1;
                rows_of(hp.L[l], c, P, r0, r1);
                total += static_cast<uint32_t>(r1 - r0) * hp.L[l].out * 4u;
            }
            mbar_expect_tx(&s_bar[1], total);
            uint32_t off = 0;
#pragma unroll 1
            for (int l = 0; l < hp.nl; ++l) {
                if (!(hp.pref_mask >> l & 1)) continue;
                int r0, r1;
                rows_of(hp.L[l], c, P, r0, r1);
                const uint32_t bytes = static_cast<uint32_t>(r1 - r0) * hp.L[l].out * 4u;
                if (bytes)
                    bulk_g2s(s_pref + off, hp.L[l].rec + static_cast<size_t>(r0) * hp.L[l].out, bytes, &s_bar[1]);
                off += bytes;
            }
        }
    } else if (threadIdx.x < 32 + 2 * hp.nl && threadIdx.x >= 32) {
        // every layer's records and pair planes start streaming from HBM into
        // L2 now, sliced over the CTAs, so the dependent gathers and bulk
        // copies below hit L2 (the whole head is ~13 MB of a ~126 MB L2)
        const DevLayer& L = hp.L[(threadIdx.x - 32) >> 1];
        if (threadIdx.x & 1)
            prefetch_l2_slice(L.pair8, static_cast<size_t>(L.K) * (L.G - 1) * 2, c, P);
        else
            prefetch_l2_slice(L.rec, static_cast<size_t>(L.in) * L.out * 4, c, P);
    }
    // bias sums needed late (layer-1 row reduction, final reduction) are
    // loaded into registers now; the loads complete off the critical path
    double b1_reg = 0.0, bf_reg = 0.0;
    if (hp.nl >= 2) {
        int r0, r1;
        rows_of(hp.L[1], c, P, r0, r1);
        if (threadIdx.x < r1 - r0) b1_reg = hp.L[0].bias_sum[r0 + threadIdx.x];
    }
    if (threadIdx.x < hp.L[hp.nl - 1].out) bf_reg = hp.L[hp.nl - 1].bias_sum[threadIdx.x];
    __syncthreads();
    stamp(h, 1);
    int* s_m = reinterpret_cast<int*>(smem);  // row-split scratch (after layer 0)
    uint32_t pref_off = 0;
    bool pref_ready = false;
#pragma unroll 1
    for (int l = 0; l < h.nl; ++l) {
        const DevLayer& L = h.L[l];
        float* part_out = h.part[l & 1];
        if (l == 0 && h.planes0) {
            planes_layer0(h, smem, &s_bar[2], &s_bar[0], part_out);
        } else {
            int r0, r1;
            rows_of(L, c, P, r0, r1);
            const int nr = r1 - r0;
            float* s_t = reinterpret_cast<float*>(s_m + nr);
            float* s_acc = s_t + nr;
            if (l == 0) {
                for (int q = threadIdx.x; q < nr; q += kT) fast_locate(L, h.x[r0 + q], h.err, s_m[q], s_t[q]);
            } else {
                // bias sums: staged for layer 1, straight from memory deeper in
                float* s_red = s_acc + kW * L.out;
                double* bias = s_bias;
                if (l == 1 && nr <= kT) {
                    s_bias[threadIdx.x] = b1_reg;
                } else {
                    bias = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(s_red + P * nr) + 15) & ~uintptr_t(15));
                    for (int q = threadIdx.x; q < nr; q += kT) bias[q] = h.L[l - 1].bias_sum[r0 + q];
                }
                reduce_rows(h.part[(l - 1) & 1], L.in, P, bias, L, r0, r1, s_m, s_t, s_red, h.err);
            }
            const uint32_t* s_rec = nullptr;
            if (h.pref_mask >> l & 1) {
                if (!pref_ready) {
                    mbar_wait(&s_bar[1], 0);
                    pref_ready = true;
                }
                s_rec = reinterpret_cast<const uint32_t*>(s_pref + pref_off);
                pref_off += static_cast<uint32_t>(nr) * L.out * 4u;
            }
            __syncthreads();
            stamp(h, l == 0 ? 8 : 9);
            rowsplit_layer(L, r0, r1, s_m, s_t, s_rec, s_acc, part_out);
        }
        stamp(h, l == 0 ? 6 : 10);
        if (l + 1 < h.nl) {
            grid_sync();
            stamp(h, l == 0 ? 7 : 11);
        }
    }
    // last layer: the last CTA to arrive reduces every output, one warp each
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned old = atomicAdd(h.done, 1u);
        s_last = old - h.epoch == static_cast<unsigned>(P - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    stamp(h, 12);
    const DevLayer& L = h.L[h.nl - 1];
    const float* part = h.part[(h.nl - 1) & 1];
    const int total = P * L.out;
    s_bias[threadIdx.x] = bf_reg;
    if (static_cast<size_t>(total) * 4 <= h.pref_offset && L.out <= kT) {
        // the [P][out] partial block, loaded coalesced into shared memory,
        // then C lanes per output in ascending z and a fixed butterfly
        float* s_fin = reinterpret_cast<float*>(smem);
#pragma unroll 1
        for (int e0 = threadIdx.x; e0 < total; e0 += 8 * kT) {
            float v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = e0 + u * kT < total ? __ldcg(part + e0 + u * kT) : 0.f;
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (e0 + u * kT < total) s_fin[e0 + u * kT] = v[u];
        }
        __syncthreads();
        int C = 1;
        while (C < 32 && (C * 2) * L.out <= kT) C <<= 1;
        const int cl = threadIdx.x & (C - 1), groups = kT / C;
        for (int pass = 0; pass < L.out; pass += groups) {
            const int q = pass + threadIdx.x / C;
            const int j = min(q, L.out - 1);
            double v = 0.0;
#pragma unroll 4
            for (int z = cl; z < P; z += C) v += static_cast<double>(s_fin[z * L.out + j]);
            for (int o = C >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
            if (cl == 0 && q < L.out) h.y[j] = v + s_bias[j];
        }
    } else {
        __syncthreads();
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll 1
        for (int j = warp; j < L.out; j += kW) {
            double v = 0.0;
#pragma unroll 1
            for (int z0 = lane; z0 < P; z0 += 8 * 32) {  // all loads of a lane issued at once
                float buf[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int z = z0 + 32 * u;
                    buf[u] = z < P ? __ldcg(part + static_cast<size_t>(z) * L.out + j) : 0.f;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) v += static_cast<double>(buf[u]);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
            if (lane == 0) h.y[j] = v + (j < kT ? s_bias[j] : L.bias_sum[j]);
        }
    }
    stamp(h, 13);
    stamp_clock(h, 15);
    // every CTA has arrived: the counters restart at 0 for the next launch
    // (stream order makes the reset visible to it), so a launch's
    // parameters never change from call to call (CUDA-graph replay)
    if (threadIdx.x == 0) {
        h.done[0] = 0u;
        h.done[1] = 0u;
    }
}

// ===========================================================================
// v2: the two-layer head [wide int8 layer] -> [narrow last layer] (the
// detection-head shape), same algorithm and summation orders as v1 but a
// shorter critical path, shaped by measured costs (tools/mb_handoff.cu,
// profiles/r2/): a warp's scattered 4-byte loads of other CTAs' partials cost
// ~2.7k cycles where one coalesced 16-byte load per thread of a contiguous
// block costs ~0.7k, so every cross-CTA hand-off is laid out contiguously
// for its consumer.
//   * x goes straight into registers with coalesced 16-byte loads: thread
//     (w, l) owns inputs 256w + 64q + 2l + e (q < 4, e < 2);
//   * per-warp bracket counts (REDUX); every warp derives the bucket
//     allocation and its offset into the CTA's bucket from them, and ranks
//     its rows with ballots: one block barrier between "x arrived" and
//     "records requested", each thread bulk-copies the records of the rows
//     it found;
//   * layer 1's records (bulk copy at kernel start) and its edges' codebook
//     rows (one 16-byte row per edge, all knots) are in shared memory before
//     layer 0 ends: after the grid barrier layer 1 makes one dependent load;
//   * layer 0's partials are written consumer-blocked, part0[d][c][0..nr1):
//     consumer d reads one contiguous P x nr1 block;
//   * the last layer's partials part1[c][0..out) are contiguous for the last
//     arriving CTA, which reduces them.
constexpr int kPer2 = 8;  // layer-0 inputs per thread: in0 <= kT * kPer2

__device__ __forceinline__ float t_of(const DevLayer& L, double x, double nlo, double nhi) {
    if (!(x > L.lo)) return 0.f;
    if (!(x < L.hi) || x >= nhi) return 1.f;
    return fminf(fmaxf(__double2float_rn(__dsub_rn(x, nlo)) * L.inv_dx_f, 0.f), 1.f);
}

__global__ void __launch_bounds__(kT, 1) k_head_b1v2(const __grid_constant__ HeadB1Args hp) {
    extern __shared__ __align__(128) unsigned char smem[];
    // The parameters this kernel reads (layers 0-1 and the launch fields) are
    // copied into shared memory once, all words in parallel: afterwards no
    // phase pays a constant-cache miss on a parameter line it touches first.
    __shared__ __align__(16) HeadB1Args s_h;
    __shared__ __align__(8) uint64_t s_bar[2];  // [0] plane + layer-0 records, [1] layer-1 records + rows
    __shared__ int s_wcnt[kW][32];              // per-warp bracket counts
    __shared__ int s_rows[kMaxRows];
    __shared__ float s_trow[kMaxRows];
    __shared__ double s_bias1[kW];              // layer 0's bias sums of my layer-1 rows
    __shared__ double s_bfin[32];               // layer 1's bias sums
    __shared__ int s_last;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int P = gridDim.x, c = blockIdx.x;
    // x first: four coalesced loads per thread (straight from the parameters)
    double xr[kPer2];
    {
        const int in0 = hp.L[0].in;
        const double* x = hp.x;
        const int base = 256 * warp + 2 * lane;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int i = base + 64 * q;
            if (hp.x_tma && i + 1 < in0) {
                const double2 v = __ldg(reinterpret_cast<const double2*>(x + i));
                xr[2 * q] = v.x;
                xr[2 * q + 1] = v.y;
            } else {
                xr[2 * q] = i < in0 ? x[i] : 0.0;
                xr[2 * q + 1] = i + 1 < in0 ? x[i + 1] : 0.0;
            }
        }
    }
    {
        constexpr int a1 = static_cast<int>((offsetof(HeadB1Args, L) + 2 * sizeof(DevLayer)) / 4);
        constexpr int b0 = static_cast<int>(offsetof(HeadB1Args, planes0) / 4);
        constexpr int b1 = static_cast<int>(sizeof(HeadB1Args) / 4);
        static_assert(offsetof(HeadB1Args, planes0) % 4 == 0 && a1 + (b1 - b0) <= kT, "parameter copy");
        const uint32_t* src = reinterpret_cast<const uint32_t*>(&hp);
        uint32_t* dst = reinterpret_cast<uint32_t*>(&s_h);
        if (tid < a1) dst[tid] = src[tid];
        else if (tid - a1 < b1 - b0) dst[b0 + tid - a1] = src[b0 + tid - a1];
    }
    __syncthreads();
    const HeadB1Args& h = s_h;
    const DevLayer& L = h.L[0];
    const DevLayer& L1 = h.L[1];
    stamp(h, 0);
    if (h.exit_at == 100) return;
    unsigned char* s_pref = smem + h.pref_offset;
    uint4* s_cb = reinterpret_cast<uint4*>(smem + h.cbrow_offset);
    int r10, r11;
    rows_of(L1, c, P, r10, r11);
    const int nr = r11 - r10;
    if (tid == 0) {
        // layer 1's records and its edges' codebook rows (pre-gathered at
        // upload, one 16-byte row per edge) for my rows: no dependent gather
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        const uint32_t n1 = static_cast<uint32_t>(nr) * L1.out;
        mbar_expect_tx(&s_bar[1], n1 * 4u + n1 * 16u);
        bulk_g2s(s_pref, L1.rec + static_cast<size_t>(r10) * L1.out, n1 * 4u, &s_bar[1]);
        bulk_g2s(s_cb, h.l1rows + static_cast<size_t>(r10) * L1.out, n1 * 16u, &s_bar[1]);
    } else if (warp == 1 && lane < 2) {
        // layer 0 streams HBM -> L2 from the first microsecond, sliced over the CTAs
        if (lane == 0) prefetch_l2_slice(L.rec, static_cast<size_t>(L.in) * L.out * 4, c, P);
        else prefetch_l2_slice(L.pair8, static_cast<size_t>(L.K) * (L.G - 1) * 2, c, P);
    }
    const double b1_reg = tid < nr ? L.bias_sum[r10 + tid] : 0.0;
    const double bf_reg = tid < L1.out ? L1.bias_sum[tid] : 0.0;
    stamp(h, 1);
    if (h.exit_at == 1) return;
    // brackets: fp32 estimate, exact double comparisons where undecided
    const int GP = L.G - 1;
    int mb[kPer2];
    unsigned hard = 0;
#pragma unroll
    for (int q = 0; q < kPer2; ++q) {
        const int i = 256 * warp + 64 * (q >> 1) + 2 * lane + (q & 1);
        mb[q] = 0xFF;
        if (i < L.in && !bracket_f32(L, xr[q], mb[q])) hard |= 1u << q;
    }
#pragma unroll 1
    for (; hard; hard &= hard - 1) {
        const int q = __ffs(hard) - 1;
        double x = 0.0;
        int est = 0;
#pragma unroll
        for (int u = 0; u < kPer2; ++u)
            if (u == q) {
                x = xr[u];
                est = mb[u];
            }
        int mm;
        if (!finite_bits(x) || !(L.qf_eps >= 0.f)) {
            float tt;
            fast_locate(L, x, h.err, mm, tt);
        } else {
            mm = bracket_exact(h.node0, L, x, est);
        }
#pragma unroll
        for (int u = 0; u < kPer2; ++u)
            if (u == q) mb[u] = mm;
    }
    stamp(h, 11);
    const uint32_t w0 = static_cast<uint32_t>(mb[0]) | mb[1] << 8 | mb[2] << 16 | static_cast<uint32_t>(mb[3]) << 24;
    const uint32_t w1 = static_cast<uint32_t>(mb[4]) | mb[5] << 8 | mb[6] << 16 | static_cast<uint32_t>(mb[7]) << 24;
#pragma unroll 1
    for (int b = 0; b < GP; ++b) {  // per-warp counts (integer: order-free)
        const uint32_t pat = static_cast<uint32_t>(b) * 0x01010101u;
        const int n = __popc(__vcmpeq4(w0, pat) & 0x01010101u) + __popc(__vcmpeq4(w1, pat) & 0x01010101u);
        const int tot = __reduce_add_sync(0xFFFFFFFFu, n);
        if (lane == 0) s_wcnt[warp][b] = tot;
    }
    stamp(h, 2);
    if (h.exit_at == 2) return;
    __syncthreads();
    // every warp: bucket totals (lane b), the allocation of CTAs to buckets
    // (1 + floor((P - nonempty) * n_b / in) each, v1's rule), this CTA's
    // bucket and row range, and the bucket's count in earlier warps
    int nb = 0, before = 0;
    if (lane < GP) {
#pragma unroll 4
        for (int w = 0; w < kW; ++w) {
            const int v = s_wcnt[w][lane];
            nb += v;
            before += w < warp ? v : 0;
        }
    }
    const int nonempty = __popc(__ballot_sync(0xFFFFFFFFu, nb > 0));
    const int alloc = nb > 0 ? 1 + idiv_small((P - nonempty) * nb, L.in) : 0;
    int incl = alloc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    const bool mine = c >= incl - alloc && c < incl;
    const unsigned bal = __ballot_sync(0xFFFFFFFFu, mine);
    const int bucket = bal ? __ffs(bal) - 1 : GP;  // GP: spare CTA, no rows
    int lo = 0, hi = 0;
    if (mine) {
        const int q = c - (incl - alloc);
        lo = idiv_small(nb * q, alloc);
        hi = idiv_small(nb * (q + 1), alloc);
    }
    const int src = bucket < GP ? bucket : 0;
    lo = __shfl_sync(0xFFFFFFFFu, lo, src);
    hi = __shfl_sync(0xFFFFFFFFu, hi, src);
    before = __shfl_sync(0xFFFFFFFFu, before, src);
    const int nrows = min(hi - lo, kMaxRows);
    const int rec_rows = min(nrows, h.rec_cap);
    const uint16_t* s_plane = reinterpret_cast<const uint16_t*>(smem);
    const uint32_t plane_bytes = static_cast<uint32_t>(L.K) * 2u;
    uint32_t* s_rec = reinterpret_cast<uint32_t*>(smem + ((plane_bytes + 127u) & ~127u));
    const uint32_t row_bytes = static_cast<uint32_t>(L.out) * 4u;
    if (tid == 0 && bucket < GP) {
        mbar_expect_tx(&s_bar[0], plane_bytes + static_cast<uint32_t>(rec_rows) * row_bytes);
        bulk_g2s(smem, L.pair8 + static_cast<size_t>(bucket) * L.K, plane_bytes, &s_bar[0]);
    }
    stamp(h, 8);
    // my rows of the bucket in ascending i: within the warp i = 64q + 2l + e
    if (bucket < GP) {
        const uint32_t pat = static_cast<uint32_t>(bucket) * 0x01010101u;
        const uint32_t m0 = __vcmpeq4(w0, pat), m1 = __vcmpeq4(w1, pat);
        const double nlo = h.node0[bucket], nhi = h.node0[bucket + 1];
        const unsigned lt = (1u << lane) - 1u;
        int base = before - lo;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t m = q < 2 ? m0 : m1;
            const bool e0 = (m >> (16 * (q & 1))) & 1u, e1 = (m >> (16 * (q & 1) + 8)) & 1u;
            const unsigned B0 = __ballot_sync(0xFFFFFFFFu, e0), B1 = __ballot_sync(0xFFFFFFFFu, e1);
            int r = base + __popc(B0 & lt) + __popc(B1 & lt);
            const int i = 256 * warp + 64 * q + 2 * lane;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                if (e ? e1 : e0) {
                    if (r >= 0 && r < nrows) {
                        s_rows[r] = i + e;
                        s_trow[r] = t_of(L, xr[2 * q + e], nlo, nhi);
                        if (r < rec_rows)
                            bulk_g2s(s_rec + static_cast<size_t>(r) * L.out,
                                     L.rec + static_cast<size_t>(i + e) * L.out, row_bytes, &s_bar[0]);
                    }
                    ++r;
                }
            }
            base += __popc(B0) + __popc(B1);
        }
    }
    stamp(h, 9);
    stamp(h, 3);
    if (h.exit_at == 3) return;
    __syncthreads();
    if (bucket < GP) mbar_wait(&s_bar[0], 0);
    stamp(h, 4);
    if (h.exit_at == 4) return;
    // layer 0: thread t owns outputs 4t..4t+3 over this CTA's rows, ascending;
    // its four sums go straight to the consumer-blocked partials
    // part0[d][c][j - r0(d)], d = the CTA whose layer-1 rows hold j
    {
        const int j = tid * 4;
        if (j < L.out) {
            float a[4] = {0.f, 0.f, 0.f, 0.f};
            auto edge4 = [&](const uint4& r, float t) {
                float c0, dc;
                pair_to_f(s_plane[r.x & 0xFFFFu], c0, dc);
                a[0] = fmaf(gain_of_rec(L, r.x), fmaf(t, dc, c0), a[0]);
                pair_to_f(s_plane[r.y & 0xFFFFu], c0, dc);
                a[1] = fmaf(gain_of_rec(L, r.y), fmaf(t, dc, c0), a[1]);
                pair_to_f(s_plane[r.z & 0xFFFFu], c0, dc);
                a[2] = fmaf(gain_of_rec(L, r.z), fmaf(t, dc, c0), a[2]);
                pair_to_f(s_plane[r.w & 0xFFFFu], c0, dc);
                a[3] = fmaf(gain_of_rec(L, r.w), fmaf(t, dc, c0), a[3]);
            };
            const uint4* srec = reinterpret_cast<const uint4*>(s_rec + j);
            const int rstride = L.out / 4;
#pragma unroll 2
            for (int rr = 0; rr < rec_rows; ++rr) edge4(srec[rr * rstride], s_trow[rr]);
#pragma unroll 1
            for (int rr = rec_rows; rr < nrows; ++rr)
                edge4(__ldg(reinterpret_cast<const uint4*>(L.rec + static_cast<size_t>(s_rows[rr]) * L.out + j)),
                      s_trow[rr]);
            stamp(h, 10);
            const int NR = h.nr1;
            float* part0 = h.part[0];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int jj = j + u;
                // largest d with floor(in1 * d / P) <= jj
                const int d = idiv_small((jj + 1) * P - 1, L1.in);
                const int r0 = idiv_small(L1.in * d, P);
                part0[(static_cast<size_t>(d) * P + c) * NR + (jj - r0)] = a[u];
            }
        }
    }
    if (tid < nr) s_bias1[tid] = b1_reg;
    if (tid < L1.out) s_bfin[tid] = bf_reg;
    stamp(h, 5);
    if (h.exit_at == 5) return;
    grid_barrier(h.done + 1, h.epoch + static_cast<unsigned>(P));
    stamp(h, 6);
    // layer 1: my consumer block (P x NR, contiguous) -> shared memory
    {
        const int NR = h.nr1;
        float* s_red = reinterpret_cast<float*>(smem);
        float* s_term = s_red + P * NR;
        const float* blk = h.part[0] + static_cast<size_t>(c) * P * NR;
        const int n4 = P * NR / 4;
#pragma unroll 1
        for (int e = tid; e < n4; e += kT)
            reinterpret_cast<float4*>(s_red)[e] = __ldcg(reinterpret_cast<const float4*>(blk) + e);
        for (int e = 4 * n4 + tid; e < P * NR; e += kT) s_red[e] = __ldcg(blk + e);
        __syncthreads();
        mbar_wait(&s_bar[1], 0);
        // warp w: row r10 + w.  Lanes sum z = lane, lane + 32, ... in order, a
        // fixed butterfly, lane 0's value; locate; lane j forms edge (w, j)
        if (warp < nr) {
            double v = 0.0;
#pragma unroll 1
            for (int z = lane; z < P; z += 32) v += static_cast<double>(s_red[z * NR + warp]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
            v = __shfl_sync(0xFFFFFFFFu, v, 0) + s_bias1[warp];
            int m;
            float t;
            fast_locate(L1, v, h.err, m, t);
            if (lane < L1.out) {
                const int e = warp * L1.out + lane;
                const int8_t* cb = reinterpret_cast<const int8_t*>(s_cb + e);
                const float c0 = static_cast<float>(cb[m]);
                const float dc = static_cast<float>(cb[m + 1]) - c0;
                s_term[e] = gain_of_rec(L1, reinterpret_cast<const uint32_t*>(s_pref)[e]) * fmaf(t, dc, c0);
            }
        }
        __syncthreads();
        if (tid < L1.out) {
            float s = 0.f;
#pragma unroll 1
            for (int w = 0; w < nr; ++w) s += s_term[w * L1.out + tid];
            h.part[1][static_cast<size_t>(c) * L1.out + tid] = s;
        }
    }
    stamp(h, 7);
    if (h.exit_at == 7) return;
    // the last CTA to arrive reduces the [P][out] block (contiguous)
    __syncthreads();
    if (tid == 0) s_last = arrive_acq_rel(h.done) - h.epoch == static_cast<unsigned>(P - 1);
    __syncthreads();
    if (!s_last) return;
    stamp(h, 12);
    {
        const float* part = h.part[1];
        const int total = P * L1.out;
        float* s_fin = reinterpret_cast<float*>(smem);
#pragma unroll 1
        for (int e0 = tid; e0 < total; e0 += 8 * kT) {
            float v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = e0 + u * kT < total ? __ldcg(part + e0 + u * kT) : 0.f;
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (e0 + u * kT < total) s_fin[e0 + u * kT] = v[u];
        }
        __syncthreads();
        int C = 1;
        while (C < 32 && (C * 2) * L1.out <= kT) C <<= 1;
        const int cl = tid & (C - 1), groups = kT / C;
        for (int pass = 0; pass < L1.out; pass += groups) {
            const int q = pass + tid / C;
            const int j = min(q, L1.out - 1);
            double v = 0.0;
#pragma unroll 4
            for (int z = cl; z < P; z += C) v += static_cast<double>(s_fin[z * L1.out + j]);
            for (int o = C >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
            if (cl == 0 && q < L1.out) h.y[j] = v + s_bfin[j];
        }
    }
    stamp(h, 13);
    if (tid == 0) {  // all CTAs arrived: restart the counters at 0 (see k_head_b1)
        h.done[0] = 0u;
        h.done[1] = 0u;
    }
}

}  // namespace

// Eligibility: every layer int8 with <= 65536-row codebooks (4-byte
// records), G-1 <= 32 brackets.
bool head_b1_supported(const DevLayer* L, int nl) {
    if (nl < 1 || nl > kMaxHeadLayers) return false;
    for (int l = 0; l < nl; ++l) {
        if (L[l].fmt != FMT_I8_R32 || L[l].G - 1 > 32 || L[l].out > 16384) return false;
    }
    return true;
}

// Shared-memory plan: [phase region][prefetched row-split records].  The
// phase region holds layer 0's plane + staged records (pair-plane layer) or
// a row-split layer's brackets and per-warp accumulators.  Fills
// h->planes0 / rec_cap / pref_mask / pref_offset.
size_t head_b1_smem(const DevLayer* L, int nl, int num_sms, HeadB1Args* h) {
    static const int force_v1 = [] {
        const char* e = std::getenv("SKAN_B1_V1");  // A/B experiment: the general batch-1 kernel
        return e && e[0] == '1';
    }();
    static const int exit_at = [] {
        const char* e = std::getenv("SKAN_B1_EXIT_AT");  // timing experiment
        return e ? std::atoi(e) : 0;
    }();
    h->exit_at = exit_at;
    const DevLayer& L0 = L[0];
    const size_t kBudget = 218 * 1024;  // dynamic; + ~7 KB static + 1 KB reserved <= 227 KB
    const int spare = num_sms - (L0.G - 1);
    h->planes0 = L0.out % 4 == 0 && L0.out <= 4 * kT && L0.in <= kMaxPer * kT && L0.K % 8 == 0 &&
                 static_cast<size_t>(L0.K) * 2 <= 160 * 1024 && L0.G - 1 <= 32 &&
                 static_cast<long long>(L0.in) * L0.out >= 256LL * 1024 && spare > 0 &&
                 L0.in / spare + 2 <= kMaxRows;
    const size_t plane = (static_cast<size_t>(L0.K) * 2 + 127) / 128 * 128;
    const size_t row = static_cast<size_t>(L0.out) * 4;
    const int want = spare > 0 ? L0.in / spare + 2 : 0;  // rows per CTA < in / (P - buckets) + 1
    h->part_floats = static_cast<unsigned>(static_cast<size_t>(num_sms) * 16384);  // refined below
    // v2: the two-layer head whose last layer is narrow
    const int nr1 = nl == 2 ? (L[1].in + num_sms - 1) / num_sms : 0;
    const bool v2 = !force_v1 && h->planes0 && nl == 2 && L0.in <= kPer2 * kT && nr1 <= kW && L[1].out <= 32 &&
                    L[1].rs == 16;
    if (v2) {
        h->version = 2;
        h->nr1 = nr1;
        h->pref_mask = 2;
        h->cbrow_mask = 2;
        const size_t out_b = 0;
        const size_t pref_b = (static_cast<size_t>(nr1) * L[1].out * 4 + 127) / 128 * 128;
        const size_t cb_b = static_cast<size_t>(nr1) * L[1].out * 16;
        const size_t avail = kBudget > plane + out_b + pref_b + cb_b ? kBudget - plane - out_b - pref_b - cb_b : 0;
        size_t cap = avail / row;
        if (cap > static_cast<size_t>(want)) cap = want;
        if (cap > static_cast<size_t>(kMaxRows)) cap = kMaxRows;
        h->rec_cap = static_cast<int>(cap);
        const size_t recs = (cap * row + 127) / 128 * 128;
        h->out_offset = 0;
        h->pref_offset = static_cast<uint32_t>(plane + recs);
        h->cbrow_offset = static_cast<uint32_t>(plane + recs + pref_b);
        h->part_floats = static_cast<unsigned>(std::max<size_t>(static_cast<size_t>(num_sms) * num_sms * nr1,
                                                                static_cast<size_t>(num_sms) * L[1].out));
        return h->cbrow_offset + cb_b;
    }
    h->version = 1;
    // prefetch: row-split layers whose per-CTA record block is small
    size_t pref = 0;
    h->pref_mask = 0;
    h->cbrow_mask = 0;
    for (int l = h->planes0 ? 1 : 0; l < nl; ++l) {
        const int rows = (L[l].in + num_sms - 1) / num_sms;
        const size_t b = static_cast<size_t>(rows) * L[l].out * 4;
        if (L[l].out % 4 == 0 && pref + b <= kPrefetchBytes) {
            h->pref_mask |= 1 << l;
            pref += b;
        }
    }
    size_t phase = 0;
    h->rec_cap = 0;
    int maxw = 0;
    for (int l = 0; l < nl; ++l) maxw = std::max({maxw, L[l].in, L[l].out});
    h->part_floats = static_cast<unsigned>(static_cast<size_t>(num_sms) * maxw);
    if (h->planes0) {
        const size_t avail = kBudget > plane + pref ? kBudget - plane - pref : 0;
        size_t cap = avail / row;
        if (cap > static_cast<size_t>(want)) cap = want;
        if (cap > static_cast<size_t>(kMaxRows)) cap = kMaxRows;
        h->rec_cap = static_cast<int>(cap);
        // the record region doubles as the input staging area (x, t, bracket)
        const size_t staging = static_cast<size_t>(L0.in) * (sizeof(double) + sizeof(float) + 1) + 128;
        phase = plane + (cap * row > staging ? cap * row : staging);
    }
    for (int l = 0; l < nl; ++l) {
        if (l == 0 && h->planes0) continue;
        // s_m, s_t, per-warp accumulators, the partial block, bias fallback
        const int nr = (L[l].in + num_sms - 1) / num_sms + 1;
        const size_t s = static_cast<size_t>(nr) * 8 + static_cast<size_t>(kW) * L[l].out * sizeof(float) +
                         static_cast<size_t>(num_sms) * nr * sizeof(float) + static_cast<size_t>(nr) * 8 + 32;
        if (s > phase) phase = s;
    }
    phase = (phase + 127) / 128 * 128;
    h->pref_offset = static_cast<uint32_t>(phase);
    return phase + pref;
}

int head_b1_max_grid(size_t smem, int num_sms) {
    // The attribute is per function and device, shared by every head: only
    // ever raise it, so a head planned later with a smaller footprint cannot
    // make an earlier head's launch exceed the limit.
    static std::mutex mu;
    static size_t set_max[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lk(mu);
        if (dev < 0 || dev >= 64) return 0;
        if (smem > set_max[dev]) {
            for (auto k : {k_head_b1, k_head_b1v2})
                if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
                    cudaSuccess) {
                    cudaGetLastError();
                    return 0;
                }
            set_max[dev] = smem;
        }
    }
    int per_sm = 0, per_sm2 = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_head_b1, kT, smem) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, k_head_b1v2, kT, smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return per_sm >= 1 && per_sm2 >= 1 ? num_sms : 0;
}

__global__ void k_b1_rows(const uint32_t* __restrict__ rec, const int8_t* __restrict__ cb8, int rs, uint4* dst,
                          int n) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x)
        dst[e] = *reinterpret_cast<const uint4*>(cb8 + static_cast<size_t>(rec[e] & 0xFFFFu) * rs);
}

size_t head_b1_rows_bytes(const HeadB1Args& h) {
    return h.version == 2 ? static_cast<size_t>(h.L[1].in) * h.L[1].out * 16 : 0;
}

cudaError_t head_b1_build_rows(const HeadB1Args& h, uint4* dst, cudaStream_t s) {
    const int n = h.L[1].in * h.L[1].out;
    k_b1_rows<<<std::max(1, std::min((n + 255) / 256, 148 * 8)), 256, 0, s>>>(h.L[1].rec, h.L[1].cb8, h.L[1].rs, dst,
                                                                              n);
    return cudaGetLastError();
}

cudaError_t launch_head_b1(const HeadB1Args& h, int grid, size_t smem, cudaStream_t s) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return h.version == 2 ? cudaLaunchKernelEx(&cfg, k_head_b1v2, h) : cudaLaunchKernelEx(&cfg, k_head_b1, h);
}

}  // namespace skan
