// sm_100a kernels for the LUTHAM forward (SHARe-KAN compressed KAN heads).
//
//   K1  knot selection, bit-exact with holoquant::locate (kan.cpp:28-58):
//       inline in the first layer's fused kernel, in the finisher of every
//       layer for the next one, or standalone (k_locate_input / k_locate_raw)
//   K2  fused decode + gather + interpolate + accumulate (fast path):
//         k_fwd_small  rows-in-warps, outputs-in-lanes (small batches):
//                      coalesced 128-bit record loads, one 2-byte codebook
//                      pair gather per edge-sample
//         k_fwd_large  samples-in-lanes (large batches): each edge decoded
//                      once per CTA into shared memory as gained (c0, dc)
//                      pairs, read back as warp broadcasts
//       both end in a fixed-order split reduction (no float atomics) done by
//       the last CTA of each output tile, fused with the next layer's K1
//   K2x k_gather_exact  fp64, reference operation order, sequential i:
//                      bitwise equal to compressed_forward (lutham.cpp:793-814)
//   K5  k_unpack_indices SKAN v1 LSB-first index unpack (lutham.cpp:114-137)
//       k_pli_lookup     batched single-edge primitive (lutham.cpp:730-739)
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "skan_device.cuh"
#include "skan_internal.hpp"

namespace skan {
namespace {

using namespace dev;

constexpr int kThreads = 128;  // threads per exact-kernel CTA
constexpr int kIC = 64;        // inputs whose brackets are staged per smem pass (exact kernel)

// x is [rows][width] row-major.  Brackets are written in the same layout, or
// input-major ([width][rows], rows = samples) when `rows_tr` > 0 -- the
// layout the fast-path kernels read (sample-contiguous).  With btd (exact
// path) t is locate()'s double; without it (fast path) the division-free
// fast_locate is used.
__global__ void k_locate_input(const double* __restrict__ x, long long n, DevLayer L, int* __restrict__ bm,
                               float* __restrict__ btf, double* __restrict__ btd, int* __restrict__ err,
                               int width, int rows_tr) {
    pdl_trigger();
    pdl_wait();
    for (long long p = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; p < n;
         p += static_cast<long long>(gridDim.x) * blockDim.x) {
        int m;
        long long src = p;
        if (rows_tr > 0) src = (p % rows_tr) * width + p / rows_tr;  // p = i*rows + s
        if (btd) {
            double t;
            bracket_of(L.lo, L.hi, L.G, L.dx, x[src], err, m, t);
            btf[p] = static_cast<float>(t);
            btd[p] = t;
        } else {
            float t;
            fast_locate(L, x[src], err, m, t);
            btf[p] = t;
        }
        bm[p] = m;
    }
}

// Fast-path brackets of x [rows][width] written input-major ([width][rows])
// through a 32 x 32 shared-memory tile: both the read of x and the write of
// the brackets are coalesced.
__global__ void __launch_bounds__(1024) k_locate_transpose(const double* __restrict__ x, int rows, int width,
                                                          DevLayer L, int* __restrict__ bm, float* __restrict__ bt,
                                                          int* __restrict__ err) {
    __shared__ int s_m[32][33];
    __shared__ float s_t[32][33];
    pdl_trigger();
    pdl_wait();
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 32: one entry per thread
    const int i0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    {
        const int r = r0 + ty, i = i0 + tx;
        int m = 0;
        float t = 0.f;
        if (r < rows && i < width) fast_locate(L, x[static_cast<size_t>(r) * width + i], err, m, t);
        s_m[ty][tx] = m;
        s_t[ty][tx] = t;
    }
    __syncthreads();
    const int i = i0 + ty, r = r0 + tx;
    if (r < rows && i < width) {
        bm[static_cast<size_t>(i) * rows + r] = s_m[tx][ty];
        bt[static_cast<size_t>(i) * rows + r] = s_t[tx][ty];
    }
}

// Shared finisher: runs in the last CTA of an output tile and reduces the
// tile's split partials.  C lanes cooperate on one (sample, output) entry
// (lane c sums splits c, c+C, ... in ascending order; a fixed segmented
// butterfly then combines the C lane sums) and every thread keeps kFinNB
// entries in flight.  C and the entry-to-thread map depend only on the
// launch shape, so the summation order -- hence the result bits -- never
// depends on timing.  Then bias sum, y, and the next layer's bracket.
constexpr int kFinNB = 8;

__device__ __forceinline__ void finish_entry(const FwdArgs& a, size_t p, int j, double v) {
    v += a.L.bias_sum ? a.L.bias_sum[j] : 0.0;
    a.y[p] = v;
    if (a.has_next) {
        int m;
        float t;
        fast_locate(a.N, v, a.err, m, t);
        const size_t s = p / a.L.out;
        const size_t q = static_cast<size_t>(j) * a.B + s;  // input-major for the next layer
        a.bm_out[q] = m;
        a.bt_out[q] = t;
    }
}

__device__ __forceinline__ void finish_tile(const FwdArgs& a, int nsplit, int s_begin, int s_count,
                                            int j_begin, int j_count) {
    const DevLayer& L = a.L;
    const size_t plane = static_cast<size_t>(a.B) * L.out;
    const int entries = s_count * j_count;
    int C = 1;  // lanes per entry: about 4 splits per lane, at most a warp
    while (C < 32 && C * 4 < nsplit) C <<= 1;
    const int c = threadIdx.x & (C - 1);
    const int R = blockDim.x / C;  // entry groups in flight per pass
    // uniform trip count for all threads (the butterfly needs full warps)
    for (int pass = 0; pass < entries; pass += R * kFinNB) {
        const int base = pass + (threadIdx.x / C) * kFinNB;
        double v[kFinNB];
        size_t p[kFinNB];
        int jj[kFinNB];
#pragma unroll
        for (int b = 0; b < kFinNB; ++b) {
            v[b] = 0.0;
            const int q = min(base + b, entries - 1);
            jj[b] = j_begin + q % j_count;
            p[b] = static_cast<size_t>(s_begin + q / j_count) * L.out + jj[b];
        }
#pragma unroll 2
        for (int z = c; z < nsplit; z += C) {
            const float* src = a.partial + z * plane;
#pragma unroll
            for (int b = 0; b < kFinNB; ++b) v[b] += static_cast<double>(__ldcg(src + p[b]));
        }
        for (int o = C >> 1; o > 0; o >>= 1) {
#pragma unroll
            for (int b = 0; b < kFinNB; ++b) v[b] += __shfl_xor_sync(0xFFFFFFFFu, v[b], o);
        }
        if (c == 0) {
#pragma unroll
            for (int b = 0; b < kFinNB; ++b)
                if (base + b < entries) finish_entry(a, p[b], jj[b], v[b]);
        }
    }
}

// Consumer-side reduction (after a pair-plane layer): brackets of the rows
// [r0, rend) x samples [s0, s0+nS) of THIS layer from the previous layer's
// split partials, same fixed C-lane order as finish_tile.  Writes
// s_m/s_t[sl*R + rl] for sl < S (padding entries get (0, 0)).
__device__ __forceinline__ void reduce_prev_rows(const FwdArgs& a, int r0, int rend, int s0, int nS, int S,
                                                 int R, int* s_m, float* s_t) {
    const DevLayer& L = a.L;
    const size_t plane = static_cast<size_t>(a.B) * L.in;
    const int entries = S * R;
    int C = 1;
    while (C < 32 && C * 4 < a.prev_nsplit) C <<= 1;
    const int c = threadIdx.x & (C - 1);
    const int groups = blockDim.x / C;
    for (int pass = 0; pass < entries; pass += groups * kFinNB) {
        const int base = pass + (threadIdx.x / C) * kFinNB;
        double v[kFinNB];
        size_t idx[kFinNB];
#pragma unroll
        for (int b = 0; b < kFinNB; ++b) {
            v[b] = 0.0;
            const int q = base + b, sl = q / R, i = r0 + q % R;
            const bool ok = q < entries && sl < nS && i < rend;
            idx[b] = ok ? static_cast<size_t>(s0 + sl) * L.in + i : 0;
        }
#pragma unroll 2
        for (int z = c; z < a.prev_nsplit; z += C) {
            const float* src = a.prev_partial + z * plane;
#pragma unroll
            for (int b = 0; b < kFinNB; ++b) v[b] += static_cast<double>(__ldcg(src + idx[b]));
        }
        for (int o = C >> 1; o > 0; o >>= 1) {
#pragma unroll
            for (int b = 0; b < kFinNB; ++b) v[b] += __shfl_xor_sync(0xFFFFFFFFu, v[b], o);
        }
        if (c == 0) {
#pragma unroll
            for (int b = 0; b < kFinNB; ++b) {
                const int q = base + b, sl = q / R, i = r0 + q % R;
                if (q >= entries) continue;
                int m = 0;
                float t = 0.f;
                if (sl < nS && i < rend) fast_locate(L, v[b] + a.prev_bias_sum[i], a.err, m, t);
                s_m[q] = m;
                s_t[q] = t;
            }
        }
    }
}

// Arrival counting: returns true in exactly one CTA per tile (the last).
__device__ __forceinline__ bool arrive_last(unsigned* counter, unsigned expected, int* s_flag) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(counter, 1u);
        *s_flag = prev == expected - 1;
        if (*s_flag) *counter = 0;  // ready for the next launch (stream ordered)
    }
    __syncthreads();
    if (*s_flag) __threadfence();
    return *s_flag;
}

// ---------------------------------------------------------------------------
// k_fwd_small: CTA = 8 warps; tile = (32*VJ outputs) x (8*RW input rows) x
// (S samples).  Warp w owns RW consecutive rows; lane l owns outputs
// j0 + l*VJ .. +VJ-1.  Records of a row are read with one coalesced 4*VJ-byte
// load per lane, all RW rows issued before the dependency wait; then one
// 2-byte gather per edge-sample from the pair table.  Per-lane fp32
// accumulation over the warp's rows, fixed-order sum over warps in smem,
// one fp32 partial per (split, sample, output).

template <int FMT, int VJ>
struct SmallEdges;

template <int VJ>
struct SmallEdges<FMT_I8_R32, VJ> {
    uint32_t r[VJ];
    __device__ __forceinline__ void load(const DevLayer& L, size_t e) {
        if constexpr (VJ == 4) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(L.rec + e));
            r[0] = v.x; r[1] = v.y; r[2] = v.z; r[3] = v.w;
        } else {
#pragma unroll
            for (int v = 0; v < VJ; ++v) r[v] = __ldg(L.rec + e + v);
        }
    }
    __device__ __forceinline__ uint32_t row(int v) const { return r[v] & 0xFFFFu; }
    __device__ __forceinline__ int gcode(int v) const { return (r[v] >> 16) & 0xFF; }
};

template <int VJ>
struct SmallEdges<FMT_I8_WIDE, VJ> {
    uint32_t k[VJ];
    uint16_t g[VJ];
    __device__ __forceinline__ void load(const DevLayer& L, size_t e) {
#pragma unroll
        for (int v = 0; v < VJ; ++v) {
            k[v] = L.idx ? __ldg(L.idx + e + v) : 0u;
            g[v] = __ldg(L.gb + e + v);
        }
    }
    __device__ __forceinline__ uint32_t row(int v) const { return k[v]; }
    __device__ __forceinline__ int gcode(int v) const { return g[v] & 0xFF; }
};

template <int VJ>
struct SmallEdges<FMT_F32, VJ> {
    uint32_t k[VJ];
    float g[VJ];
    __device__ __forceinline__ void load(const DevLayer& L, size_t e) {
#pragma unroll
        for (int v = 0; v < VJ; ++v) {
            k[v] = L.idx ? __ldg(L.idx + e + v) : 0u;
            g[v] = __ldg(L.gain + e + v);
        }
    }
};

template <int VJ>
struct SmallEdges<FMT_DENSE, VJ> {
    __device__ __forceinline__ void load(const DevLayer&, size_t) {}
};

template <int FMT, int VJ, int S, int RW>
__global__ void __launch_bounds__(256) k_fwd_small(FwdArgs a) {
    constexpr int W = 8;
    constexpr int JW = 32 * VJ;
    constexpr int R = W * RW;
    __shared__ int s_m[S][R];
    __shared__ float s_t[S][R];
    __shared__ float s_red[W][S][JW];
    __shared__ float s_lut[256];
    __shared__ int s_last;
    pdl_trigger();
    const DevLayer& L = a.L;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int jg = blockIdx.x, sg = blockIdx.z;
    const int j0 = jg * JW + lane * VJ;
    const int r0 = blockIdx.y * a.rows_per_cta;
    const int rend = min(L.in, r0 + a.rows_per_cta);
    const int s0 = sg * S;
    const int nS = min(S, a.B - s0);
    const bool jok = j0 < L.out;
    constexpr bool kI8 = FMT == FMT_I8_R32 || FMT == FMT_I8_WIDE;
    if constexpr (kI8) {
        for (int q = tid; q < 256; q += 256) s_lut[q] = L.lutf[q];
    }
    // 1. records of this warp's rows: independent of the previous kernel
    SmallEdges<FMT, VJ> ed[RW];
#pragma unroll
    for (int r = 0; r < RW; ++r) {
        const int i = r0 + warp * RW + r;
        if (jok && i < rend) ed[r].load(L, static_cast<size_t>(i) * L.out + j0);
    }
    // 2. brackets (produced by the previous kernel, or located inline)
    pdl_wait();
    if (a.prev_partial) reduce_prev_rows(a, r0, rend, s0, nS, S, R, &s_m[0][0], &s_t[0][0]);
    else for (int q = tid; q < S * R; q += 256) {
        const int sl = q / R, rl = q % R, i = r0 + rl;
        int m = 0;
        float t = 0.f;
        if (sl < nS && i < rend) {
            const size_t p = static_cast<size_t>(s0 + sl) * L.in + i;
            if (a.x) {
                fast_locate(L, a.x[p], a.err, m, t);
            } else {
                const size_t pt = static_cast<size_t>(i) * a.B + s0 + sl;  // input-major
                m = a.bm_in[pt];
                t = a.bt_in[pt];
            }
        }
        s_m[sl][rl] = m;
        s_t[sl][rl] = t;
    }
    __syncthreads();
    // 3. gather + interpolate + accumulate
    float acc[S][VJ];
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
        for (int v = 0; v < VJ; ++v) acc[s][v] = 0.f;
    if (jok) {
        const int G = L.G;
#pragma unroll
        for (int r = 0; r < RW; ++r) {
            const int rl = warp * RW + r;
            if (r0 + rl >= rend) break;
#pragma unroll
            for (int v = 0; v < VJ; ++v) {
                if (j0 + v >= L.out) break;
                float g = 1.f;
                if constexpr (kI8) g = s_lut[ed[r].gcode(v)];
                if constexpr (FMT == FMT_F32) g = ed[r].g[v];
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const int m = s_m[s][rl];
                    const float t = s_t[s][rl];
                    float c0, c1;
                    if constexpr (kI8) {
                        const uint32_t p = __ldg(L.pair8 + static_cast<size_t>(m) * L.K + ed[r].row(v));
                        c0 = i8lo(p);
                        c1 = i8hi(p);
                    } else if constexpr (FMT == FMT_F32) {
                        const float* row = L.cb32 + static_cast<size_t>(ed[r].k[v]) * G + m;
                        c0 = __ldg(row);
                        c1 = __ldg(row + 1);
                    } else {
                        c0 = dense_at(L, r0 + rl, j0 + v, m);
                        c1 = dense_at(L, r0 + rl, j0 + v, m + 1);
                    }
                    acc[s][v] = fmaf(g, fmaf(t, c1 - c0, c0), acc[s][v]);
                }
            }
        }
    }
    // 4. fixed-order reduction over warps, one partial per split
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
        for (int v = 0; v < VJ; ++v) s_red[warp][s][lane * VJ + v] = acc[s][v];
    __syncthreads();
    const size_t plane = static_cast<size_t>(a.B) * L.out;
    for (int q = tid; q < S * JW; q += 256) {
        const int s = q / JW, jl = q % JW, j = jg * JW + jl;
        if (s >= nS || j >= L.out) continue;
        float sum = 0.f;
#pragma unroll
        for (int w = 0; w < W; ++w) sum += s_red[w][s][jl];
        a.partial[blockIdx.y * plane + static_cast<size_t>(s0 + s) * L.out + j] = sum;
    }
    // 5. the last CTA of this (output tile, sample tile) finishes it
    if (!arrive_last(a.counters + jg * gridDim.z + sg, gridDim.y, &s_last)) return;
    finish_tile(a, gridDim.y, s0, nS, jg * JW, min(JW, L.out - jg * JW));
}

// ---------------------------------------------------------------------------
// k_fwd_planes (batch 1, int8 tables, non-final layer): at batch 1 every edge
// of input row i reads the same bracket m_i, i.e. only the pair plane
// P_m[k] = (c[k][m], c[k][m+1]) (K x 2 bytes: 128 KB at K=65536).  Each CTA
// (one per SM) takes a share of the rows of ONE bracket bucket, stages that
// plane into shared memory with a TMA bulk copy, and serves every codebook
// gather of its rows from shared memory instead of L1/L2 (where a random
// 2-byte gather costs a full 32-byte sector and an L1 wavefront).
// Rows -> buckets is a deterministic function of the bracket histogram
// (largest remainder), rows within a bucket are taken in ascending order,
// warps take rows round-robin: the fp32 summation order is fixed.  Output:
// one fp32 partial vector per CTA; the next layer reduces them.

template <int NV>  // 128-output groups per row (out <= 128*NV), 4 outputs per lane per group
__global__ void __launch_bounds__(256, 1) k_fwd_planes(FwdArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int kMaxB = 32;  // brackets (G-1) supported
    __shared__ int s_cnt[kMaxB];
    __shared__ int s_scan[256];
    __shared__ int s_bucket, s_lo, s_hi;
    __shared__ float s_lut[256];
    __shared__ __align__(8) uint64_t s_bar;
    const DevLayer& L = a.L;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int GP = L.G - 1;
    uint16_t* s_plane = reinterpret_cast<uint16_t*>(smem);
    const uint32_t plane_bytes = static_cast<uint32_t>(L.K) * 2u;
    int* s_rows = reinterpret_cast<int*>(smem + ((plane_bytes + 127u) & ~127u));
    pdl_trigger();
    s_lut[tid] = L.lutf[tid];
    if (tid < kMaxB) s_cnt[tid] = 0;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    pdl_wait();  // brackets of this layer's inputs
    // 1. histogram of brackets (order-free integer counts)
    const int per = (L.in + 255) / 256;  // rows per thread, contiguous
    const int i0 = tid * per, i1 = min(L.in, i0 + per);
    int mine[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) mine[q] = (q < i1 - i0) ? a.bm_in[i0 + q] : -1;
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; ++q)
        if (mine[q] >= 0) atomicAdd(&s_cnt[mine[q]], 1);
    __syncthreads();
    // 2. CTA -> bucket (same in every CTA): warp 0, lane b = bucket b.  Each
    //    non-empty bucket gets 1 + floor((P - nonempty) * n_b / in) CTAs
    //    (sum <= P; the few spare CTAs idle); CTA c serves the bucket whose
    //    CTA range contains c and an even share of its rows (ascending i).
    if (warp == 0) {
        const int P = gridDim.x;
        const int n = lane < GP ? s_cnt[lane] : 0;
        const int nonempty = __popc(__ballot_sync(0xFFFFFFFFu, n > 0));
        const int alloc = n > 0 ? 1 + static_cast<int>(static_cast<long long>(P - nonempty) * n / L.in) : 0;
        int incl = alloc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += y;
        }
        const int c = blockIdx.x;
        const unsigned hit = __ballot_sync(0xFFFFFFFFu, c >= incl - alloc && c < incl);
        if (lane == 0) s_bucket = hit ? (__ffs(hit) - 1) : GP;
        if (hit && lane == __ffs(hit) - 1) {
            const int q = c - (incl - alloc);
            s_lo = static_cast<int>(static_cast<long long>(n) * q / alloc);
            s_hi = static_cast<int>(static_cast<long long>(n) * (q + 1) / alloc);
        }
        if (!hit && lane == 0) s_lo = s_hi = 0;
        __syncwarp();
        if (lane == 0 && hit) {  // 3. stage plane b: TMA bulk copies, 32 KB each
            const int b = __ffs(hit) - 1;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&s_bar)),
                         "r"(plane_bytes)
                         : "memory");
            const char* src = reinterpret_cast<const char*>(L.pair8 + static_cast<size_t>(b) * L.K);
            for (uint32_t off = 0; off < plane_bytes; off += 32768u) {
                const uint32_t len = min(32768u, plane_bytes - off);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_u32(smem + off)),
                    "l"(src + off), "r"(len), "r"(smem_u32(&s_bar))
                    : "memory");
            }
        }
    }
    __syncthreads();
    const int bucket = s_bucket, lo = s_lo, hi = s_hi;
    // 4. my rows: rank within the bucket = exclusive scan of per-thread counts
    int cnt = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) cnt += mine[q] == bucket;
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_scan[warp] = incl;
    __syncthreads();
    int wbase = 0;
    for (int w = 0; w < warp; ++w) wbase += s_scan[w];
    int rank = wbase + incl - cnt;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        if (mine[q] == bucket) {
            if (rank >= lo && rank < hi) s_rows[rank - lo] = i0 + q;
            ++rank;
        }
    }
    __syncthreads();
    const int nrows = hi - lo;
    // 5. stream this CTA's rows: warp w takes rows w, w+8, ...; records are
    //    prefetched one row ahead; codebook pairs come from the staged plane.
    float acc[NV][4];
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[v][e] = 0.f;
    uint4 rec[NV], nxt[NV];
    auto load_row = [&](int rr, uint4* dst) {
        const int i = s_rows[rr];
        const uint32_t* base = L.rec + static_cast<size_t>(i) * L.out;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const int j = v * 128 + lane * 4;
            dst[v] = j < L.out ? __ldg(reinterpret_cast<const uint4*>(base + j)) : make_uint4(0, 0, 0, 0);
        }
    };
    if (warp < nrows) load_row(warp, rec);
    if (bucket < GP) {
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(smem_u32(&s_bar))
                : "memory");
        }
    }
    for (int rr = warp; rr < nrows; rr += 8) {
        const bool more = rr + 8 < nrows;
        if (more) load_row(rr + 8, nxt);
        const float t = a.bt_in[s_rows[rr]];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const uint32_t r4[4] = {rec[v].x, rec[v].y, rec[v].z, rec[v].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const uint32_t p = s_plane[r4[e] & 0xFFFFu];
                const float c0 = i8lo(p), c1 = i8hi(p);
                acc[v][e] = fmaf(s_lut[(r4[e] >> 16) & 0xFF], fmaf(t, c1 - c0, c0), acc[v][e]);
            }
        }
        if (more) {
#pragma unroll
            for (int v = 0; v < NV; ++v) rec[v] = nxt[v];
        }
    }
    // 6. fixed-order reduction over warps (plane region reused), one partial per CTA
    __syncthreads();
    float* s_red = reinterpret_cast<float*>(smem);  // [8][128*NV]
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        const int j = v * 128 + lane * 4;
        *reinterpret_cast<float4*>(s_red + warp * (128 * NV) + j) =
            make_float4(acc[v][0], acc[v][1], acc[v][2], acc[v][3]);
    }
    __syncthreads();
    for (int j = tid; j < L.out; j += 256) {
        float sum = 0.f;
#pragma unroll
        for (int w = 0; w < 8; ++w) sum += s_red[w * (128 * NV) + j];
        a.partial[static_cast<size_t>(blockIdx.x) * L.out + j] = sum;
    }
}

size_t planes_smem(const DevLayer& L, int nv) {
    const size_t plane = (static_cast<size_t>(L.K) * 2 + 127) / 128 * 128;
    const size_t red = static_cast<size_t>(8) * 128 * nv * sizeof(float);  // [8 warps][128*NV]
    return (plane + static_cast<size_t>(L.in) * sizeof(int)) > red ? plane + static_cast<size_t>(L.in) * sizeof(int)
                                                                     : red;
}

// ---------------------------------------------------------------------------
// k_fwd_large: samples in lanes.  CTA = 8 warps = 4 sample-warps (128
// samples) x 2 output-warps (VJ outputs each) -> tile 128 samples x 2*VJ
// outputs, over a split of the input rows processed in chunks of IC rows.
// Per chunk every edge of the tile is decoded ONCE (record + 16-byte padded
// codebook row) into shared memory as gained pairs (g*c[m], g*(c[m+1]-c[m])),
// m = 0..G-2; a thread then evaluates its VJ outputs for its sample with one
// broadcast LDS.64 per edge-sample (lanes of a warp hit <= G-1 distinct
// pairs of one edge) at an immediate offset when G is a compile-time
// constant (GPT > 0).  A row's bracket and t arrive as one 8-byte word.
// Staging of chunk c+1 is prefetched into registers while chunk c is
// computed.  int8 tables, G <= 16.

constexpr int kLgSW = 4;                // sample-warps
constexpr int kLgJW = 2;                // output-warps
constexpr int kLgS = 32 * kLgSW;        // samples per CTA

template <int FMT, int EPT, int GPT, int VJ>  // EPT: staged edges per thread per chunk; GPT: G-1 or 0
__global__ void __launch_bounds__(256) k_fwd_large(FwdArgs a) {
    constexpr int kJ = kLgJW * VJ;       // outputs per CTA
    constexpr int IC = EPT * 256 / kJ;   // input rows per chunk
    extern __shared__ __align__(128) unsigned char smem[];
    const DevLayer& L = a.L;
    const int G = L.G;
    const int GP = GPT > 0 ? GPT : G - 1;
    // layout: pairs[2][IC][kJ][GP] float2 | mt[2][IC][kLgS] {m, t} | lut[256]
    float2* s_pair = reinterpret_cast<float2*>(smem);
    const size_t pair_buf = static_cast<size_t>(IC) * kJ * GP;
    int2* s_mt = reinterpret_cast<int2*>(s_pair + 2 * pair_buf);
    float* s_lut = reinterpret_cast<float*>(s_mt + 2 * IC * kLgS);
    __shared__ int s_last;
    pdl_trigger();

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int sw = warp % kLgSW, jw = warp / kLgSW;
    const int jbase = blockIdx.x * kJ;
    const int s0 = blockIdx.z * kLgS;
    const int nS = min(kLgS, a.B - s0);
    const int r0 = blockIdx.y * a.rows_per_cta;
    const int rend = min(L.in, r0 + a.rows_per_cta);
    const int nchunks = (rend - r0 + IC - 1) / IC;
    for (int q = tid; q < 256; q += 256) s_lut[q] = L.lutf[q];

    // staging assignment: edge slot q = tid + 256*u -> (row il, output jl)
    uint32_t rec[EPT];
    uint4 row[EPT];
    unsigned ok = 0;  // bit u: staged edge slot u exists
    auto load_recs = [&](int c) {
        ok = 0;
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            const int q = tid + 256 * u, il = q / kJ, jl = q % kJ;
            const int i = r0 + c * IC + il, j = jbase + jl;
            if (i < rend && j < L.out) {
                ok |= 1u << u;
                const size_t e = static_cast<size_t>(i) * L.out + j;
                if constexpr (FMT == FMT_I8_R32) {
                    rec[u] = __ldg(L.rec + e);
                } else {
                    const uint32_t k = L.idx ? __ldg(L.idx + e) : 0u;
                    rec[u] = __ldg(L.gb + e);  // gain code in bits 0-7
                    row[u].x = k;              // row index parked until load_rows
                }
            }
        }
    };
    auto load_rows = [&]() {
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            if (!(ok & (1u << u))) continue;
            uint32_t k;
            if constexpr (FMT == FMT_I8_R32) k = rec[u] & 0xFFFFu; else k = row[u].x;
            row[u] = __ldg(reinterpret_cast<const uint4*>(L.cb8 + static_cast<size_t>(k) * L.rs));
        }
    };
    auto store_pairs = [&](int buf) {
        float2* dst = s_pair + buf * pair_buf;
#pragma unroll
        for (int u = 0; u < EPT; ++u) {
            const int q = tid + 256 * u, il = q / kJ, jl = q % kJ;
            float2* d = dst + (static_cast<size_t>(il) * kJ + jl) * GP;
            float g = 0.f;  // absent edges stage zeros
            if (ok & (1u << u)) {
                int gc;
                if constexpr (FMT == FMT_I8_R32) gc = (rec[u] >> 16) & 0xFF; else gc = rec[u] & 0xFF;
                g = s_lut[gc];
            }
            const uint64_t lo = row[u].x | (static_cast<uint64_t>(row[u].y) << 32);
            const uint64_t hi = row[u].z | (static_cast<uint64_t>(row[u].w) << 32);
            auto code = [&](int b) -> float {  // static b after unrolling
                const uint64_t w = b < 8 ? (lo >> (8 * b)) : (hi >> (8 * (b - 8)));
                return static_cast<float>(static_cast<int8_t>(w & 0xFF));
            };
            float prev = g * code(0);
#pragma unroll
            for (int m = 0; m < 15; ++m) {
                if (m < GP) {
                    const float nxt = g * code(m + 1);
                    d[m] = make_float2(prev, nxt - prev);
                    prev = nxt;
                }
            }
        }
    };
    auto store_brackets = [&](int c, int buf) {
        for (int q = tid; q < IC * kLgS; q += 256) {
            const int il = q / kLgS, sl = q % kLgS, i = r0 + c * IC + il;
            int m = 0;
            float t = 0.f;
            if (sl < nS && i < rend) {
                const size_t p = static_cast<size_t>(i) * a.B + s0 + sl;  // input-major: coalesced
                m = a.bm_in[p];
                t = a.bt_in[p];
            }
            s_mt[(buf * IC + il) * kLgS + sl] = make_int2(m, __float_as_int(t));
        }
    };

    float acc[VJ];
#pragma unroll
    for (int v = 0; v < VJ; ++v) acc[v] = 0.f;
    const int sl = sw * 32 + lane;

    if (nchunks > 0) {
        load_recs(0);
        __syncthreads();  // s_lut visible
        load_rows();
        pdl_wait();
        store_pairs(0);
        store_brackets(0, 0);
        if (nchunks > 1) load_recs(1);
        __syncthreads();
    } else {
        pdl_wait();
    }
#pragma unroll 1
    for (int c = 0; c < nchunks; ++c) {
        const int buf = c & 1;
        const bool more = c + 1 < nchunks;
        if (more) load_rows();  // rows of chunk c+1 fly while chunk c is computed
        const float2* P = s_pair + buf * pair_buf + static_cast<size_t>(jw * VJ) * GP;
        const int2* MT = s_mt + buf * IC * kLgS + sl;
        const int nrow = min(IC, rend - (r0 + c * IC));
#pragma unroll 2
        for (int il = 0; il < nrow; ++il) {
            const int2 mt = MT[il * kLgS];
            const float t = __int_as_float(mt.y);
            const float2* e = P + static_cast<size_t>(il) * kJ * GP + mt.x;
#pragma unroll
            for (int v = 0; v < VJ; ++v) {
                const float2 p = e[v * GP];
                acc[v] += fmaf(t, p.y, p.x);
            }
        }
        if (more) {
            store_pairs(buf ^ 1);
            store_brackets(c + 1, buf ^ 1);
            if (c + 2 < nchunks) load_recs(c + 2);
        }
        __syncthreads();
    }
    // one partial per (split, sample, output): each thread owns distinct entries
    const size_t plane = static_cast<size_t>(a.B) * L.out;
    if (sl < nS) {
#pragma unroll
        for (int v = 0; v < VJ; ++v) {
            const int j = jbase + jw * VJ + v;
            if (j < L.out) a.partial[blockIdx.y * plane + static_cast<size_t>(s0 + sl) * L.out + j] = acc[v];
        }
    }
    if (!arrive_last(a.counters + blockIdx.x * gridDim.z + blockIdx.z, gridDim.y, &s_last)) return;
    finish_tile(a, gridDim.y, s0, nS, jbase, min(kJ, L.out - jbase));
}

// ---------------------------------------------------------------------------
// K2 exact: one split (ascending i), every double op in the reference's
// order with explicit _rn intrinsics (no FMA):
//   compressed: y += (g*c0 + b)*w0 + (g*c1 + b)*t      lutham.cpp:810
//   dense:      y += c0*w0 + c1*t                      lutham.cpp:787-788

template <int FMT>
struct Edge;

template <>
struct Edge<FMT_I8_R32> {
    const int8_t* row;
    uint32_t r;
    __device__ __forceinline__ void load(const DevLayer& L, size_t e) {
        r = __ldg(L.rec + e);
        row = L.cb8 + static_cast<size_t>(r & 0xFFFFu) * L.rs;
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
        row = L.cb8 + static_cast<size_t>(k) * L.rs;
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
    int i, j;
    __device__ __forceinline__ void load(const DevLayer& L, size_t e) {
        i = static_cast<int>(e / static_cast<size_t>(L.out));
        j = static_cast<int>(e - static_cast<size_t>(i) * L.out);
    }
};

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
#pragma unroll 4
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
                } else if constexpr (FMT == FMT_DENSE) {
                    c0 = static_cast<double>(dense_at(L, ed.i, ed.j, m));
                    c1 = static_cast<double>(dense_at(L, ed.i, ed.j, m + 1));
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
// Exact mode at small batch, in two passes.  k_gather_exact gives each
// (sample, output) one thread that walks the inputs in order: at batch 1 that
// is ~1.4k threads chasing dependent record -> codebook loads, far below the
// machine.  Bitwise equality only needs each output's SUM in input order, so:
//   k_exact_terms: every (input, output, sample) term in parallel, with
//     exactly k_gather_exact's operations (lutham.cpp:810, no contraction),
//     for a block of inputs, into a scratch buffer;
//   k_exact_sum:   per (sample, output), acc = acc + term in input order over
//     the block (coalesced across outputs), acc carried across blocks.
template <int FMT>
__global__ void __launch_bounds__(256) k_exact_terms(DevLayer L, int B, const int* __restrict__ bm,
                                                     const double* __restrict__ btd, int i0, int ni,
                                                     double* __restrict__ terms) {
    // one thread per (sample group of kExS, input, output): the record is
    // loaded once per group, the groups re-read it from L2 (groups of 16
    // measured faster than 4 or 8: batch 8 171 -> 163 us, 128 2.30 -> 2.12 ms)
    constexpr int kExS = 16;
    const int ng = (B + kExS - 1) / kExS, njb = (L.out + 31) >> 5;
    const size_t n = static_cast<size_t>(ni) * L.out, nt = n * ng;
    for (size_t qq = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; qq < nt;
         qq += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int sg = static_cast<int>(qq / n);
        const size_t q = qq - static_cast<size_t>(sg) * n;
        const int il = static_cast<int>(q / L.out), j = static_cast<int>(q - static_cast<size_t>(il) * L.out);
        const int i = i0 + il;
        Edge<FMT> ed;
        ed.load(L, static_cast<size_t>(i) * L.out + j);
        double g = 0.0, b = 0.0;
        if constexpr (FMT == FMT_I8_R32 || FMT == FMT_I8_WIDE) {
            g = __ldg(L.lutd + ed.gcode());
            b = __dmul_rn(static_cast<double>(ed.bcode()), L.bs);
        }
        if constexpr (FMT == FMT_F32) {
            g = static_cast<double>(ed.g);
            b = static_cast<double>(ed.b);
        }
        const int s1 = min(B, (sg + 1) * kExS);
        for (int sm = sg * kExS; sm < s1; ++sm) {
            const int m = __ldg(bm + static_cast<size_t>(sm) * L.in + i);
            const double t = __ldg(btd + static_cast<size_t>(sm) * L.in + i);
            const double w0 = __dsub_rn(1.0, t);
            double c0, c1, term;
            if constexpr (FMT == FMT_I8_R32 || FMT == FMT_I8_WIDE) {
                c0 = __dmul_rn(static_cast<double>(__ldg(ed.row + m)), L.cs);
                c1 = __dmul_rn(static_cast<double>(__ldg(ed.row + m + 1)), L.cs);
            } else if constexpr (FMT == FMT_DENSE) {
                c0 = static_cast<double>(dense_at(L, ed.i, ed.j, m));
                c1 = static_cast<double>(dense_at(L, ed.i, ed.j, m + 1));
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
            // [sample][output block of 32][input][32]: a sum block's chunk of
            // inputs is one contiguous run for a bulk copy
            terms[((static_cast<size_t>(sm) * njb + (j >> 5)) * ni + il) * 32 + (j & 31)] = term;
        }
    }
}

// int8 layers, all inputs in one term block: the terms in the order of the
// inputs' brackets.  Every edge of input i at bracket m reads the pair plane
// m (c[k][m] | c[k][m+1] << 8, the same int8 codes as the codebook row), so a
// CTA working through inputs of one bracket keeps that 128 KB plane in L1
// instead of pulling a 32-byte sector of a random codebook row per edge from
// L2.  k_exact_locate_order brackets the inputs and sorts them by bracket (a
// counting sort; the order within a bracket is irrelevant: terms land at
// their input's slot).  Batch 1 only: from batch 2 the sample-grouped
// kernel, which decodes each record once for up to 16 samples, is faster.
// Batch 1: the layer's exact brackets (k_locate_input's bracket_of) and
// their counting sort in one block, one launch instead of two.
__global__ void __launch_bounds__(1024) k_exact_locate_order(const double* __restrict__ x, DevLayer L,
                                                             int* __restrict__ bm, float* __restrict__ btf,
                                                             double* __restrict__ btd, int* __restrict__ err,
                                                             int* __restrict__ order) {
    __shared__ int cnt[64], off[64];
    const int nb = L.G - 1, in = L.in;
    if (threadIdx.x < 64) cnt[threadIdx.x] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < in; i += blockDim.x) {
        int m;
        double t;
        bracket_of(L.lo, L.hi, L.G, L.dx, x[i], err, m, t);
        btf[i] = static_cast<float>(t);
        btd[i] = t;
        bm[i] = m;
        atomicAdd(&cnt[min(max(m, 0), nb - 1)], 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int a = 0;
        for (int m = 0; m < nb; ++m) {
            off[m] = a;
            a += cnt[m];
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < in; i += blockDim.x) {
        const int pos = atomicAdd(&off[min(max(bm[i], 0), nb - 1)], 1);
        order[pos] = i;
    }
}

__global__ void __launch_bounds__(256) k_exact_terms_planes(DevLayer L, int B, const int* __restrict__ bm,
                                                            const double* __restrict__ btd,
                                                            const int* __restrict__ order,
                                                            double* __restrict__ terms) {
    const int njb = (L.out + 31) >> 5;
    const size_t per_s = static_cast<size_t>(L.in) * L.out, nt = per_s * B;
    for (size_t qq = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; qq < nt;
         qq += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int sm = static_cast<int>(qq / per_s);
        const size_t rem = qq - static_cast<size_t>(sm) * per_s;
        const int p = static_cast<int>(rem / L.out), j = static_cast<int>(rem - static_cast<size_t>(p) * L.out);
        const int i = __ldg(order + static_cast<size_t>(sm) * L.in + p);
        const uint32_t r = __ldg(L.rec + static_cast<size_t>(i) * L.out + j);
        const int m = __ldg(bm + static_cast<size_t>(sm) * L.in + i);
        const double t = __ldg(btd + static_cast<size_t>(sm) * L.in + i);
        const uint32_t pr = __ldg(L.pair8 + static_cast<size_t>(m) * L.K + (r & 0xFFFFu));
        // exactly k_exact_terms' operations (lutham.cpp:810, no contraction)
        const double g = __ldg(L.lutd + ((r >> 16) & 0xFFu));
        const double b = __dmul_rn(static_cast<double>(static_cast<int8_t>(r >> 24)), L.bs);
        const double w0 = __dsub_rn(1.0, t);
        const double c0 = __dmul_rn(static_cast<double>(static_cast<int8_t>(pr & 0xFFu)), L.cs);
        const double c1 = __dmul_rn(static_cast<double>(static_cast<int8_t>(pr >> 8)), L.cs);
        const double term = __dadd_rn(__dmul_rn(__dadd_rn(__dmul_rn(g, c0), b), w0),
                                      __dmul_rn(__dadd_rn(__dmul_rn(g, c1), b), t));
        terms[((static_cast<size_t>(sm) * njb + (j >> 5)) * L.in + i) * 32 + (j & 31)] = term;
    }
}

// Each (sample, output) chain is a strictly ordered run of dependent adds (a
// dependent DADD is ~8 clocks, tools/micro/dadd_lat.cu), and at small batch
// there are few chains, so the terms must stream in far ahead of the adds.
// One warp per (sample, block of 32 outputs); its chunks of kExKc inputs x 32
// outputs are contiguous 32 KB runs, so lane 0 keeps kExSt of them in flight
// with TMA bulk copies on per-stage mbarriers, and each lane adds its column
// from shared memory.  With 4 stages one warp has ~128 KB in flight; long
// chunks keep the per-chunk wait/refill overhead off the add chain (8 KB
// chunks: 89 us at batch 1, 16 KB: 79, 32 KB: 75).
constexpr int kExKc = 128;

template <int kExSt>
__global__ void __launch_bounds__(32) k_exact_sum(int out, int ni, const double* __restrict__ terms,
                                                  double* __restrict__ acc, double* __restrict__ y, int first,
                                                  int last) {
    extern __shared__ __align__(128) double sbuf[];  // [kExSt][kExKc][32]
    __shared__ __align__(8) uint64_t bar[kExSt];
    const int lane = threadIdx.x;
    const int njb = (out + 31) >> 5;
    const int sm = blockIdx.x / njb, j = (blockIdx.x - sm * njb) * 32 + lane;
    const bool act = j < out;
    const double* tb = terms + static_cast<size_t>(blockIdx.x) * ni * 32;
    const int nch = (ni + kExKc - 1) / kExKc;
    auto issue = [&](int c) {
        if (lane == 0 && c < nch) {
            const int st = c % kExSt;
            const uint32_t bytes = static_cast<uint32_t>(min(kExKc, ni - c * kExKc)) * 32u * 8u;
            dev::mbar_expect_tx(&bar[st], bytes);
            dev::bulk_g2s(sbuf + static_cast<size_t>(st) * kExKc * 32, tb + static_cast<size_t>(c) * kExKc * 32,
                          bytes, &bar[st]);
        }
    };
    if (lane == 0) {
#pragma unroll
        for (int st = 0; st < kExSt; ++st) dev::mbar_init(&bar[st], 1);
    }
    __syncwarp();
#pragma unroll
    for (int c = 0; c < kExSt; ++c) issue(c);
    const size_t q = static_cast<size_t>(sm) * out + j;
    double a = (act && !first) ? acc[q] : 0.0;  // the reference's y starts at 0.0 (0.0 + -0.0 = +0.0 matters)
    for (int c = 0; c < nch; ++c) {
        const int st = c % kExSt;
        dev::mbar_wait(&bar[st], static_cast<unsigned>(c / kExSt) & 1u);
        const double* src = sbuf + static_cast<size_t>(st) * kExKc * 32 + lane;
        const int rn = min(kExKc, ni - c * kExKc);
        if (rn == kExKc) {
#pragma unroll
            for (int r = 0; r < kExKc; ++r) a = __dadd_rn(a, src[r * 32]);
        } else {
            for (int r = 0; r < rn; ++r) a = __dadd_rn(a, src[r * 32]);
        }
        __syncwarp();      // every lane is done with this stage ...
        issue(c + kExSt);  // ... before it is refilled
    }
    if (!act) return;
    if (last) y[q] = a;
    else acc[q] = a;
}

// the in-order sums of one term block (first: acc starts at 0, last: write y)
void launch_exact_sum(int out, int B, int ni, const double* terms, double* acc, double* y, cudaStream_t s,
                      int first = 1, int last = 1) {
    static const bool attr = [] {  // 64 KB of dynamic shared memory and more (opt-in above 48 KB)
        return cudaFuncSetAttribute(k_exact_sum<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    4 * kExKc * 32 * 8) == cudaSuccess &&
               cudaFuncSetAttribute(k_exact_sum<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    2 * kExKc * 32 * 8) == cudaSuccess;
    }();
    (void)attr;
    const int nb = B * ((out + 31) / 32);
    if (nb <= 2 * 148) k_exact_sum<4><<<nb, 32, 4 * kExKc * 32 * 8, s>>>(out, ni, terms, acc, y, first, last);
    else k_exact_sum<2><<<nb, 32, 2 * kExKc * 32 * 8, s>>>(out, ni, terms, acc, y, first, last);
}

template <int FMT>
int dispatch_exact_split(const DevLayer& L, int B, const int* bm, const double* btd, double* y, double* terms,
                         size_t term_doubles, double* acc, cudaStream_t s) {
    const size_t outp = static_cast<size_t>((L.out + 31) / 32) * 32;  // the blocked term layout pads outputs
    const int per = static_cast<int>(std::max<size_t>(1, term_doubles / (static_cast<size_t>(B) * outp)));
    int launches = 0;
    for (int i0 = 0; i0 < L.in; i0 += per) {
        const int ni = std::min(per, L.in - i0);
        const size_t n = static_cast<size_t>(ni) * L.out * ((B + 15) / 16);
        const int blocks = static_cast<int>(std::min<size_t>((n + 255) / 256, 148ull * 64));
        k_exact_terms<FMT><<<blocks > 0 ? blocks : 1, 256, 0, s>>>(L, B, bm, btd, i0, ni, terms);
        launch_exact_sum(L.out, B, ni, terms, acc, y, s, i0 == 0 ? 1 : 0, i0 + ni >= L.in ? 1 : 0);
        launches += 2;
    }
    return launches;
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

// ---- launch helpers ----------------------------------------------------------

template <typename K, typename... Args>
void launch_ex(K kernel, dim3 grid, dim3 block, size_t smem, bool pdl, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cuda_check(cudaLaunchKernelEx(&cfg, kernel, args...), "kernel launch");
}

template <int FMT, int VJ, int S>
void dispatch_small_rw(const FwdArgs& a, const LaunchCfg& c, bool pdl, cudaStream_t s) {
    const dim3 grid(c.jt, c.nsplit, c.st);
    if (c.rw == 8) launch_ex(k_fwd_small<FMT, VJ, S, 8>, grid, dim3(256), 0, pdl, s, a);
    else if (c.rw == 4) launch_ex(k_fwd_small<FMT, VJ, S, 4>, grid, dim3(256), 0, pdl, s, a);
    else launch_ex(k_fwd_small<FMT, VJ, S, 1>, grid, dim3(256), 0, pdl, s, a);
}

template <int FMT, int VJ>
void dispatch_small_s(const FwdArgs& a, const LaunchCfg& c, bool pdl, cudaStream_t s) {
    switch (c.spt) {
        case 1: dispatch_small_rw<FMT, VJ, 1>(a, c, pdl, s); break;
        case 2: dispatch_small_rw<FMT, VJ, 2>(a, c, pdl, s); break;
        case 4: dispatch_small_rw<FMT, VJ, 4>(a, c, pdl, s); break;
        default: dispatch_small_rw<FMT, VJ, 8>(a, c, pdl, s); break;
    }
}

template <int FMT, int VJ, int S>
void dispatch_exact_spt(const DevLayer& L, const LaunchCfg& c, int B, const int* bm,
                        const double* btd, double* y, cudaStream_t s) {
    (void)VJ;
    dim3 grid(c.jt, c.st, 1);
    switch (c.tj) {
        case 32: k_gather_exact<FMT, 32, S><<<grid, kThreads, 0, s>>>(L, B, bm, btd, y); break;
        case 64: k_gather_exact<FMT, 64, S><<<grid, kThreads, 0, s>>>(L, B, bm, btd, y); break;
        default: k_gather_exact<FMT, 128, S><<<grid, kThreads, 0, s>>>(L, B, bm, btd, y); break;
    }
}

template <int FMT>
void dispatch_exact(const DevLayer& L, const LaunchCfg& c, int B, const int* bm, const double* btd,
                    double* y, cudaStream_t s) {
    switch (c.spt) {
        case 1: dispatch_exact_spt<FMT, 0, 1>(L, c, B, bm, btd, y, s); break;
        case 2: dispatch_exact_spt<FMT, 0, 2>(L, c, B, bm, btd, y, s); break;
        case 4: dispatch_exact_spt<FMT, 0, 4>(L, c, B, bm, btd, y, s); break;
        default: dispatch_exact_spt<FMT, 0, 8>(L, c, B, bm, btd, y, s); break;
    }
}

size_t large_smem(int G, int ept, int vj) {
    const size_t kj = static_cast<size_t>(kLgJW) * vj;
    const size_t ic = static_cast<size_t>(ept) * 256 / kj;
    return 2 * ic * kj * (G - 1) * sizeof(float2) + 2 * ic * kLgS * sizeof(int2) + 256 * sizeof(float);
}

// Shared-memory budget of one large-batch CTA: two fit per SM.
constexpr size_t kLgSmemBudget = 110 * 1024;

template <int FMT, int EPT, int VJ>
void (*large_kernel_g(int G))(FwdArgs) {
    return G == 10 ? k_fwd_large<FMT, EPT, 9, VJ> : k_fwd_large<FMT, EPT, 0, VJ>;
}

template <int FMT>
void (*large_kernel(int G, int ept, int vj))(FwdArgs) {
    if (vj == 32) return ept == 2 ? large_kernel_g<FMT, 2, 32>(G) : large_kernel_g<FMT, 1, 32>(G);
    return ept == 2 ? large_kernel_g<FMT, 2, 16>(G) : large_kernel_g<FMT, 1, 16>(G);
}

}  // namespace

// ---------------------------------------------------------------------------

LaunchCfg choose_cfg(const DevLayer& L, int B, bool exact, int num_sms, bool allow_planes) {
    LaunchCfg c{};
    const int sms = num_sms > 0 ? num_sms : 148;
    if (!exact && allow_planes && B == 1 && L.fmt == FMT_I8_R32 && L.out % 4 == 0 && L.out <= 1536 &&
        L.in <= 4096 && L.K % 8 == 0 && static_cast<size_t>(L.K) * 2 <= 160 * 1024 && L.G - 1 <= 32 &&
        static_cast<long long>(L.in) * L.out >= 256LL * 1024) {
        c.kind = 2;
        const int groups = (L.out + 127) / 128;
        c.vj = groups <= 2 ? 2 : (groups <= 4 ? 4 : (groups <= 8 ? 8 : 12));
        c.nsplit = sms;  // one CTA per SM, each a share of one bracket bucket
        c.jt = 1;
        c.st = 1;
        c.ichunk = L.in;
        c.smem = planes_smem(L, c.vj);
        return c;
    }
    if (exact) {
        c.tj = L.out <= 32 ? 32 : (L.out <= 64 ? 64 : 128);
        c.spt = B >= 8 ? 8 : (B >= 4 ? 4 : (B >= 2 ? 2 : 1));
        const int sc = (kThreads / c.tj) * c.spt;
        c.jt = (L.out + c.tj - 1) / c.tj;
        c.st = (B + sc - 1) / sc;
        c.nsplit = 1;
        c.ichunk = L.in;
        return c;
    }
    static const int gemm_min_out = [] {
        const char* e = std::getenv("SKAN_GEMM_MIN_OUT");  // experiment: narrowest layer routed to the GEMM
        return e ? std::atoi(e) : 16;
    }();
    // (up to batch 512: above it the staged brackets leave few rows per CTA and
    // the split partials grow with the batch; the generic kernels take over)
    // (int8 layers up to batch 128: at 256 the one-tile GEMM and its 88-plane
    // reduction beat the narrow kernel's 148 planes, 98 vs 101 us)
    static const int i8_maxb = [] {
        const char* e = std::getenv("SKAN_NARROW_I8_MAXB");  // experiment: largest batch for narrow int8 layers
        return e ? std::atoi(e) : 128;
    }();
    if (B >= g_gemm_min_batch && B <= (L.fmt == FMT_DENSE ? 512 : i8_maxb) && dense_narrow_ok(L))
        return dense_narrow_cfg(L, B, sms);
    if (B >= g_gemm_min_batch && L.out >= gemm_min_out && gemm_supported(L)) return gemm_cfg(L, B, sms);  // tensor cores
    const bool i8 = L.fmt == FMT_I8_R32 || L.fmt == FMT_I8_WIDE;
    if (i8 && L.G <= 16 && B >= 64) {
        // samples in lanes: tile 128 samples x (32 or 64) outputs x split of the rows
        c.kind = 1;
        c.tj = 32;                        // outputs per CTA (64 measured slower: more staging conflicts)
        c.spt = c.tj / kLgJW;             // outputs per thread (VJ)
        int ept = 2;
        while (ept > 1 && large_smem(L.G, ept, c.spt) > kLgSmemBudget) ept >>= 1;
        c.vj = ept;
        c.ic = ept * 256 / c.tj;
        c.jt = (L.out + c.tj - 1) / c.tj;
        c.st = (B + kLgS - 1) / kLgS;
        const long long base = static_cast<long long>(c.jt) * c.st;
        long long ns = (2LL * sms + base - 1) / base;  // ~2 CTAs per SM, one wave
        if (ns > 16) ns = 16;                          // bounds the finisher's work (last CTA per tile)
        const long long maxns = (L.in + c.ic - 1) / c.ic;
        ns = ns < 1 ? 1 : (ns > maxns ? maxns : ns);
        const int chunks = static_cast<int>((L.in + c.ic - 1) / c.ic);
        const int per = (chunks + static_cast<int>(ns) - 1) / static_cast<int>(ns);
        c.ichunk = per * c.ic;
        c.nsplit = (L.in + c.ichunk - 1) / c.ichunk;
        c.smem = large_smem(L.G, ept, c.spt);
        return c;
    }
    // rows in warps: 8 warps x rw rows, 32*vj outputs, S samples
    c.kind = 0;
    c.vj = (L.fmt == FMT_I8_R32 && L.out % 4 == 0 && L.out >= 128) ? 4 : 1;
    c.spt = B >= 8 ? 8 : (B >= 4 ? 4 : (B >= 2 ? 2 : 1));
    c.tj = 32 * c.vj;
    c.jt = (L.out + c.tj - 1) / c.tj;
    c.st = (B + c.spt - 1) / c.spt;
    // rows per warp: 8 (deepest record prefetch, fewest splits) unless that
    // leaves SMs idle
    const long long tiles = static_cast<long long>(c.jt) * c.st;
    c.rw = 8;
    for (int rw : {8, 4, 1}) {
        c.rw = rw;
        const long long ctas = tiles * ((L.in + 8LL * rw - 1) / (8LL * rw));
        if (ctas >= sms) break;
    }
    c.ichunk = 8 * c.rw;
    c.nsplit = (L.in + c.ichunk - 1) / c.ichunk;
    return c;
}

void launch_locate_input(const double* x, int n_rows, int width, const DevLayer& L, int* bm,
                         float* btf, double* btd, int* err, cudaStream_t s, bool input_major) {
    const long long n = static_cast<long long>(n_rows) * width;
    if (n == 0) return;
    if (input_major && !btd) {
        k_locate_transpose<<<dim3((width + 31) / 32, (n_rows + 31) / 32), 1024, 0, s>>>(x, n_rows, width, L, bm, btf,
                                                                                      err);
        return;
    }
    k_locate_input<<<grid_for(n, 256), 256, 0, s>>>(x, n, L, bm, btf, btd, err, width, input_major ? n_rows : 0);
}

int launch_fwd_fast(const FwdArgs& a, const LaunchCfg& c, bool pdl, cudaStream_t s) {
    if (c.kind == 4) return launch_layer_gemm(a, c, pdl, s);
    if (c.kind == 5) return launch_dense_narrow(a, c, pdl, s);
    if (c.kind == 2) {
        void (*k)(FwdArgs);
        switch (c.vj) {
            case 2: k = k_fwd_planes<2>; break;
            case 4: k = k_fwd_planes<4>; break;
            case 8: k = k_fwd_planes<8>; break;
            default: k = k_fwd_planes<12>; break;
        }
        ensure_smem(k, c.smem);
        launch_ex(k, dim3(c.nsplit), dim3(256), c.smem, pdl, s, a);
        return 1;
    }
    if (c.kind == 1) {
        void (*k)(FwdArgs) = a.L.fmt == FMT_I8_R32 ? large_kernel<FMT_I8_R32>(a.L.G, c.vj, c.spt)
                                                    : large_kernel<FMT_I8_WIDE>(a.L.G, c.vj, c.spt);
        ensure_smem(k, c.smem);
        launch_ex(k, dim3(c.jt, c.nsplit, c.st), dim3(256), c.smem, pdl, s, a);
        return 1;
    }
    switch (a.L.fmt) {
        case FMT_I8_R32:
            if (c.vj == 4) dispatch_small_s<FMT_I8_R32, 4>(a, c, pdl, s);
            else dispatch_small_s<FMT_I8_R32, 1>(a, c, pdl, s);
            break;
        case FMT_I8_WIDE: dispatch_small_s<FMT_I8_WIDE, 1>(a, c, pdl, s); break;
        case FMT_F32: dispatch_small_s<FMT_F32, 1>(a, c, pdl, s); break;
        default: dispatch_small_s<FMT_DENSE, 1>(a, c, pdl, s); break;
    }
    return 1;
}

int launch_exact_split(const DevLayer& L, int B, const int* bm, const double* btd, double* y, double* terms,
                       size_t term_doubles, double* acc, cudaStream_t s) {
    switch (L.fmt) {
        case FMT_I8_R32: return dispatch_exact_split<FMT_I8_R32>(L, B, bm, btd, y, terms, term_doubles, acc, s);
        case FMT_I8_WIDE: return dispatch_exact_split<FMT_I8_WIDE>(L, B, bm, btd, y, terms, term_doubles, acc, s);
        case FMT_F32: return dispatch_exact_split<FMT_F32>(L, B, bm, btd, y, terms, term_doubles, acc, s);
        default: return dispatch_exact_split<FMT_DENSE>(L, B, bm, btd, y, terms, term_doubles, acc, s);
    }
}

int launch_exact_b1(const DevLayer& L, const double* xin, int* bm, float* btf, double* btd, int* err, double* y,
                    double* terms, size_t term_doubles, double* acc, cudaStream_t s) {
    if (L.fmt != FMT_I8_R32 || !L.pair8 || L.K <= 0 || L.G - 1 > 64) return 0;
    const size_t outp = static_cast<size_t>((L.out + 31) / 32) * 32;
    const size_t need = outp * L.in, order_d = (static_cast<size_t>(L.in) + 1) / 2;
    if (need + order_d > term_doubles) return 0;
    int* order = reinterpret_cast<int*>(terms + need);
    k_exact_locate_order<<<1, 1024, 0, s>>>(xin, L, bm, btf, btd, err, order);
    const size_t n = static_cast<size_t>(L.in) * L.out;
    const int blocks = static_cast<int>(std::min<size_t>((n + 255) / 256, 148ull * 64));
    k_exact_terms_planes<<<blocks, 256, 0, s>>>(L, 1, bm, btd, order, terms);
    launch_exact_sum(L.out, 1, L.in, terms, acc, y, s);
    return 3;
}

void launch_gather_exact(const DevLayer& L, const LaunchCfg& c, int B, const int* bm,
                         const double* btd, double* y, cudaStream_t s) {
    switch (L.fmt) {
        case FMT_I8_R32: dispatch_exact<FMT_I8_R32>(L, c, B, bm, btd, y, s); break;
        case FMT_I8_WIDE: dispatch_exact<FMT_I8_WIDE>(L, c, B, bm, btd, y, s); break;
        case FMT_F32: dispatch_exact<FMT_F32>(L, c, B, bm, btd, y, s); break;
        default: dispatch_exact<FMT_DENSE>(L, c, B, bm, btd, y, s); break;
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
