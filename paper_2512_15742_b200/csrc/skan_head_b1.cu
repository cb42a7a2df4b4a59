// Batch-1 latency path: the whole head in ONE persistent, cooperative kernel.
//
// At batch 1 the head is a chain of dependent memory round trips, so the
// design minimises round trips, not bytes:
//   * one CTA per SM, grid barriers between layers (no kernel boundaries);
//   * layer 0 (the wide one, e.g. 2048 -> 1408): every edge of input row i
//     uses the same bracket m_i, so rows are bucketed by bracket and each CTA
//     serves a share of ONE bucket with that bucket's codebook pair plane
//     P_m[k] = (c[k][m], c[k][m+1]) staged in shared memory by a TMA bulk
//     copy, together with its rows' records (one more bulk copy per row):
//     a single DRAM round trip, then every 2-byte codebook gather hits
//     shared memory instead of costing a 32-byte sector + an L1 wavefront;
//   * later layers are split by input rows across CTAs; each CTA reduces
//     exactly the previous-layer outputs it consumes (fixed order, double),
//     adds their bias sums and locates them; its records were bulk-copied
//     to shared memory at kernel start;
//   * the last layer's partials are reduced by a few CTAs into y.
// All summation orders are fixed functions of the launch shape and the
// bracket histogram: results are bitwise reproducible run to run.
// int8 tables with <= 65536-row codebooks (FMT_I8_R32); other heads use the
// multi-kernel path.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "skan_device.cuh"
#include "skan_internal.hpp"

namespace skan {
namespace {

using namespace dev;

constexpr int kT = 256;  // threads per CTA
constexpr int kW = kT / 32;
constexpr size_t kPrefetchBytes = 16 * 1024;  // row-split records prefetched at kernel start

// Optional phase timeline (profiling hook): thread 0 of each CTA stamps
// %globaltimer (ns) at fixed phase ids.
__device__ __forceinline__ void stamp(const HeadB1Args& h, int phase) {
    if (h.timeline && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        h.timeline[blockIdx.x * 16 + phase] = t;
    }
}

// Grid barrier: cooperative_groups' grid sync, measured on this part at
// ~1.8k cycles vs 3.5-12.5k for hand-rolled same-address-atomic, two-level
// tree, or per-CTA-flag barriers (tools/microbench3.cu): 148 pollers
// hammering a few L2 lines, or 148 serialised atomics, cost more than the
// driver-provided barrier.
__device__ __forceinline__ void grid_sync() { cooperative_groups::this_grid().sync(); }

// Reduce rows [r0, r1) of the previous layer's per-CTA partials
// prev[z*width + i] (z < nz): C lanes per row, ascending z per lane, then a
// fixed butterfly; + bias; then locate with layer L's grid.  All of a
// thread's loads are issued before any is consumed.
__device__ void reduce_rows(const float* prev, int width, int nz, const double* bias, const DevLayer& L,
                            const long long* skey, const double* snode, int r0, int r1, int* s_m, float* s_t,
                            int* err) {
    const int n = r1 - r0;
    int C = 1;
    while (C < 32 && (C * 2) * n <= kT) C <<= 1;
    const int c = threadIdx.x & (C - 1), groups = kT / C;
    for (int pass = 0; pass < n; pass += groups) {
        const int q = pass + threadIdx.x / C;
        const int i = r0 + min(q, n - 1);
        double v = 0.0;
        for (int z0 = c; z0 < nz; z0 += 16 * C) {
            float buf[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int z = z0 + u * C;
                buf[u] = z < nz ? __ldcg(prev + static_cast<size_t>(z) * width + i) : 0.f;
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) v += static_cast<double>(buf[u]);
        }
        for (int o = C >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
        if (c == 0 && q < n) {
            int m;
            float t;
            fast_locate_tab(skey, snode, L.G, L.lo, L.inv_dx, L.inv_dx_f, v + (bias ? bias[i] : 0.0), err, m, t, L.q_eps);
            s_m[q] = m;
            s_t[q] = t;
        }
    }
}

// Row-split layer: this CTA's rows [r0, r1) (brackets in s_m/s_t), all
// outputs.  Warp w takes rows w, w+8, ...; lane l outputs l, l+32, ...;
// records from shared memory when prefetched (s_rec != nullptr); per-warp
// accumulators in shared memory; fixed-order sum over warps.
__device__ void rowsplit_layer(const DevLayer& L, int r0, int r1, const int* s_m, const float* s_t,
                               const uint32_t* s_rec, const float* s_lut, float* s_acc, float* part_out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int q = threadIdx.x; q < kW * L.out; q += kT) s_acc[q] = 0.f;
    __syncthreads();
    float* acc = s_acc + warp * L.out;
    for (int rl = warp; rl < r1 - r0; rl += kW) {
        const int m = s_m[rl];
        const float t = s_t[rl];
        const uint32_t* rec = s_rec ? s_rec + static_cast<size_t>(rl) * L.out
                                    : L.rec + static_cast<size_t>(r0 + rl) * L.out;
        const uint16_t* plane = L.pair8 + static_cast<size_t>(m) * L.K;
        for (int j = lane; j < L.out; j += 128) {  // 4 independent edges per lane per step
            uint32_t r[4], p[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) r[e] = j + 32 * e < L.out ? rec[j + 32 * e] : 0u;
#pragma unroll
            for (int e = 0; e < 4; ++e) p[e] = j + 32 * e < L.out ? __ldg(plane + (r[e] & 0xFFFFu)) : 0u;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if (j + 32 * e >= L.out) break;
                float c0, dc;
                pair_to_f(p[e], c0, dc);
                acc[j + 32 * e] = fmaf(s_lut[(r[e] >> 16) & 0xFF], fmaf(t, dc, c0), acc[j + 32 * e]);
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

// Pair-plane layer 0.  Shared memory: [plane K*2 B][records rec_cap rows x
// out x 4 B]; rows beyond rec_cap (only for very skewed shapes) read their
// records from global memory.
template <int NV>
__device__ void planes_layer0(const HeadB1Args& h, unsigned char* smem, const float* s_lut, const long long* skey,
                              const double* snode, uint64_t* bar, float* part_out) {
    const DevLayer& L = h.L[0];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int GP = L.G - 1;
    __shared__ int s_whist[kW][32];
    __shared__ int s_cnt[32];
    __shared__ int s_scan[kW];
    __shared__ int s_bucket, s_lo, s_hi;
    __shared__ int s_rows[128];
    __shared__ float s_trow[128];
    uint16_t* s_plane = reinterpret_cast<uint16_t*>(smem);
    const uint32_t plane_bytes = static_cast<uint32_t>(L.K) * 2u;
    uint32_t* s_rec = reinterpret_cast<uint32_t*>(smem + ((plane_bytes + 127u) & ~127u));
    const uint32_t row_bytes = static_cast<uint32_t>(L.out) * 4u;

    // Code size matters more than instruction count here: each warp runs this
    // prologue once, from an instruction cache that the per-call L2 flush
    // leaves cold, so loops stay rolled (#pragma unroll 1).
    // 1. inputs staged in the record region (free until the records land),
    //    brackets of all inputs -> shared memory, integer histogram per warp
    double* s_x = reinterpret_cast<double*>(s_rec);
    float* s_tall = reinterpret_cast<float*>(s_x + L.in);
    uint8_t* s_bm = reinterpret_cast<uint8_t*>(s_tall + L.in);
#pragma unroll 4
    for (int i = tid; i < L.in; i += kT) s_x[i] = h.x[i];
    s_whist[warp][lane] = 0;
    __syncthreads();
    stamp(h, 13);
#pragma unroll 1
    for (int i = tid; i < L.in; i += kT) {
        int m;
        fast_locate_tab(skey, snode, L.G, L.lo, L.inv_dx, L.inv_dx_f, s_x[i], h.err, m, s_tall[i], L.q_eps);
        s_bm[i] = static_cast<uint8_t>(m);
        atomicAdd(&s_whist[warp][m], 1);  // integer counts: order-free, deterministic
    }
    __syncthreads();
    stamp(h, 2);
    if (tid < 32) {
        int s = 0;
#pragma unroll
        for (int w = 0; w < kW; ++w) s += s_whist[w][tid];
        s_cnt[tid] = s;
    }
    __syncthreads();
    // 3. CTA -> bucket (warp 0, lane b = bucket b; 32-bit math), plane TMA
    if (warp == 0) {
        const int P = gridDim.x;
        const int n = lane < GP ? s_cnt[lane] : 0;
        const int nonempty = __popc(__ballot_sync(0xFFFFFFFFu, n > 0));
        const int alloc = n > 0 ? 1 + (P - nonempty) * n / L.in : 0;
        int incl = alloc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += y;
        }
        const int c = blockIdx.x;
        const unsigned hit = __ballot_sync(0xFFFFFFFFu, c >= incl - alloc && c < incl);
        const int b = hit ? __ffs(hit) - 1 : GP;
        if (lane == 0) {
            s_bucket = b;
            s_lo = s_hi = 0;
        }
        __syncwarp();
        if (hit && lane == b) {
            const int q = c - (incl - alloc);
            s_lo = n * q / alloc;
            s_hi = n * (q + 1) / alloc;
        }
    }
    __syncthreads();
    const int bucket = s_bucket, lo = s_lo, hi = s_hi;
    const int nrows = min(hi - lo, 128);
    const int rec_rows = min(nrows, h.rec_cap);
    if (tid == 0 && bucket < GP) {
        mbar_expect_tx(bar, plane_bytes + static_cast<uint32_t>(rec_rows) * row_bytes);
        const char* src = reinterpret_cast<const char*>(L.pair8 + static_cast<size_t>(bucket) * L.K);
        for (uint32_t off = 0; off < plane_bytes; off += 32768u)
            bulk_g2s(smem + off, src + off, min(32768u, plane_bytes - off), bar);
    }
    stamp(h, 3);
    // 4. my rows: rank within the bucket (thread t scans a contiguous slice;
    //    exclusive scan of the slice counts), then one record bulk copy per row
    const int per = (L.in + kT - 1) / kT;
    const int i0 = min(tid * per, L.in), i1 = min(i0 + per, L.in);
    int cnt = 0;
#pragma unroll 1
    for (int i = i0; i < i1; ++i) cnt += s_bm[i] == bucket;
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_scan[warp] = incl;
    __syncthreads();
    int rank = incl - cnt;
#pragma unroll 1
    for (int w = 0; w < warp; ++w) rank += s_scan[w];
#pragma unroll 1
    for (int i = i0; i < i1; ++i) {
        if (s_bm[i] != bucket) continue;
        const int r = rank++ - lo;
        if (r >= 0 && r < nrows) {
            s_rows[r] = i;
            s_trow[r] = s_tall[i];
        }
    }
    __syncthreads();  // staging area free: records may land now
    if (tid < rec_rows)
        bulk_g2s(s_rec + static_cast<size_t>(tid) * L.out, L.rec + static_cast<size_t>(s_rows[tid]) * L.out,
                 row_bytes, bar);
    stamp(h, 4);
    if (bucket < GP) mbar_wait(bar, 0);
    stamp(h, 5);
    // 5. rows: warp w takes rows w, w+8, ...; gathers from the staged plane
    float acc[NV][4];
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[v][e] = 0.f;
    for (int rr = warp; rr < nrows; rr += kW) {
        const float t = s_trow[rr];
        const uint32_t* base = rr < rec_rows ? s_rec + static_cast<size_t>(rr) * L.out
                                             : L.rec + static_cast<size_t>(s_rows[rr]) * L.out;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const int j = v * 128 + lane * 4;
            if (j >= L.out) break;
            const uint4 r = *reinterpret_cast<const uint4*>(base + j);
            const uint32_t r4[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                float c0, dc;
                pair_to_f(s_plane[r4[e] & 0xFFFFu], c0, dc);
                acc[v][e] = fmaf(s_lut[(r4[e] >> 16) & 0xFF], fmaf(t, dc, c0), acc[v][e]);
            }
        }
    }
    stamp(h, 6);
    // 6. fixed-order reduction over warps -> this CTA's partial
    __syncthreads();
    float* s_red = reinterpret_cast<float*>(smem);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        const int j = v * 128 + lane * 4;
        *reinterpret_cast<float4*>(s_red + warp * (128 * NV) + j) =
            make_float4(acc[v][0], acc[v][1], acc[v][2], acc[v][3]);
    }
    __syncthreads();
    for (int j = tid; j < L.out; j += kT) {
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < kW; ++w) s += s_red[w * (128 * NV) + j];
        part_out[static_cast<size_t>(blockIdx.x) * L.out + j] = s;
    }
}

__device__ __forceinline__ void rows_of(const DevLayer& L, int c, int P, int& r0, int& r1) {
    r0 = L.in * c / P;  // 32-bit: in <= 16384, c <= P <= 256 (a 64-bit divide is ~60 instructions)
    r1 = L.in * (c + 1) / P;
}

template <int NV>
__global__ void __launch_bounds__(kT, 1) k_head_b1(HeadB1Args h) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ float s_luts[kMaxHeadLayers][256];
    __shared__ long long s_nkey[kMaxHeadLayers][33];  // node keys / positions (G <= 33)
    __shared__ double s_node[kMaxHeadLayers][33];
    __shared__ __align__(8) uint64_t s_bar[2];  // [0] layer-0 staging, [1] row-split prefetch
    const int P = gridDim.x, c = blockIdx.x;
    stamp(h, 0);
    if (threadIdx.x == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
    }
    __syncthreads();
    // row-split layers' records of this CTA (contiguous rows) are bulk-copied
    // now into the tail of shared memory, consumed after the grid barriers
    unsigned char* s_pref = smem + h.pref_offset;
    if (threadIdx.x == 0 && h.pref_mask) {
        uint32_t total = 0;
        for (int l = 0; l < h.nl; ++l) {
            if (!(h.pref_mask >> l & 1)) continue;
            int r0, r1;
            rows_of(h.L[l], c, P, r0, r1);
            total += static_cast<uint32_t>(r1 - r0) * h.L[l].out * 4u;
        }
        mbar_expect_tx(&s_bar[1], total);
        uint32_t off = 0;
        for (int l = 0; l < h.nl; ++l) {
            if (!(h.pref_mask >> l & 1)) continue;
            int r0, r1;
            rows_of(h.L[l], c, P, r0, r1);
            const uint32_t bytes = static_cast<uint32_t>(r1 - r0) * h.L[l].out * 4u;
            if (bytes) bulk_g2s(s_pref + off, h.L[l].rec + static_cast<size_t>(r0) * h.L[l].out, bytes, &s_bar[1]);
            off += bytes;
        }
    }
    for (int l = 0; l < h.nl; ++l) {
        s_luts[l][threadIdx.x] = h.L[l].lutf[threadIdx.x];
        if (threadIdx.x < h.L[l].G) {
            s_nkey[l][threadIdx.x] = h.L[l].nkey[threadIdx.x];
            s_node[l][threadIdx.x] = h.L[l].node[threadIdx.x];
        }
    }
    __syncthreads();
    stamp(h, 1);
    int* s_m = reinterpret_cast<int*>(smem);  // row-split scratch (after layer 0)
    uint32_t pref_off = 0;
    bool pref_ready = false;
    for (int l = 0; l < h.nl; ++l) {
        const DevLayer& L = h.L[l];
        float* part_out = h.part[l & 1];
        const float* s_lut = s_luts[l];
        if (l == 0 && h.planes0) {
            planes_layer0<NV>(h, smem, s_lut, s_nkey[0], s_node[0], &s_bar[0], part_out);
        } else {
            int r0, r1;
            rows_of(L, c, P, r0, r1);
            const int nr = r1 - r0;
            float* s_t = reinterpret_cast<float*>(s_m + nr);
            float* s_acc = s_t + nr;
            if (l == 0) {
                for (int q = threadIdx.x; q < nr; q += kT)
                    fast_locate_tab(s_nkey[0], s_node[0], L.G, L.lo, L.inv_dx, L.inv_dx_f, h.x[r0 + q], h.err, s_m[q], s_t[q], L.q_eps);
            } else {
                reduce_rows(h.part[(l - 1) & 1], L.in, P, h.L[l - 1].bias_sum, L, s_nkey[l], s_node[l], r0, r1, s_m,
                            s_t, h.err);
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
            if (l == 1) stamp(h, 9);
            rowsplit_layer(L, r0, r1, s_m, s_t, s_rec, s_lut, s_acc, part_out);
        }
        stamp(h, l == 0 ? 7 : 10);
        grid_sync();
        if (l + 1 < h.nl) stamp(h, l == 0 ? 8 : 11);
    }
    // the last layer's partials are reduced by CTA 0 alone
    if (blockIdx.x != 0) return;
    stamp(h, 11);
    // final (CTA 0): every output of the last layer, one warp each
    const DevLayer& L = h.L[h.nl - 1];
    const float* part = h.part[(h.nl - 1) & 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int j = warp; j < L.out; j += kW) {
        double v = 0.0;
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
        if (lane == 0) h.y[j] = v + (L.bias_sum ? L.bias_sum[j] : 0.0);
    }
    stamp(h, 12);
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
size_t head_b1_smem(const DevLayer* L, int nl, int num_sms, HeadB1Args* h, int* nv) {
    const DevLayer& L0 = L[0];
    const size_t kBudget = 204 * 1024;  // dynamic; + ~10.5 KB static + 1 KB reserved <= 227 KB
    h->planes0 = L0.out % 4 == 0 && L0.out <= 1536 && L0.in <= 16 * kT && L0.K % 8 == 0 &&
                 static_cast<size_t>(L0.K) * 2 <= 144 * 1024 && L0.G - 1 <= 32 &&
                 static_cast<long long>(L0.in) * L0.out >= 256LL * 1024 &&
                 num_sms - (L0.G - 1) > 0 && L0.in / (num_sms - (L0.G - 1)) + 2 <= 128;  // s_rows[128]
    const int groups = (L0.out + 127) / 128;
    *nv = groups <= 2 ? 2 : (groups <= 4 ? 4 : (groups <= 8 ? 8 : 12));
    // prefetch: row-split layers whose per-CTA record block is small
    size_t pref = 0;
    h->pref_mask = 0;
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
    if (h->planes0) {
        const size_t plane = (static_cast<size_t>(L0.K) * 2 + 127) / 128 * 128;
        const size_t red = static_cast<size_t>(kW) * 128 * (*nv) * sizeof(float);
        const size_t row = static_cast<size_t>(L0.out) * 4;
        // rows per CTA < in / (P - buckets) + 1
        const int spare = num_sms - (L0.G - 1) > 0 ? num_sms - (L0.G - 1) : 1;
        const int want = L0.in / spare + 2;
        const size_t avail = kBudget > plane + pref ? kBudget - plane - pref : 0;
        size_t cap = avail / row;
        if (cap > static_cast<size_t>(want)) cap = want;
        if (cap > 128) cap = 128;
        h->rec_cap = static_cast<int>(cap);
        // the record region doubles as the input staging area (x, t, bracket)
        const size_t staging = static_cast<size_t>(L0.in) * (sizeof(double) + sizeof(float) + 1) + 128;
        phase = plane + (cap * row > staging ? cap * row : staging);
        if (red > phase) phase = red;
    }
    for (int l = 0; l < nl; ++l) {
        if (l == 0 && h->planes0) continue;
        const int nr = (L[l].in + num_sms - 1) / num_sms + 1;
        const size_t s = static_cast<size_t>(nr) * 8 + static_cast<size_t>(kW) * L[l].out * sizeof(float);
        if (s > phase) phase = s;
    }
    phase = (phase + 127) / 128 * 128;
    h->pref_offset = static_cast<uint32_t>(phase);
    return phase + pref;
}

static void (*head_b1_kernel(int nv))(HeadB1Args) {
    switch (nv) {
        case 2: return k_head_b1<2>;
        case 4: return k_head_b1<4>;
        case 8: return k_head_b1<8>;
        default: return k_head_b1<12>;
    }
}

int head_b1_max_grid(size_t smem, int nv, int num_sms) {
    auto k = head_b1_kernel(nv);
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kT, smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return per_sm >= 1 ? num_sms : 0;
}

void launch_head_b1(const HeadB1Args& h, int grid, size_t smem, int nv, cudaStream_t s) {
    auto k = head_b1_kernel(nv);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
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
    cudaLaunchKernelEx(&cfg, k, h);
}

}  // namespace skan
