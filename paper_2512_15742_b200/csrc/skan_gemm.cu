// tcgen05 kind::tf32 GEMM, three-pass split precision ("3xTF32"):
//     A*B ~= A_hi*B_hi + A_hi*B_lo + A_lo*B_hi
// with x_hi = the tensor core's own tf32 truncation of x and x_lo = x - x_hi
// (exact in f32), accumulated in f32 in TMEM: ~2^-21 relative per product,
// inside the fast path's 1e-5 (L1-scaled) bar where a single tf32 pass
// (~2^-11) is not.
//
// k_debug_gemm is the self-test of the building blocks in skan_tc.cuh: one
// CTA, 128 x N (N <= 256) x K (K <= 64) from row-major f32 A [128][K] and
// B [K][N] staged by plain threads into the canonical K-major layout.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "skan_internal.hpp"
#include "skan_tc.cuh"

namespace skan {
namespace {

__global__ void __launch_bounds__(128, 1) k_debug_gemm(const float* __restrict__ A, const float* __restrict__ B,
                                                      float* __restrict__ D, int N, int K, int passes, int M) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t s_bar;
    __shared__ uint32_t s_tmem;
    unsigned char* a_hi = smem;
    unsigned char* a_lo = a_hi + M * K * 4;
    unsigned char* b_hi = a_lo + M * K * 4;
    unsigned char* b_lo = b_hi + N * K * 4;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int q = tid; q < M * K; q += 128) {
        const int r = q / K, k = q % K;
        const float x = A[q];
        *reinterpret_cast<float*>(a_hi + tc::kmajor_off(r, k, M)) = x;
        *reinterpret_cast<float*>(a_lo + tc::kmajor_off(r, k, M)) = tc::tf32_lo(x);
    }
    for (int q = tid; q < N * K; q += 128) {
        const int k = q / N, n = q % N;
        const float x = B[q];
        *reinterpret_cast<float*>(b_hi + tc::kmajor_off(n, k, N)) = x;
        *reinterpret_cast<float*>(b_lo + tc::kmajor_off(n, k, N)) = tc::tf32_lo(x);
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc::smem_addr(&s_bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc::fence_proxy_async();
    if (warp == 0) tc::tmem_alloc<256>(&s_tmem);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = s_tmem;
    if (tid == 0) {
        const uint32_t idesc = tc::idesc_tf32(M, N);
        const uint32_t lbo_a = (M / 8) * 128, lbo_b = (N / 8) * 128;
        for (int s = 0; s < K / 8; ++s) {
            const uint32_t oa = s * 2 * lbo_a, ob = s * 2 * lbo_b;
            const uint64_t ah = tc::make_desc(tc::smem_addr(a_hi) + oa, lbo_a, 128);
            const uint64_t al = tc::make_desc(tc::smem_addr(a_lo) + oa, lbo_a, 128);
            const uint64_t bh = tc::make_desc(tc::smem_addr(b_hi) + ob, lbo_b, 128);
            const uint64_t bl = tc::make_desc(tc::smem_addr(b_lo) + ob, lbo_b, 128);
            tc::mma_tf32(tmem, ah, bh, idesc, s > 0);
            if (passes >= 3) {
                tc::mma_tf32(tmem, ah, bl, idesc, true);
                tc::mma_tf32(tmem, al, bh, idesc, true);
            }
        }
        tc::mma_commit(&s_bar);
    }
    __syncwarp();
    // wait for the MMAs
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(tc::smem_addr(&s_bar))
            : "memory");
    }
    tc::fence_after_sync();
    const int row = warp * 32 + lane;  // TMEM lane (== row for M = 128; raw lanes are dumped for M = 64)
    for (int c = 0; c < N; c += 8) {
        float v[8];
        tc::tmem_ld8(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c, v);
#pragma unroll
        for (int q = 0; q < 8; ++q) D[row * N + c + q] = v[q];
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_free<256>(tmem);
}

}  // namespace
}  // namespace skan

extern "C" skan_status skan_debug_gemm_tf32(const float* dA, const float* dB, float* dD, int N, int K, int passes,
                                            void* stream) {
    // passes >= 100: M = 64 variant (passes - 100), D receives the raw 128 TMEM lanes
    const int M = passes >= 100 ? 64 : 128;
    if (passes >= 100) passes -= 100;
    if (N < 8 || N > 256 || N % 16 || K < 8 || K > 64 || K % 8)
        return skan::set_error(SKAN_SHAPE_ERROR, "debug gemm: N in [16,256] step 16, K in [8,64] step 8", 0,
                               SKAN_FAULT_NONE);
    const size_t smem = static_cast<size_t>(2 * 128 * K + 2 * N * K) * 4;
    cudaFuncSetAttribute(skan::k_debug_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    skan::k_debug_gemm<<<1, 128, smem, static_cast<cudaStream_t>(stream)>>>(dA, dB, dD, N, K, passes, M);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return skan::set_error(SKAN_CUDA_ERROR, cudaGetErrorString(e), 0, SKAN_FAULT_NONE);
    return SKAN_OK;
}

// ===========================================================================
// K4: a fast-path layer as a tensor-core GEMM, used at large batch.
//
// The reference's per-edge interpolation, bias included (lutham.cpp:810:
// (g c0 + b)(1-t) + (g c1 + b) t), is a contraction over the knot basis:
//     y[b][j] = sum_i sum_m  A[b][i*G+m] * W[i*G+m][j]
//     A[b][i*G+m] = hat weight of knot m at x_bi: 1-t at the bracket, t at
//                   the next knot, 0 elsewhere (kan.cpp:28-58 brackets)
//     W[i*G+m][j] = g_ij * c_kij[m] + b_ij  (the reconstructed per-edge grid,
//                   to_dense_network, lutham.cpp:304), or the dense grid
// so a layer is Y[B x out] = A[B x in*G] * W[in*G x out].  Each CTA owns a
// 128-sample x 128-output tile and a split of the inputs; per chunk of IC
// inputs its 256 threads write A (from the brackets) and W (decoded from the
// compressed records + codebook, or read from the dense grid) into shared
// memory in the canonical K-major layout, split into tf32 hi/lo, and one
// thread issues 3 x (IC*G/8) tcgen05.mma (3xTF32) into a TMEM accumulator;
// the next chunk is generated while the tensor core runs (two stages,
// mbarrier-tracked).  Split partials are reduced in fixed order (f64) by
// k_split_reduce, which also locates the next layer's inputs.
// ===========================================================================

#include "skan_device.cuh"

namespace skan {
namespace {

using namespace dev;

constexpr int kGmM = 128;  // samples per tile (MMA M)
constexpr int kGmN = 128;  // outputs per tile (MMA N, TMEM columns)
constexpr int kGmP = 512;        // producers: 4 knot groups x 128 output columns (W), 128 samples x 4 inputs (A)
constexpr int kGmT = kGmP + 32;  // + one warp that issues the tensor-core MMAs
constexpr int kStg = 3;          // DENSE: grid-slab staging slots (TMA bulk copies, 3 chunks ahead)

__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, unsigned parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(tc::smem_addr(bar)), "r"(parity)
            : "memory");
    }
}

// Per-thread staging of one edge (i, j), loaded one chunk ahead: I8 the
// 16-byte codebook row plus gain and bias already decoded (the record that
// names the row is loaded one chunk earlier still, so the row load never
// waits on it); F32 the row index, gain and bias; DENSE the grid values at
// the thread's knots.
struct EdgeRaw {
    uint4 row;
    uint32_t k;
    float g, b;
    float v[4];
};

// record word of an int8 edge: (row, gain code, bias code); WIDE also the
// u32 row index.  Only the loads are issued here: nothing consumes them
// until the next chunk.
template <int FMT>
__device__ __forceinline__ void rec_load(const DevLayer& L, size_t e, uint32_t& rec, uint32_t& k) {
    if constexpr (FMT == FMT_I8_R32) {
        rec = __ldg(L.rec + e);
    } else {
        k = L.idx ? __ldg(L.idx + e) : 0u;
        rec = __ldg(L.gb + e);
    }
}

// W value of a staged edge at its u-th knot m (fast-path decode); int8
// codes become floats through the 2^23 + (u ^ 0x80) bit pattern (no I2F).
template <int FMT>
__device__ __forceinline__ float edge_w(const DevLayer& L, const EdgeRaw& r, int m, int u) {
    if constexpr (FMT == FMT_DENSE) {
        return r.v[u];
    } else if constexpr (FMT == FMT_F32) {
        return fmaf(r.g, __ldg(L.cb32 + static_cast<size_t>(r.k) * L.G + m), r.b);
    } else {
        const uint32_t w = m < 4 ? r.row.x : (m < 8 ? r.row.y : (m < 12 ? r.row.z : r.row.w));
        const float code = __int_as_float(static_cast<int>(((w >> (8 * (m & 3))) & 0xFFu) ^ 0x4B000080u)) - 8388736.0f;
        return fmaf(r.g, code, r.b);
    }
}

// Chunk K order: k = m * IC + il (knot-major), so the IC inputs of one
// edge column at one knot are contiguous 4-float groups of the K-major
// tile: W is written with 16-byte stores.  IC is 4 (G even) or 8 (G odd).
// Thread t: W for output column t % 128 at knots t/128, t/128 + 4, ...;
// A for sample t % 128 at input t / 128 (and + 4 when IC = 8).
template <int FMT, int IC, int MT>  // MT: samples per tile (MMA M = 64 or 128)
__global__ void __launch_bounds__(kGmT, 1) k_layer_gemm(FwdArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t s_bar[2];   // stage free: committed by the MMA warp
    __shared__ __align__(8) uint64_t s_full[2];  // stage written: every producer arrives
    __shared__ __align__(8) uint64_t s_stg[kStg];  // DENSE: grid slab of chunk c landed in staging slot c % kStg
    __shared__ uint32_t s_tmem;
    __shared__ float s_lut[256];
    const DevLayer& L = a.L;
    const int G = L.G, KC = IC * G;
    const uint32_t tile_a = MT * KC * 4, tile_w = kGmN * KC * 4;
    const uint32_t stage_bytes = 2 * tile_a + 2 * tile_w;  // [A_hi][A_lo][W_hi][W_lo]
    constexpr uint32_t kLboA = (MT / 8) * 128, kLboW = (kGmN / 8) * 128;
    constexpr int kAU = (IC * MT + kGmP - 1) / kGmP;  // A slots per producer (1 or 2)
    // DENSE: the grid slab of a chunk (IC inputs x 128 columns x G floats) is
    // bulk-copied into a staging ring behind the two operand stages
    const bool stg = FMT == FMT_DENSE && a.tma_w;
    const uint32_t slab = kGmN * static_cast<uint32_t>(G) * 4;  // bytes per input row of the slab
    unsigned char* s_slab = smem + 2 * stage_bytes;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int j0 = blockIdx.x * kGmN, s0 = blockIdx.z * MT;
    const int nS = min(MT, a.B - s0), nJ = min(kGmN, L.out - j0);
    const int r0 = blockIdx.y * a.rows_per_cta, rend = min(L.in, r0 + a.rows_per_cta);
    const int nchunks = rend > r0 ? (rend - r0 + IC - 1) / IC : 0;
    pdl_trigger();
    if constexpr (FMT == FMT_I8_R32 || FMT == FMT_I8_WIDE) {
        if (tid < 256) s_lut[tid] = L.lutf[tid];
    }
    // the A tiles are sparse (2 of G weights per sample and input): zero both
    // stages once, then write and clear only the nonzeros
    for (uint32_t q = tid * 16; q < 2 * stage_bytes; q += kGmT * 16) {
        const uint32_t st = q / stage_bytes, o = q % stage_bytes;
        if (o < 2 * tile_a) *reinterpret_cast<uint4*>(smem + st * stage_bytes + o) = make_uint4(0, 0, 0, 0);
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc::smem_addr(&s_bar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc::smem_addr(&s_bar[1])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc::smem_addr(&s_full[0])), "r"(kGmP));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc::smem_addr(&s_full[1])), "r"(kGmP));
        for (int q = 0; q < kStg; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc::smem_addr(&s_stg[q])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tc::tmem_alloc<kGmN>(&s_tmem);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = s_tmem;
    const uint32_t idesc = tc::idesc_tf32(MT, kGmN);

    const int rl = tid & (kGmN - 1), grp = tid >> 7;  // W: output column, knot group 0..3
    const uint32_t rbase = tc::kmajor_off(rl, 0, kGmN);  // row part of the W offset
    EdgeRaw er[IC];
    unsigned evalid = 0;   // edges of the staged chunk inside the layer
    uint32_t recn[IC], kn[IC];  // I8: records of the chunk after the staged one
    unsigned nvalid = 0;
    int bm[kAU];
    float bt[kAU];
    uint32_t aoff0[kAU], aoff1[kAU];  // nonzero A offsets written into stage 0 / 1 (cleared on reuse)
#pragma unroll
    for (int u = 0; u < kAU; ++u) aoff0[u] = aoff1[u] = 0xFFFFFFFFu;
    constexpr bool kI8 = FMT == FMT_I8_R32 || FMT == FMT_I8_WIDE;
    const float bs_f = static_cast<float>(L.bs);
    auto load_recs = [&](int c) {  // I8 records of chunk c
        const int ib = r0 + c * IC;
        nvalid = 0;
#pragma unroll
        for (int il = 0; il < IC; ++il) {
            const int i = ib + il;
            if (rl < nJ && i < rend) {
                nvalid |= 1u << il;
                rec_load<FMT>(L, static_cast<size_t>(i) * L.out + j0 + rl, recn[il], kn[il]);
            }
        }
    };
    auto load_chunk = [&](int c) {  // stage chunk c's edge data and brackets into registers
        const int ib = r0 + c * IC;
        if constexpr (kI8) {
            evalid = nvalid;
#pragma unroll
            for (int il = 0; il < IC; ++il) {
                if (!(evalid >> il & 1)) continue;
                const uint32_t r = recn[il];
                const uint32_t k = FMT == FMT_I8_R32 ? (r & 0xFFFFu) : kn[il];
                const uint32_t gb = FMT == FMT_I8_R32 ? (r >> 16) : r;  // gain code | bias code << 8
                er[il].row = __ldg(reinterpret_cast<const uint4*>(L.cb8 + static_cast<size_t>(k) * L.rs));
                er[il].g = s_lut[gb & 0xFFu];  // float(gain(code) * codebook scale)
                er[il].b = static_cast<float>(static_cast<int8_t>((gb >> 8) & 0xFFu)) * bs_f;
            }
        } else {
            evalid = 0;
#pragma unroll
            for (int il = 0; il < IC; ++il) {
                const int i = ib + il;
                if (!(rl < nJ && i < rend)) continue;
                evalid |= 1u << il;
                const size_t e = static_cast<size_t>(i) * L.out + j0 + rl;
                if constexpr (FMT == FMT_F32) {
                    er[il].k = L.idx ? __ldg(L.idx + e) : 0u;
                    er[il].g = __ldg(L.gain + e);
                    er[il].b = __ldg(L.bias + e);
                } else if (!stg) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int m = grp + 4 * u;
                        er[il].v[u] = m < G ? __ldg(L.cb32 + e * static_cast<size_t>(G) + m) : 0.f;
                    }
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kAU; ++u) {
            const int q = tid + kGmP * u, ra = q % MT, ila = q / MT, i = ib + ila;
            bm[u] = -2;
            bt[u] = 0.f;
            if (ila < IC && ra < nS && i < rend) {
                const size_t p = static_cast<size_t>(i) * a.B + s0 + ra;
                bm[u] = a.bm_in[p];
                bt[u] = a.bt_in[p];
            }
        }
        if constexpr (kI8) {
            if (c + 1 < nchunks) load_recs(c + 1);
        }
    };
    pdl_wait();  // brackets come from the previous kernel
    __syncthreads();  // s_lut visible
    if (tid < kGmP) {
        // producers: write stage c as soon as the MMAs of chunk c-2 released it
        if (nchunks > 0) {
            if constexpr (kI8) load_recs(0);
            load_chunk(0);
        }
#pragma unroll 1
        for (int c = 0; c < nchunks; ++c) {
            const int buf = c & 1;
            unsigned char* st = smem + buf * stage_bytes;
            if (c >= 2) mbar_wait_parity(&s_bar[buf], ((c - 2) >> 1) & 1);
            const float* slabf = nullptr;
            if constexpr (FMT == FMT_DENSE) {
                if (stg) {
                    mbar_wait_parity(&s_stg[c % kStg], (c / kStg) & 1);
                    slabf = reinterpret_cast<const float*>(s_slab + (c % kStg) * IC * slab);
                }
            }
            // W: this thread's knots, the IC inputs' values as 16-byte groups
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int m = grp + 4 * u;
                if (m >= G) break;
#pragma unroll
                for (int h = 0; h < IC / 4; ++h) {
                    float v[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int il = 4 * h + q;
                        if constexpr (FMT == FMT_DENSE) {
                            if (stg) {
                                v[q] = (evalid >> il & 1) ? slabf[(il * kGmN + rl) * G + m] : 0.f;
                                continue;
                            }
                        }
                        v[q] = (evalid >> il & 1) ? edge_w<FMT>(L, er[il], m, u) : 0.f;
                    }
                    const uint32_t o = (m * (IC / 4) + h) * kLboW + rbase;
                    *reinterpret_cast<float4*>(st + 2 * tile_a + o) = make_float4(v[0], v[1], v[2], v[3]);
                    *reinterpret_cast<float4*>(st + 2 * tile_a + tile_w + o) =
                        make_float4(tc::tf32_lo(v[0]), tc::tf32_lo(v[1]), tc::tf32_lo(v[2]), tc::tf32_lo(v[3]));
                }
            }
            // A: clear the two weights chunk c-2 left, write this chunk's
#pragma unroll
            for (int u = 0; u < kAU; ++u) {
                const int qa = tid + kGmP * u, ra = qa % MT, il = qa / MT;
                const uint32_t rbase_a = tc::kmajor_off(ra, 0, MT);
                uint32_t& ao = buf ? aoff1[u] : aoff0[u];
                if (ao != 0xFFFFFFFFu) {
                    const uint32_t o0 = ao & 0xFFFFu, o1 = ao >> 16;
                    *reinterpret_cast<float*>(st + o0) = 0.f;
                    *reinterpret_cast<float*>(st + tile_a + o0) = 0.f;
                    *reinterpret_cast<float*>(st + o1) = 0.f;
                    *reinterpret_cast<float*>(st + tile_a + o1) = 0.f;
                    ao = 0xFFFFFFFFu;
                }
                if (bm[u] >= 0) {
                    const int k0 = bm[u] * IC + il, k1 = k0 + IC;
                    const uint32_t o0 = rbase_a + (k0 >> 2) * kLboA + (k0 & 3) * 4;
                    const uint32_t o1 = rbase_a + (k1 >> 2) * kLboA + (k1 & 3) * 4;
                    const float w0 = 1.f - bt[u], w1 = bt[u];
                    *reinterpret_cast<float*>(st + o0) = w0;
                    *reinterpret_cast<float*>(st + tile_a + o0) = tc::tf32_lo(w0);
                    *reinterpret_cast<float*>(st + o1) = w1;
                    *reinterpret_cast<float*>(st + tile_a + o1) = tc::tf32_lo(w1);
                    ao = o0 | (o1 << 16);
                }
            }
            if (c + 1 < nchunks) load_chunk(c + 1);  // next chunk's tables fly while this one multiplies
            tc::fence_proxy_async();                 // this thread's stage writes -> the tensor core
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_addr(&s_full[buf])) : "memory");
        }
    } else {
        // the MMA warp: one lane issues 3 x (KC/8) tcgen05.mma per chunk, in
        // order (and, for dense layers, the grid-slab bulk copies kStg chunks ahead)
        auto issue_slab = [&](int c) {
            if constexpr (FMT == FMT_DENSE) {
                if (!stg || c >= nchunks) return;
                const int ib = r0 + c * IC;
                const uint32_t bytes = static_cast<uint32_t>(nJ) * G * 4;
                int nv = 0;
                for (int il = 0; il < IC; ++il) nv += ib + il < rend;
                uint64_t* bar = &s_stg[c % kStg];
                mbar_expect_tx(bar, nv * bytes);
                unsigned char* dst = s_slab + (c % kStg) * IC * slab;
                for (int il = 0; il < IC; ++il)
                    if (ib + il < rend)
                        bulk_g2s(dst + il * slab, L.cb32 + (static_cast<size_t>(ib + il) * L.out + j0) * G, bytes, bar);
            }
        };
        if (lane == 0)
            for (int c = 0; c < kStg; ++c) issue_slab(c);
#pragma unroll 1
        for (int c = 0; c < nchunks; ++c) {
            const int buf = c & 1;
            mbar_wait_parity(&s_full[buf], (c >> 1) & 1);
            if (lane == 0) {
                issue_slab(c + kStg);  // the producers are done with chunk c's slab
                tc::fence_after_sync();
                const uint32_t base = tc::smem_addr(smem + buf * stage_bytes);
#pragma unroll 1
                for (int s = 0; s < KC / 8; ++s) {
                    const uint32_t oa = s * 2 * kLboA, ow = s * 2 * kLboW;
                    const uint64_t ah = tc::make_desc(base + oa, kLboA, 128);
                    const uint64_t al = tc::make_desc(base + tile_a + oa, kLboA, 128);
                    const uint64_t wh = tc::make_desc(base + 2 * tile_a + ow, kLboW, 128);
                    const uint64_t wl = tc::make_desc(base + 2 * tile_a + tile_w + ow, kLboW, 128);
                    tc::mma_tf32(tmem, ah, wh, idesc, c > 0 || s > 0);
                    tc::mma_tf32(tmem, ah, wl, idesc, true);
                    tc::mma_tf32(tmem, al, wh, idesc, true);
                }
                tc::mma_commit(&s_bar[buf]);
            }
            __syncwarp();
        }
    }
    if (nchunks > 0) mbar_wait_parity(&s_bar[(nchunks - 1) & 1], ((nchunks - 1) >> 1) & 1);
    tc::fence_after_sync();
    // epilogue: producer warp w reads TMEM lanes (w%4)*32.. (its samples), columns (w/4)*32..+32
    const int q4 = warp & 3, cq = warp >> 2;
    if (warp < kGmP / 32) {
    // M = 128: sample r in TMEM lane r; M = 64: sample r in lane (r/16)*32 + r%16
    const int row = MT == 128 ? q4 * 32 + lane : (lane < 16 ? q4 * 16 + lane : MT);
    const size_t plane = static_cast<size_t>(a.B) * L.out;
    float* dst = a.partial + blockIdx.y * plane + static_cast<size_t>(s0 + min(row, MT - 1)) * L.out + j0;
#pragma unroll 1
    for (int c8 = cq * 32; c8 < cq * 32 + 32; c8 += 8) {
        float v[8];
        if (nchunks > 0) {
            tc::tmem_ld8(tmem + (static_cast<uint32_t>(q4 * 32) << 16) + c8, v);
        } else {
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = 0.f;
        }
        if (row < nS) {
            if (c8 + 8 <= nJ && (L.out & 3) == 0) {
                *reinterpret_cast<float4*>(dst + c8) = make_float4(v[0], v[1], v[2], v[3]);
                *reinterpret_cast<float4*>(dst + c8 + 4) = make_float4(v[4], v[5], v[6], v[7]);
            } else {
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (c8 + u < nJ) dst[c8 + u] = v[u];
            }
        }
    }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_free<kGmN>(tmem);
}

__device__ __forceinline__ void reduce_finish(const FwdArgs& a, size_t p, double v, int add_bias) {
    const DevLayer& L = a.L;
    const int j = static_cast<int>(p % L.out);
    if (add_bias && L.bias_sum) v += L.bias_sum[j];
    a.y[p] = v;
    if (a.has_next) {
        int m;
        float t;
        fast_locate(a.N, v, a.err, m, t);
        const size_t q = static_cast<size_t>(j) * a.B + p / L.out;
        a.bm_out[q] = m;
        a.bt_out[q] = t;
    }
}

// Fixed-order (ascending split) f64 reduction of the split partials, one
// thread per (sample, output); + bias sums when the layer's bias was not
// folded into W; y; next layer's bracket (input-major).
__global__ void k_split_reduce(FwdArgs a, int nsplit, int add_bias) {
    pdl_trigger();
    pdl_wait();
    const size_t plane = static_cast<size_t>(a.B) * a.L.out;
    for (size_t p = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; p < plane;
         p += static_cast<size_t>(gridDim.x) * blockDim.x) {
        double v = 0.0;
        int z = 0;
        for (; z + 4 <= nsplit; z += 4) {  // four loads in flight, summed in split order
            float f[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) f[u] = __ldcg(a.partial + (z + u) * plane + p);
#pragma unroll
            for (int u = 0; u < 4; ++u) v += static_cast<double>(f[u]);
        }
        for (; z < nsplit; ++z) v += static_cast<double>(__ldcg(a.partial + z * plane + p));
        reduce_finish(a, p, v, add_bias);
    }
}

// Many splits, few entries (narrow layers): one warp per entry, lane l sums
// splits l, l+32, ... in order, then a fixed butterfly.
__global__ void k_split_reduce_warp(FwdArgs a, int nsplit, int add_bias) {
    pdl_trigger();
    pdl_wait();
    const size_t plane = static_cast<size_t>(a.B) * a.L.out;
    const int lane = threadIdx.x & 31;
    for (size_t p = (blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x) / 32; p < plane;
         p += static_cast<size_t>(gridDim.x) * blockDim.x / 32) {
        double v = 0.0;
        for (int z = lane; z < nsplit; z += 32) v += static_cast<double>(__ldcg(a.partial + z * plane + p));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
        if (lane == 0) reduce_finish(a, p, v, add_bias);
    }
}

template <typename K, typename... Args>
void launch_pdl(K kernel, dim3 grid, dim3 block, size_t smem, bool pdl, cudaStream_t s, Args... args) {
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
    cudaLaunchKernelEx(&cfg, kernel, args...);
}

}  // namespace

// Inputs per chunk: IC*G must be a multiple of the tf32 MMA K (8), and IC
// a multiple of 4 (16-byte W groups): 4 for even G, 8 for odd G.
int gemm_ic(int G) { return G % 2 == 0 ? 4 : 8; }

size_t gemm_smem(int G, bool dense, int mt = kGmM) {
    const size_t kc = static_cast<size_t>(gemm_ic(G)) * G;
    return 2 * (2 * static_cast<size_t>(mt) * kc * 4 + 2 * kGmN * kc * 4) + (dense ? kStg * kc * kGmN * 4 : 0);
}

bool gemm_supported(const DevLayer& L) {
    const int ic = gemm_ic(L.G);
    return ic > 0 && L.G <= 16 && gemm_smem(L.G, L.fmt == FMT_DENSE) <= 222 * 1024 &&
           (L.fmt == FMT_I8_R32 || L.fmt == FMT_I8_WIDE || L.fmt == FMT_F32 || L.fmt == FMT_DENSE);
}

LaunchCfg gemm_cfg(const DevLayer& L, int B, int num_sms) {
    LaunchCfg c{};
    c.kind = 4;
    c.ic = gemm_ic(L.G);
    c.jt = (L.out + kGmN - 1) / kGmN;
    c.spt = B <= 64 ? 64 : kGmM;  // samples per tile: the M = 64 MMA when the batch fits it
    c.st = (B + c.spt - 1) / c.spt;
    c.tj = kGmN;
    const int sms = num_sms > 0 ? num_sms : 148;
    // one CTA per SM: the fewest input splits whose waves are >= 90% full
    const long long base = static_cast<long long>(c.jt) * c.st;
    const long long maxns = std::max<long long>(1, std::min<long long>(64, (L.in + c.ic - 1) / c.ic));
    long long ns = 1;
    double best = 0.0;
    for (long long k = 1; k <= maxns; ++k) {
        const long long ctas = base * k, waves = (ctas + sms - 1) / sms;
        const double eff = static_cast<double>(ctas) / static_cast<double>(waves * sms);
        if (eff > best + 1e-9) {
            best = eff;
            ns = k;
        }
        if (eff >= 0.9) break;
    }
    const int chunks = (L.in + c.ic - 1) / c.ic;
    const int per = (chunks + static_cast<int>(ns) - 1) / static_cast<int>(ns);
    c.ichunk = per * c.ic;
    c.nsplit = (L.in + c.ichunk - 1) / c.ichunk;
    c.smem = gemm_smem(L.G, L.fmt == FMT_DENSE, c.spt);
    return c;
}

template <int MT>
void (*gemm_kernel(int fmt, int ic))(FwdArgs) {
    const bool i4 = ic == 4;
    switch (fmt) {
        case FMT_I8_R32: return i4 ? k_layer_gemm<FMT_I8_R32, 4, MT> : k_layer_gemm<FMT_I8_R32, 8, MT>;
        case FMT_I8_WIDE: return i4 ? k_layer_gemm<FMT_I8_WIDE, 4, MT> : k_layer_gemm<FMT_I8_WIDE, 8, MT>;
        case FMT_F32: return i4 ? k_layer_gemm<FMT_F32, 4, MT> : k_layer_gemm<FMT_F32, 8, MT>;
        default: return i4 ? k_layer_gemm<FMT_DENSE, 4, MT> : k_layer_gemm<FMT_DENSE, 8, MT>;
    }
}

void launch_layer_gemm(const FwdArgs& a, const LaunchCfg& c, bool pdl, cudaStream_t s) {
    void (*k)(FwdArgs) = c.spt == 64 ? gemm_kernel<64>(a.L.fmt, c.ic) : gemm_kernel<128>(a.L.fmt, c.ic);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(c.smem));
    FwdArgs g = a;
    // dense slabs by TMA when every slab row is 16-byte aligned
    g.tma_w = a.L.fmt == FMT_DENSE && (static_cast<long long>(a.L.out) * a.L.G) % 4 == 0 &&
              (reinterpret_cast<uintptr_t>(a.L.cb32) & 15) == 0;
    launch_pdl(k, dim3(c.jt, c.nsplit, c.st), dim3(kGmT), c.smem, pdl, s, g);
    // bias: folded into W for compressed layers; dense layers have none
    const long long n = static_cast<long long>(a.B) * a.L.out;
    if (c.nsplit >= 16 && n < 148LL * 256) {
        const int blocks = static_cast<int>(std::min<long long>((n * 32 + 255) / 256, 148LL * 16));
        launch_pdl(k_split_reduce_warp, dim3(blocks > 0 ? blocks : 1), dim3(256), 0, true, s, a, c.nsplit, 0);
    } else {
        const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, 148LL * 8));
        launch_pdl(k_split_reduce, dim3(blocks > 0 ? blocks : 1), dim3(256), 0, true, s, a, c.nsplit, 0);
    }
}

}  // namespace skan
