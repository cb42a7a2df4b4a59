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
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cmath>

#include "skan_internal.hpp"
#include "skan_tc.cuh"

namespace skan {
namespace {

// kind::f16 self-test: one CTA, D[128 x N] = A[128 x K] B[K x N] with A and B
// rounded to fp16 and staged K-major (element (r, k) at (k / 8) * LBO +
// (r / 8) * 128 + (r % 8) * 16 + (k % 8) * 2), K <= 64.
__global__ void __launch_bounds__(128, 1) k_debug_gemm_f16(const float* __restrict__ A, const float* __restrict__ B,
                                                          float* __restrict__ D, int N, int K) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t s_bar;
    __shared__ uint32_t s_tmem;
    unsigned char* a_s = smem;
    unsigned char* b_s = smem + 128 * K * 2;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t lbo_a = (128 / 8) * 128, lbo_b = (N / 8) * 128;
    for (int q = tid; q < 128 * K; q += 128) {
        const int r = q / K, k = q % K;
        *reinterpret_cast<__half*>(a_s + (k >> 3) * lbo_a + (r >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2) = __float2half_rn(A[q]);
    }
    for (int q = tid; q < N * K; q += 128) {
        const int k = q / N, n = q % N;
        *reinterpret_cast<__half*>(b_s + (k >> 3) * lbo_b + (n >> 3) * 128 + (n & 7) * 16 + (k & 7) * 2) = __float2half_rn(B[q]);
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
    if (warp == 0) {
        const uint32_t idesc = tc::idesc_f16(128, N);
        for (int s = 0; s < K / 16; ++s)
            tc::mma_f16_ss_warp(tmem, tc::make_desc(tc::smem_addr(a_s) + s * 2 * lbo_a, lbo_a, 128),
                                tc::make_desc(tc::smem_addr(b_s) + s * 2 * lbo_b, lbo_b, 128), idesc, s > 0);
        tc::mma_commit_warp(&s_bar);
    }
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(tc::smem_addr(&s_bar))
            : "memory");
    }
    tc::fence_after_sync();
    const int row = warp * 32 + lane;
    for (int c = 0; c < N; c += 8) {
        float v[8];
        tc::tmem_ld8(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c, v);
        for (int q = 0; q < 8; ++q) D[row * N + c + q] = v[q];
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_free<256>(tmem);
}

__global__ void __launch_bounds__(128, 1) k_debug_gemm(const float* __restrict__ A, const float* __restrict__ B,
                                                      float* __restrict__ D, int N, int K, int passes, int M, int ts) {
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
    if (warp == 0) tc::tmem_alloc<512>(&s_tmem);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = s_tmem;
    // TS form (M = 128): row r of A_hi / A_lo in TMEM lane r, columns 256 + k / 256 + K + k
    const uint32_t ta_hi = tmem + 256, ta_lo = tmem + 256 + K;
    if (ts == 1) {
        const int r = warp * 32 + lane;
        for (int c = 0; c < K; c += 8) {
            float h[8], l[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                h[q] = A[r * K + c + q];
                l[q] = tc::tf32_lo(h[q]);
            }
            tc::tmem_st8(ta_hi + (static_cast<uint32_t>(warp * 32) << 16) + c, h);
            tc::tmem_st8(ta_lo + (static_cast<uint32_t>(warp * 32) << 16) + c, l);
        }
        tc::tmem_wait_st();
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (tid == 0) {
        const uint32_t idesc = tc::idesc_tf32(M, N);
        const uint32_t lbo_a = (M / 8) * 128, lbo_b = (N / 8) * 128;
        if (ts == 2)  // A staged in shared memory, copied into TMEM by the tensor pipe
            for (int s = 0; s < K / 8; ++s) {
                const uint32_t oa = s * 2 * lbo_a;
                tc::cp_128x256b(ta_hi + s * 8, tc::make_desc(tc::smem_addr(a_hi) + oa, lbo_a, 128));
                tc::cp_128x256b(ta_lo + s * 8, tc::make_desc(tc::smem_addr(a_lo) + oa, lbo_a, 128));
            }
        for (int s = 0; s < K / 8; ++s) {
            const uint32_t oa = s * 2 * lbo_a, ob = s * 2 * lbo_b;
            const uint64_t ah = tc::make_desc(tc::smem_addr(a_hi) + oa, lbo_a, 128);
            const uint64_t al = tc::make_desc(tc::smem_addr(a_lo) + oa, lbo_a, 128);
            const uint64_t bh = tc::make_desc(tc::smem_addr(b_hi) + ob, lbo_b, 128);
            const uint64_t bl = tc::make_desc(tc::smem_addr(b_lo) + ob, lbo_b, 128);
            if (ts) {
                tc::mma_tf32_ts(tmem, ta_hi + s * 8, bh, idesc, s > 0);
                if (passes >= 3) {
                    tc::mma_tf32_ts(tmem, ta_hi + s * 8, bl, idesc, true);
                    tc::mma_tf32_ts(tmem, ta_lo + s * 8, bh, idesc, true);
                }
            } else {
                tc::mma_tf32(tmem, ah, bh, idesc, s > 0);
                if (passes >= 3) {
                    tc::mma_tf32(tmem, ah, bl, idesc, true);
                    tc::mma_tf32(tmem, al, bh, idesc, true);
                }
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
    if (warp == 0) tc::tmem_free<512>(tmem);
}

}  // namespace
}  // namespace skan

extern "C" skan_status skan_debug_gemm_tf32(const float* dA, const float* dB, float* dD, int N, int K, int passes,
                                            void* stream) {
    if (passes == 1000) {  // kind::f16 (SS) self-test, M = 128
        if (N < 16 || N > 256 || N % 16 || K < 16 || K > 64 || K % 16)
            return skan::set_error(SKAN_SHAPE_ERROR, "debug gemm f16: N in [16,256] step 16, K in [16,64] step 16", 0,
                                   SKAN_FAULT_NONE);
        const size_t smem = static_cast<size_t>(128 * K + N * K) * 2;
        cudaFuncSetAttribute(skan::k_debug_gemm_f16, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        skan::k_debug_gemm_f16<<<1, 128, smem, static_cast<cudaStream_t>(stream)>>>(dA, dB, dD, N, K);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return skan::set_error(SKAN_CUDA_ERROR, cudaGetErrorString(e), 0, SKAN_FAULT_NONE);
        return SKAN_OK;
    }
    // passes >= 300: A from TMEM, copied there from shared memory by
    // tcgen05.cp; >= 200: A from TMEM written by tcgen05.st (TS form, M =
    // 128); >= 100: M = 64 variant (passes - 100), D receives the raw 128 TMEM lanes
    const int ts = passes >= 300 ? 2 : (passes >= 200 ? 1 : 0);
    passes -= 100 * ts + (ts ? 100 : 0);
    const int M = passes >= 100 ? 64 : 128;
    if (passes >= 100) passes -= 100;
    if (N < 8 || N > 256 || N % 16 || K < 8 || K > 64 || K % 8)
        return skan::set_error(SKAN_SHAPE_ERROR, "debug gemm: N in [16,256] step 16, K in [8,64] step 8", 0,
                               SKAN_FAULT_NONE);
    const size_t smem = static_cast<size_t>(2 * 128 * K + 2 * N * K) * 4;
    cudaFuncSetAttribute(skan::k_debug_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    skan::k_debug_gemm<<<1, 128, smem, static_cast<cudaStream_t>(stream)>>>(dA, dB, dD, N, K, passes, M, ts);
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

constexpr int kGmM = 128;        // TMEM lanes = MMA M
constexpr int kGmN = 128;        // outputs per tile (MMA N, accumulator columns)
constexpr int kGmP = 512;        // producers: 4 knot groups x 128 output columns (W); 4 x 128 TMEM lanes (A)
constexpr int kGmT = kGmP + 32;  // + one warp that issues the tensor-core MMAs

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
// waits on it); F32 the row index, gain and bias.
struct EdgeRaw {
    uint4 row;
    uint32_t k;
    float g, b;
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

// W value of a staged edge at knot m (fast-path decode); int8 codes become
// floats through the 2^23 + (u ^ 0x80) bit pattern (no I2F).
template <int FMT>
__device__ __forceinline__ float edge_w(const DevLayer& L, const EdgeRaw& r, int m) {
    if constexpr (FMT == FMT_F32) {
        return fmaf(r.g, __ldg(L.cb32 + static_cast<size_t>(r.k) * L.G + m), r.b);
    } else {
        const uint32_t w = m < 4 ? r.row.x : (m < 8 ? r.row.y : (m < 12 ? r.row.z : r.row.w));
        const float code = __int_as_float(static_cast<int>(((w >> (8 * (m & 3))) & 0xFFu) ^ 0x4B000080u)) - 8388736.0f;
        return fmaf(r.g, code, r.b);
    }
}

// Chunk K order: k = m * IC + il (knot-major).  IC is 4 (G even) or 8
// (G odd), so a chunk is KC = IC * G columns, a multiple of the MMA K (8).
//
// Operands of one chunk (both from shared memory, canonical K-major):
//   A (hat weights, 128 rows x KC), written SPARSELY: 2 nonzeros per sample
//     and input; the thread that owns a (row, input) slot clears its two
//     entries of the chunk that last used the buffer and writes the new
//     ones.  STACK (batch <= 64): rows 0-63 = A_hi of samples 0-63, rows
//     64-127 = their A_lo; else rows = 128 samples and A_hi, A_lo are two
//     tiles.  Two buffers.
//   W (KC x 256 "outputs"): rows 0-127 the 128 outputs' W_hi (raw f32: the
//     tensor core truncates to tf32), rows 128-255 their W_lo, so ONE
//     N = 256 MMA multiplies A by both planes (the N = 256 step costs ~0.78
//     of two N = 128 steps, tools/mb_mma.cu).  `wst` stages.  Compressed
//     layers: decoded by the producers from the records + codebook; dense
//     layers: the resident pre-tiled grid (DevLayer::wt, 128-output tiles)
//     arrives by TMA bulk copy in a ring of slots the producers release as
//     soon as they copied it into a stage next to its lo plane.
// MMAs per K = 8 step: STACK 1 (A x [W_hi | W_lo]); else 2 (A_hi x [W_hi |
// W_lo], A_lo x W_hi into columns 0-127).  The epilogue adds the two
// 128-column halves of the accumulator (and STACK: the A_lo rows' partial
// plane is summed by the split reduction).  (Measured alternatives: A in
// TMEM runs the MMA ~1.6x faster, but filling TMEM costs more than it
// saves: tcgen05.cp moves ~40 B/clk, and tcgen05.st needs every hat
// weight, zeros included, computed in registers.)

// Debug phase stamps (skan_debug_gemm_timeline): CTA (0,0,0) only, role 0 =
// producer thread 0 (phases: 0 top, 1 W stage free, 2 W written, 3 A tile
// free, 4 arrived), role 1 = the MMA thread (0 stage full, 1 descriptors
// ready, 2 MMAs issued).
__device__ __forceinline__ void gstamp(const FwdArgs& a, int role, int c, int ph) {
    if (a.dbg && c < 64 && (blockIdx.x | blockIdx.y | blockIdx.z) == 0) a.dbg[(role * 64 + c) * 8 + ph] = clock64();
}

// sum of partial planes z = z0, z0 + dz, ... < nz in that order (f64), four
// loads in flight: the adds are ordered, the loads need not be
__device__ __forceinline__ double ordered_plane_sum(const float* __restrict__ base, size_t plane, int z0, int dz,
                                                    int nz) {
    double v = 0.0;
    int z = z0;
    for (; z + 3 * dz < nz; z += 4 * dz) {
        float f[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) f[u] = __ldcg(base + static_cast<size_t>(z + u * dz) * plane);
#pragma unroll
        for (int u = 0; u < 4; ++u) v += static_cast<double>(f[u]);
    }
    for (; z < nz; z += dz) v += static_cast<double>(__ldcg(base + static_cast<size_t>(z) * plane));
    return v;
}

template <int FMT, int IC, bool STACK, bool F16 = false, bool DUAL = false>
__global__ void __launch_bounds__(kGmT, 1) k_layer_gemm(FwdArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t s_wfree[4];  // W stage free: the MMAs of its last chunk completed
    __shared__ __align__(8) uint64_t s_full[4];   // stage written: every producer arrives
    __shared__ __align__(8) uint64_t s_afree[2];  // A buffer free: the MMAs of its last chunk completed
    __shared__ __align__(8) uint64_t s_ring[6];   // DENSE: W tile of chunk c landed in ring slot c % ring
    __shared__ uint32_t s_tmem;
    __shared__ float s_lut[256];
    constexpr bool kDense = FMT == FMT_DENSE;
    constexpr bool kI8 = FMT == FMT_I8_R32 || FMT == FMT_I8_WIDE;
    // DUAL (fp16 only): 256 samples per CTA as two 128-sample halves, each
    // with its own A_hi / A_lo tiles and TMEM accumulator, sharing every W
    // stage: W is decoded once per 256 samples instead of once per 128.  One
    // A buffer (80 KB), so the A of chunk c+1 waits for chunk c's MMAs.
    static_assert(!DUAL || (F16 && !STACK), "dual-half tiles: fp16, unstacked");
    constexpr int S = STACK ? 64 : (DUAL ? 2 * kGmM : kGmM);  // samples per tile
    constexpr int kTPC = kGmP / kGmN;               // W: threads per output column (4)
    constexpr int kEPT = IC / kTPC;                 // W: edges (inputs) per thread and chunk
    constexpr uint32_t kLboW = (2 * kGmN / 8) * 128, kLboA = (kGmM / 8) * 128;
    constexpr uint32_t kLoRows = (kGmN / 8) * 128;  // byte offset of the lo rows inside a K group
    constexpr int kAU = IC * (DUAL ? 2 * kGmM : kGmM) / kGmP;  // A slots (row, input) per thread: 1, 2 or 4
    // F16 (int8 tables, even G, IC = 8): operands in fp16 split precision
    // (kind::f16, K = 16 per MMA: half the tensor time of 3xTF32), W scaled
    // by the layer's power of two DevLayer::wsc (folded into the gain LUT
    // and the bias scale), hi / lo halves rounded to nearest
    static_assert(!F16 || (kI8 && IC == 8), "fp16 layer GEMM: int8 tables, IC = 8");
    constexpr int kEl = F16 ? 2 : 4;                // operand element bytes
    const DevLayer& L = a.L;
    const int G = L.G, KC = IC * G;
    const uint32_t tile_t = kGmN * KC * kEl;        // one 128-output plane (a dense tile)
    const uint32_t tile_a = kGmM * KC * kEl;
    const float wsc = F16 ? L.wsc : 1.f;
    const int wst = a.gemm_wst;
    const int ring = kDense ? a.gemm_ring : 1;
    // smem: two A buffers [A_hi (| A_lo)], `wst` W stages (2 planes each),
    // then (dense) the ring slots
    const uint32_t abuf = (STACK ? 1 : (DUAL ? 4 : 2)) * tile_a, wstage = 2 * tile_t;
    constexpr int kNA = DUAL ? 1 : 2;  // A buffers
    unsigned char* s_a = smem;
    unsigned char* s_w = smem + kNA * abuf;
    unsigned char* s_ringbuf = s_w + wst * wstage;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int j0 = blockIdx.x * kGmN, s0 = blockIdx.z * S;
    const int nS = min(S, a.B - s0), nJ = min(kGmN, L.out - j0);
    const int r0 = blockIdx.y * a.rows_per_cta, rend = min(L.in, r0 + a.rows_per_cta);
    const int nchunks = rend > r0 ? (rend - r0 + IC - 1) / IC : 0;
    pdl_trigger();
    if constexpr (kI8) {
        if (tid < 256) s_lut[tid] = L.lutf[tid] * wsc;
    }
    // the A tiles are sparse: zero them once; each slot owner keeps them clean
    for (uint32_t q = tid * 16; q < kNA * abuf; q += kGmT * 16)
        *reinterpret_cast<uint4*>(s_a + q) = make_uint4(0, 0, 0, 0);
    if (tid == 0) {
        for (int q = 0; q < 4; ++q) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc::smem_addr(&s_wfree[q])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc::smem_addr(&s_full[q])), "r"(kGmP));
        }
        for (int q = 0; q < 2; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc::smem_addr(&s_afree[q])));
        for (int q = 0; q < 6; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc::smem_addr(&s_ring[q])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) tc::tmem_alloc<(DUAL ? 4 : 2) * kGmN>(&s_tmem);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = s_tmem;

    // W roles: thread (column rl, lane group eg) owns the edges of inputs
    // il = eg + kTPC * v (F16: il = kEPT * eg + v, adjacent inputs: one
    // 32-bit store writes a knot of both), v < kEPT, of its column: every edge
    // record and codebook row is gathered by exactly one thread (consecutive
    // lanes: the same column's inputs, then the next column)
    const int rl = tid / kTPC, eg = tid % kTPC;
    auto il_of = [&](int v) { return F16 ? kEPT * eg + v : eg + kTPC * v; };
    const uint32_t rbase = tc::kmajor_off(rl, 0, 2 * kGmN);
    // Producer state, double-buffered: while chunk c is written from set
    // (c & 1), chunk c+1's loads land in the other set (issued at the top of
    // iteration c, so a whole iteration hides their latency).
    struct Stage {
        EdgeRaw er[kDense ? 1 : kEPT];
        unsigned valid;      // edges of the chunk inside the layer
        int bm[kAU];         // A slot brackets
        float bt[kAU];
        uint32_t aoff[kAU];  // this slot's two nonzero offsets in the A buffer of this parity, or ~0
    };
    Stage sa, sb;
#pragma unroll
    for (int u = 0; u < kAU; ++u) sa.aoff[u] = sb.aoff[u] = 0xFFFFFFFFu;
    uint32_t recn[kI8 ? kEPT : 1], kn[kI8 ? kEPT : 1];  // I8: records of the chunk after next
    unsigned nvalid = 0;
    // A roles: slot u = (row ra = q / IC, input ila = q % IC), q = tid + 512 u: a warp's
    // 32 stores then land in 32 distinct banks (8 rows x 4 inputs, IC = 4)
    const int* bm0[kAU];
    const float* bt0[kAU];
    bool aok[kAU];
#pragma unroll
    for (int u = 0; u < kAU; ++u) {
        const int q = tid + kGmP * u, ra = q / IC, ila = q % IC;
        const int smp = STACK ? (ra & 63) : ra;
        aok[u] = smp < nS;
        bm0[u] = a.bm_in + static_cast<size_t>(r0 + ila) * a.B + s0 + smp;
        bt0[u] = a.bt_in + static_cast<size_t>(r0 + ila) * a.B + s0 + smp;
    }
    const float bs_f = static_cast<float>(L.bs) * wsc;
    const size_t cbase = static_cast<size_t>(r0 / IC);  // DENSE: first chunk of this split in the tiles
    auto issue_tile = [&](int c, int slot) {  // DENSE: TMA of chunk c's pre-tiled W into ring slot `slot`
        if constexpr (kDense) {
            if (c >= nchunks) return;
            uint64_t* bar = &s_ring[slot];
            mbar_expect_tx(bar, tile_t);
            bulk_g2s(s_ringbuf + slot * tile_t,
                     L.wt + (static_cast<size_t>(blockIdx.x) * L.wt_nch + cbase + c) * (kGmN * KC), tile_t, bar);
        }
    };
    auto load_recs = [&](int c) {  // I8 records of chunk c
        if constexpr (kI8) {
            const int ib = r0 + c * IC;
            nvalid = 0;
#pragma unroll
            for (int v = 0; v < kEPT; ++v) {
                const int i = ib + il_of(v);
                if (rl < nJ && i < rend) {
                    nvalid |= 1u << v;
                    rec_load<FMT>(L, static_cast<size_t>(i) * L.out + j0 + rl, recn[v], kn[v]);
                }
            }
        }
    };
    // issue chunk c's edge loads (from the records already in registers) and
    // bracket loads into `st`, and the records of chunk c+1
    auto load_chunk = [&](Stage& st, int c) {
        const int ib = r0 + c * IC;
        if constexpr (kI8) {
            st.valid = nvalid;
#pragma unroll
            for (int v = 0; v < kEPT; ++v) {
                if (!(st.valid >> v & 1)) continue;
                const uint32_t r = recn[v];
                const uint32_t k = FMT == FMT_I8_R32 ? (r & 0xFFFFu) : kn[v];
                const uint32_t gb = FMT == FMT_I8_R32 ? (r >> 16) : r;  // gain code | bias code << 8
                st.er[v].row = __ldg(reinterpret_cast<const uint4*>(L.cb8u + static_cast<size_t>(k) * L.rs));
                st.er[v].g = s_lut[gb & 0xFFu];  // float(gain(code) * codebook scale)
                st.er[v].b = static_cast<float>(static_cast<int8_t>((gb >> 8) & 0xFFu)) * bs_f;
            }
        } else if constexpr (FMT == FMT_F32) {
            st.valid = 0;
#pragma unroll
            for (int v = 0; v < kEPT; ++v) {
                const int i = ib + eg + kTPC * v;
                if (!(rl < nJ && i < rend)) continue;
                st.valid |= 1u << v;
                const size_t e = static_cast<size_t>(i) * L.out + j0 + rl;
                st.er[v].k = L.idx ? __ldg(L.idx + e) : 0u;
                st.er[v].g = __ldg(L.gain + e);
                st.er[v].b = __ldg(L.bias + e);
            }
        }
        const size_t step = static_cast<size_t>(c) * IC * a.B;
#pragma unroll
        for (int u = 0; u < kAU; ++u) {
            const int ila = (tid + kGmP * u) % IC;
            st.bm[u] = -2;
            st.bt[u] = 0.f;
            if (aok[u] && ib + ila < rend) {
                st.bm[u] = bm0[u][step];
                st.bt[u] = bt0[u][step];
            }
        }
        if constexpr (kI8) {
            if (c + 1 < nchunks) load_recs(c + 1);
        }
    };
    int rslot = 0;  // DENSE: ring slot of chunk c (c % ring) and its phase
    unsigned rphase = 0;
    int ws = 0;     // W stage of chunk c (c % wst) and the parity of its use count
    unsigned wph = 0;
    // producer iteration c: writes chunk c from `cur` (A buffer c & 1) while
    // chunk c+1 loads into `nxt`
    auto produce = [&](Stage& cur, Stage& nxt, int c) {
        const int ab = c & 1;
        if (tid == 0) gstamp(a, 0, c, 0);
        if constexpr (kDense) {
            // ring slot of chunk c-1 was copied out by every producer (they
            // all arrived for chunk c-1): refill it with chunk c-1+ring
            if (tid == 0 && c >= 1) {
                const int pws = ws > 0 ? ws - 1 : wst - 1;
                mbar_wait_parity(&s_full[pws], ws > 0 ? wph : wph ^ 1u);
                issue_tile(c - 1 + ring, rslot > 0 ? rslot - 1 : ring - 1);
            }
        }
        if (c + 1 < nchunks) load_chunk(nxt, c + 1);
        if (c >= wst) {
            mbar_wait_parity(&s_wfree[ws], wph ^ 1u);
            if (tid == 0) gstamp(a, 0, c, 1);
        }
        unsigned char* st = s_w + ws * wstage;
        if constexpr (kDense) {
            // the landed 128-output tile (K groups of 2 KB) -> the hi rows of
            // each 4 KB K group of the stage, its tf32 remainder -> the lo rows
            mbar_wait_parity(&s_ring[rslot], rphase);
            const float4* src = reinterpret_cast<const float4*>(s_ringbuf + rslot * tile_t);
            for (int q = tid; q < static_cast<int>(tile_t / 16); q += kGmP) {
                const float4 v = src[q];
                const uint32_t o = (q >> 7) * kLboW + (q & 127) * 16;
                *reinterpret_cast<float4*>(st + o) = v;
                *reinterpret_cast<float4*>(st + o + kLoRows) =
                    make_float4(tc::tf32_lo(v.x), tc::tf32_lo(v.y), tc::tf32_lo(v.z), tc::tf32_lo(v.w));
            }
        } else if constexpr (F16) {
            // W (fp16): the thread's two edges are adjacent inputs il0 = 2 eg,
            // il0 + 1 of column rl, so knot m of both is ONE 32-bit store at
            // k = m * 8 + il0: byte (k / 8) * LBO + row part + (k % 8) * 2;
            // g and b arrive scaled by wsc (LUT, bias scale), W_hi = fp16(W),
            // W_lo = fp16(W - W_hi)
            const uint32_t ob = rbase + (kEPT * eg) * 2;
            const bool ok0 = cur.valid & 1u, ok1 = cur.valid >> 1 & 1u;
            const float2 g2 = make_float2(ok0 ? cur.er[0].g : 0.f, ok1 ? cur.er[1].g : 0.f);
            const float2 b2 = make_float2(ok0 ? cur.er[0].b : 0.f, ok1 ? cur.er[1].b : 0.f);
            const float2 off = make_float2(-8388736.0f, -8388736.0f), neg = make_float2(-1.f, -1.f);
            const uint32_t r0w[4] = {cur.er[0].row.x, cur.er[0].row.y, cur.er[0].row.z, cur.er[0].row.w};
            const uint32_t r1w[4] = {cur.er[1].row.x, cur.er[1].row.y, cur.er[1].row.z, cur.er[1].row.w};
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                if (m >= G) break;
                const uint32_t sel = static_cast<uint32_t>(m & 3) | 0x7540u;
                float2 cf = make_float2(__uint_as_float(__byte_perm(r0w[m >> 2], 0x4B000000u, sel)),
                                        __uint_as_float(__byte_perm(r1w[m >> 2], 0x4B000000u, sel)));
                cf = __fadd2_rn(cf, off);
                const float2 w = __ffma2_rn(g2, cf, b2);
                const __half2 h = __float22half2_rn(w);
                const __half2 l = __float22half2_rn(__ffma2_rn(__half22float2(h), neg, w));
                const uint32_t o = ob + m * kLboW;
                *reinterpret_cast<__half2*>(st + o) = h;
                *reinterpret_cast<__half2*>(st + o + kLoRows) = l;
            }
        } else {
            // W: every knot of this thread's edges (hi row rl, lo row 128 + rl);
            // k = m * IC + il sits at byte (k/4) * LBO + row part + (k%4) * 4
#pragma unroll
            for (int v = 0; v < kEPT; ++v) {
                const int il = eg + kTPC * v;
                const uint32_t ob = rbase + (il >> 2) * kLboW + (il & 3) * 4;
                const bool ok = cur.valid >> v & 1;
                if constexpr (kI8) {
                    // two knots per step in packed f32x2: 2^23 + u from one byte
                    // permute of the biased row (u = c ^ 0x80), minus 2^23 + 128
                    // = c exactly, then g * c + b and the tf32 remainder
                    const float g = ok ? cur.er[v].g : 0.f, bb = ok ? cur.er[v].b : 0.f;
                    const float2 g2 = make_float2(g, g), b2 = make_float2(bb, bb);
                    const float2 off = make_float2(-8388736.0f, -8388736.0f);
                    const uint32_t rw[4] = {cur.er[v].row.x, cur.er[v].row.y, cur.er[v].row.z, cur.er[v].row.w};
#pragma unroll
                    for (int m = 0; m < 16; m += 2) {
                        if (m >= G) break;
                        const uint32_t sel0 = static_cast<uint32_t>(m & 3) | 0x7540u;
                        const uint32_t sel1 = static_cast<uint32_t>((m + 1) & 3) | 0x7540u;
                        float2 cf = make_float2(__uint_as_float(__byte_perm(rw[m >> 2], 0x4B000000u, sel0)),
                                                __uint_as_float(__byte_perm(rw[(m + 1) >> 2], 0x4B000000u, sel1)));
                        cf = __fadd2_rn(cf, off);
                        const float2 w = __ffma2_rn(g2, cf, b2);
                        const float2 wt = make_float2(__uint_as_float(__float_as_uint(w.x) & 0xFFFFE000u),
                                                      __uint_as_float(__float_as_uint(w.y) & 0xFFFFE000u));
                        const float2 lo = __fadd2_rn(w, make_float2(-wt.x, -wt.y));
                        const uint32_t o0 = ob + m * (IC / 4) * kLboW, o1 = o0 + (IC / 4) * kLboW;
                        *reinterpret_cast<float*>(st + o0) = w.x;
                        *reinterpret_cast<float*>(st + o0 + kLoRows) = lo.x;
                        if (m + 1 < G) {
                            *reinterpret_cast<float*>(st + o1) = w.y;
                            *reinterpret_cast<float*>(st + o1 + kLoRows) = lo.y;
                        }
                    }
                } else {
#pragma unroll
                    for (int m = 0; m < 16; ++m) {
                        if (m >= G) break;
                        const float w = ok ? edge_w<FMT>(L, cur.er[v], m) : 0.f;
                        const uint32_t o = ob + m * (IC / 4) * kLboW;
                        *reinterpret_cast<float*>(st + o) = w;
                        *reinterpret_cast<float*>(st + o + kLoRows) = tc::tf32_lo(w);
                    }
                }
            }
        }
        // A: clear this slot's two entries of chunk c-2, write chunk c's
        if (tid == 0) gstamp(a, 0, c, 2);
        if constexpr (DUAL) {
            if (c >= 1) mbar_wait_parity(&s_afree[0], (c - 1) & 1);
        } else if (c >= 2) {
            mbar_wait_parity(&s_afree[ab], ((c >> 1) - 1) & 1);
        }
        if (tid == 0) gstamp(a, 0, c, 3);
        unsigned char* sab = s_a + (DUAL ? 0 : ab) * abuf;
#pragma unroll
        for (int u = 0; u < kAU; ++u) {
            const int q = tid + kGmP * u, ra_ = q / IC, il = q % IC;
            // DUAL: half ra_ / 128 has its own [A_hi | A_lo] tile pair
            unsigned char* sab_u = DUAL ? sab + (ra_ >> 7) * 2 * tile_a : sab;
            const int ra = DUAL ? (ra_ & 127) : ra_;
            const bool lo_row = STACK && ra >= 64;
            if constexpr (F16) {
                // fp16 hat weights: element (r, k) at (k / 8) * LBO + row part + (k % 8) * 2.
                // DUAL has one A buffer: clear what chunk c-1 wrote (the other
                // stage's record) instead of chunk c-2's
                uint32_t& old = DUAL ? nxt.aoff[u] : cur.aoff[u];
                if (old != 0xFFFFFFFFu) {
                    const uint32_t o0 = old & 0xFFFFu, o1 = old >> 16;
                    *reinterpret_cast<__half*>(sab_u + o0) = __float2half_rn(0.f);
                    *reinterpret_cast<__half*>(sab_u + o1) = __float2half_rn(0.f);
                    if constexpr (!STACK) {
                        *reinterpret_cast<__half*>(sab_u + tile_a + o0) = __float2half_rn(0.f);
                        *reinterpret_cast<__half*>(sab_u + tile_a + o1) = __float2half_rn(0.f);
                    }
                    old = 0xFFFFFFFFu;
                }
                if (cur.bm[u] >= 0) {
                    const int k0 = cur.bm[u] * IC + il, k1 = k0 + IC;
                    const uint32_t o0 = (k0 >> 3) * kLboA + (ra >> 3) * 128 + (ra & 7) * 16 + (k0 & 7) * 2;
                    const uint32_t o1 = (k1 >> 3) * kLboA + (ra >> 3) * 128 + (ra & 7) * 16 + (k1 & 7) * 2;
                    const float w0 = 1.f - cur.bt[u], w1 = cur.bt[u];
                    const __half h0 = __float2half_rn(w0), h1 = __float2half_rn(w1);
                    const __half l0 = __float2half_rn(w0 - __half2float(h0)), l1 = __float2half_rn(w1 - __half2float(h1));
                    *reinterpret_cast<__half*>(sab_u + o0) = lo_row ? l0 : h0;
                    *reinterpret_cast<__half*>(sab_u + o1) = lo_row ? l1 : h1;
                    if constexpr (!STACK) {
                        *reinterpret_cast<__half*>(sab_u + tile_a + o0) = l0;
                        *reinterpret_cast<__half*>(sab_u + tile_a + o1) = l1;
                    }
                    cur.aoff[u] = o0 | (o1 << 16);
                }
                continue;
            }
            if (cur.aoff[u] != 0xFFFFFFFFu) {
                const uint32_t o0 = cur.aoff[u] & 0xFFFFu, o1 = cur.aoff[u] >> 16;
                *reinterpret_cast<float*>(sab + o0) = 0.f;
                *reinterpret_cast<float*>(sab + o1) = 0.f;
                if constexpr (!STACK) {
                    *reinterpret_cast<float*>(sab + tile_a + o0) = 0.f;
                    *reinterpret_cast<float*>(sab + tile_a + o1) = 0.f;
                }
                cur.aoff[u] = 0xFFFFFFFFu;
            }
            if (cur.bm[u] >= 0) {
                const int k0 = cur.bm[u] * IC + il, k1 = k0 + IC;
                const uint32_t o0 = tc::kmajor_off(ra, k0, kGmM), o1 = tc::kmajor_off(ra, k1, kGmM);
                const float w0 = 1.f - cur.bt[u], w1 = cur.bt[u];
                *reinterpret_cast<float*>(sab + o0) = lo_row ? tc::tf32_lo(w0) : w0;
                *reinterpret_cast<float*>(sab + o1) = lo_row ? tc::tf32_lo(w1) : w1;
                if constexpr (!STACK) {
                    *reinterpret_cast<float*>(sab + tile_a + o0) = tc::tf32_lo(w0);
                    *reinterpret_cast<float*>(sab + tile_a + o1) = tc::tf32_lo(w1);
                }
                cur.aoff[u] = o0 | (o1 << 16);
            }
        }
        tc::fence_proxy_async();  // this thread's smem writes -> the tensor core
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_addr(&s_full[ws])) : "memory");
        if (tid == 0) gstamp(a, 0, c, 4);
        if (++rslot == ring) {
            rslot = 0;
            rphase ^= 1u;
        }
        if (++ws == wst) {
            ws = 0;
            wph ^= 1u;
        }
    };
    // the layer's own data does not depend on the previous kernel: the first
    // records (and dense W tiles) are in flight while it drains
    if (tid < kGmP) {
        if constexpr (kDense) {
            if (tid == 0)
                for (int c = 0; c < ring; ++c) issue_tile(c, c);
        }
        if (nchunks > 0) load_recs(0);
    }
    pdl_wait();  // brackets come from the previous kernel
    if (a.prev_partial) {
        // the previous GEMM layer left its split partials: this CTA reduces
        // the entries its rows and samples consume (ascending split order in
        // f64, exactly k_split_reduce's sums) and brackets them for this
        // layer, in place of a separate reduction launch (one CTA per row
        // range: the next layer is one output tile wide)
        const size_t pplane = static_cast<size_t>(a.B) * L.in;
        const int nrow = rend - r0;
        int* bm_w = const_cast<int*>(a.bm_in);
        float* bt_w = const_cast<float*>(a.bt_in);
        for (int e = tid; e < nrow * nS; e += kGmT) {
            const int sm = e / nrow, i = r0 + (e - sm * nrow), smp = s0 + sm;
            const double v = ordered_plane_sum(a.prev_partial + static_cast<size_t>(smp) * L.in + i, pplane, 0, 1,
                                               a.prev_nsplit);
            int m;
            float t;
            fast_locate(L, v, a.err, m, t);
            bm_w[static_cast<size_t>(i) * a.B + smp] = m;
            bt_w[static_cast<size_t>(i) * a.B + smp] = t;
        }
    }
    __syncthreads();  // s_lut visible (and the fused brackets)
    if (tid < kGmP) {
        // producers: W of chunk c into stage c % wst once the MMAs of chunk
        // c - wst released it; A into buffer c & 1 once chunk c-2's did
        if (nchunks > 0) load_chunk(sa, 0);
#pragma unroll 1
        for (int c = 0; c < nchunks; c += 2) {
            produce(sa, sb, c);
            if (c + 1 < nchunks) produce(sb, sa, c + 1);
        }
    } else {
        // the MMA warp: issues the chunk's tcgen05.mma in order,
        // warp-uniform (one elected lane issues); descriptors advance by
        // immediates from per-chunk bases
        const int nks = KC / (F16 ? 16 : 8);
        const uint64_t da0 = tc::make_desc(tc::smem_addr(s_a), kLboA, 128);
        const uint64_t dw0 = tc::make_desc(tc::smem_addr(s_w), kLboW, 128);
        constexpr uint64_t kStepA = (2 * kLboA) >> 4, kStepW = (2 * kLboW) >> 4;  // descriptor address units
        const uint32_t idesc2 = F16 ? tc::idesc_f16(kGmM, 2 * kGmN) : tc::idesc_tf32(kGmM, 2 * kGmN);
        const uint32_t idesc1 = F16 ? tc::idesc_f16(kGmM, kGmN) : tc::idesc_tf32(kGmM, kGmN);
#pragma unroll 1
        for (int c = 0; c < nchunks; ++c) {
            if constexpr (F16) {  // K = 16 steps (two core-matrix columns), same descriptor strides
                const int ab = DUAL ? 0 : (c & 1);
                mbar_wait_parity(&s_full[ws], wph);
                tc::fence_after_sync();
                const uint64_t da = da0 + ab * (abuf >> 4);
                const uint64_t dw = dw0 + ws * (wstage >> 4);
#pragma unroll
                for (int s = 0; s < 8; ++s) {
                    if (s >= nks) break;
#pragma unroll
                    for (int hf = 0; hf < (DUAL ? 2 : 1); ++hf) {  // DUAL: half hf's tiles -> accumulator hf
                        const uint64_t dah = da + hf * ((2 * tile_a) >> 4);
                        const uint32_t th = tmem + hf * 2 * kGmN;
                        tc::mma_f16_ss_warp(th, dah + s * kStepA, dw + s * kStepW, idesc2, (c | s) != 0);
                        if constexpr (!STACK)
                            tc::mma_f16_ss_warp(th, dah + ((tile_a >> 4) + s * kStepA), dw + s * kStepW, idesc1, 1u);
                    }
                }
                tc::mma_commit_warp(&s_afree[ab]);
                tc::mma_commit_warp(&s_wfree[ws]);
                if (++ws == wst) {
                    ws = 0;
                    wph ^= 1u;
                }
                continue;
            }
            const int ab = c & 1;
            mbar_wait_parity(&s_full[ws], wph);
            if (lane == 0) gstamp(a, 1, c, 0);
            tc::fence_after_sync();
            const uint64_t da = da0 + ab * (abuf >> 4);  // A_hi (STACK: A_hi / A_lo rows); A_lo tile next
            const uint64_t dw = dw0 + ws * (wstage >> 4);
            if (lane == 0) gstamp(a, 1, c, 1);
#pragma unroll
            for (int s = 0; s < 16; ++s) {
                if (s >= nks) break;
                if (a.gemm_skip & 16) {  // experiment: three N = 128 MMAs
                    tc::mma_tf32_ss_warp(tmem, da + s * kStepA, dw + s * kStepW, idesc1, (c | s) != 0);
                    tc::mma_tf32_ss_warp(tmem + kGmN, da + s * kStepA, dw + ((kLoRows >> 4) + s * kStepW), idesc1, (c | s) != 0);
                    if constexpr (!STACK)
                        tc::mma_tf32_ss_warp(tmem, da + ((tile_a >> 4) + s * kStepA), dw + s * kStepW, idesc1, 1u);
                } else if (a.gemm_skip & 32) {  // experiment: two N = 256 MMAs
                    tc::mma_tf32_ss_warp(tmem, da + s * kStepA, dw + s * kStepW, idesc2, (c | s) != 0);
                    if constexpr (!STACK)
                        tc::mma_tf32_ss_warp(tmem, da + ((tile_a >> 4) + s * kStepA), dw + s * kStepW, idesc2, 1u);
                } else {
                tc::mma_tf32_ss_warp(tmem, da + s * kStepA, dw + s * kStepW, idesc2, (c | s) != 0);
                if constexpr (!STACK)
                    tc::mma_tf32_ss_warp(tmem, da + ((tile_a >> 4) + s * kStepA), dw + s * kStepW, idesc1, 1u);
                }
            }
            tc::mma_commit_warp(&s_afree[ab]);
            tc::mma_commit_warp(&s_wfree[ws]);
            if (lane == 0) gstamp(a, 1, c, 2);
            if (++ws == wst) {
                ws = 0;
                wph ^= 1u;
            }
        }
    }
    if (nchunks > 0) mbar_wait_parity(&s_wfree[(nchunks - 1) % wst], ((nchunks - 1) / wst) & 1);
    tc::fence_after_sync();
    // epilogue: producer warp w reads TMEM lanes (w%4)*32.. and columns
    // (w/4)*32..+32 of both halves (W_hi and W_lo products), adds them and
    // stages the CTA's output tile in shared memory (the operand buffers are
    // free: every MMA completed); then each warp writes whole sample rows,
    // 512 contiguous bytes per instruction.  (Written straight from the
    // TMEM lanes each store was 32 scattered 16-byte pieces: ~15k cycles of
    // a ~120k-cycle CTA at bs256.)  Virtual row vr = hf * 128 + lane row:
    // STACK rows 64-127 (A_lo) go to their own partial plane, summed with
    // the A_hi plane by the split reduction.
    // Small tiles (few samples; every stacked 64-sample tile) keep the direct
    // stores: staging all rows costs more than their few scattered writes
    // (measured: +4 us at batch 3-16).
    constexpr bool kStaged = !STACK;
    if (warp < kGmP / 32 && (!kStaged || nS < 64)) {
        for (int hf = 0; hf < (DUAL ? 2 : 1); ++hf) {
            const int q4 = warp & 3, cq = warp >> 2;
            const int as = STACK ? (q4 & 1) * 32 + lane : hf * kGmM + q4 * 32 + lane;
            const size_t plane = static_cast<size_t>(a.B) * L.out;
            const int pz = STACK ? 2 * blockIdx.y + (q4 >> 1) : blockIdx.y;
            float* dst = a.partial + pz * plane + static_cast<size_t>(s0 + min(as, nS > 0 ? nS - 1 : 0)) * L.out + j0;
            const uint32_t tacc = tmem + hf * 2 * kGmN;
#pragma unroll 1
            for (int c8 = cq * 32; c8 < cq * 32 + 32 && c8 < nJ; c8 += 8) {  // (warp-uniform: narrow tiles skip)
                float v[8], w[8];
                if (nchunks > 0) {
                    tc::tmem_ld8(tacc + (static_cast<uint32_t>(q4 * 32) << 16) + c8, v);
                    tc::tmem_ld8(tacc + (static_cast<uint32_t>(q4 * 32) << 16) + kGmN + c8, w);
                    const float inv = F16 ? 1.0f / wsc : 1.0f;
#pragma unroll
                    for (int u = 0; u < 8; ++u) v[u] = (v[u] + w[u]) * inv;
                } else {
#pragma unroll
                    for (int u = 0; u < 8; ++u) v[u] = 0.f;
                }
                if (as < nS) {
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
    } else if (kStaged && warp < kGmP / 32) {
        constexpr int kOS = kGmN + 4;  // padded row: conflict-free float4 staging stores
        float* s_out = reinterpret_cast<float*>(smem);
        const float inv = F16 ? 1.0f / wsc : 1.0f;  // exact: wsc is a power of two
        for (int hf = 0; hf < (DUAL ? 2 : 1); ++hf) {  // DUAL: accumulator hf holds samples 128 hf ..
            const int q4 = warp & 3, cq = warp >> 2;
            const int vr = hf * kGmM + q4 * 32 + lane;
            const uint32_t tacc = tmem + hf * 2 * kGmN;
#pragma unroll 1
            for (int c8 = cq * 32; c8 < cq * 32 + 32 && c8 < nJ; c8 += 8) {  // (warp-uniform: narrow tiles skip)
                float v[8], w[8];
                if (nchunks > 0) {
                    tc::tmem_ld8(tacc + (static_cast<uint32_t>(q4 * 32) << 16) + c8, v);
                    tc::tmem_ld8(tacc + (static_cast<uint32_t>(q4 * 32) << 16) + kGmN + c8, w);
#pragma unroll
                    for (int u = 0; u < 8; ++u) v[u] = (v[u] + w[u]) * inv;
                } else {
#pragma unroll
                    for (int u = 0; u < 8; ++u) v[u] = 0.f;
                }
                float4* o = reinterpret_cast<float4*>(s_out + vr * kOS + c8);
                o[0] = make_float4(v[0], v[1], v[2], v[3]);
                o[1] = make_float4(v[4], v[5], v[6], v[7]);
            }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kGmP) : "memory");  // the producer warps only
        const size_t plane = static_cast<size_t>(a.B) * L.out;
        const bool vec = (L.out & 3) == 0;
        const int col = 4 * lane;
#pragma unroll 1
        for (int vr = warp; vr < (DUAL ? 2 * kGmM : kGmM); vr += kGmP / 32) {
            const int smp = STACK ? (vr & 63) : vr;
            const int pz = STACK ? 2 * blockIdx.y + (vr >> 6) : blockIdx.y;
            if (smp >= nS) continue;
            float* dst = a.partial + pz * plane + static_cast<size_t>(s0 + smp) * L.out + j0;
            const float4 v = *reinterpret_cast<const float4*>(s_out + vr * kOS + col);
            if (vec && col + 4 <= nJ) {
                *reinterpret_cast<float4*>(dst + col) = v;
            } else {
                const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (col + u < nJ) dst[col + u] = e[u];
            }
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_free<(DUAL ? 4 : 2) * kGmN>(tmem);
}

// Pre-tiled dense grid for the layer GEMM (built at upload; the only
// resident copy of such a layer): tile (jt, ch) = the chunk's KC x 128 W
// block in exactly the shared-memory byte layout above, zero-padded past
// `out` and `in`, tiles of one output block consecutive along the inputs (one
// TMA bulk copy per chunk).  Builds the chunks [ch0, ch1) of every output
// block from `src`, the natural [i][out][G] grid whose row 0 is input ch0 * IC.
__global__ void k_dense_tiles(const float* __restrict__ src, float* __restrict__ wt, int in, int out, int G,
                              int IC, int nch, int ch0, int ch1, size_t total) {
    const int KC = IC * G;
    const size_t per = static_cast<size_t>(kGmN) * KC;
    const int nc = ch1 - ch0;
    for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; q < total;
         q += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t tile = q / per;
        const int f = static_cast<int>(q % per);
        const int jt = static_cast<int>(tile / nc), ch = ch0 + static_cast<int>(tile % nc);
        // invert kmajor_off(r, k, 128) / 4 = (k/4)*512 + (r/8)*32 + (r%8)*4 + k%4
        const int k = (f >> 9) * 4 + (f & 3), r = ((f >> 5) & 15) * 8 + ((f >> 2) & 7);
        const int m = k / IC, i = ch * IC + k % IC, j = jt * kGmN + r;
        wt[(static_cast<size_t>(jt) * nch + ch) * per + f] =
            (i < in && j < out) ? src[(static_cast<size_t>(i - ch0 * IC) * out + j) * G + m] : 0.f;
    }
}

// ---------------------------------------------------------------------------
// Dense layers at batch <= 64 (cfg4: the 1.13 GB grid streamed once per call):
// a persistent kernel, one CTA per SM.  The (output tile, chunk) work of the
// layer is flattened tile-major and cut into P equal contiguous ranges, so
// every SM streams the same number of W tiles (no waves, no tail); a range
// covers the end of one tile and the start of the next (a "segment" each),
// whose accumulators are drained to their own partial planes.
//   * TMA warp: each chunk's pre-tiled W (DevLayer::wt, 20 KB at G = 10) lands
//     by ONE bulk copy in a ring slot: that slot is the N = 128 W_hi operand
//     itself (no copy); kDnRing slots, refilled as the MMAs release them.
//     (Ten 2 KB copies per chunk into interleaved [W_hi | W_lo] stages were
//     measured issue-bound at ~160 cycles per copy.)  The chunk's brackets
//     (input-major [in][B]: IC rows of B, contiguous) arrive the same way.
//   * A warps (0-7), two sets of four taking alternate chunks: the stacked A
//     tile (hat weights of 64 samples: A_hi in rows 0-63, A_lo in rows
//     64-127) written into TMEM with tcgen05.st, so the MMAs read only W from
//     shared memory (the "TS" form, ~N/2 cycles per K = 8 step).
//   * lo warps (8-15), two sets of four taking alternate chunks: W_lo =
//     W - tf32(W), read from L2 (the TMA just brought the tile there) rather
//     than from the ring: shared memory bandwidth, not the tensor core, is
//     what a chunk costs (TMA 20 KB + MMA 40 KB + W_lo 20 KB written).
//   * MMA warp: per K = 8 step, A x W_hi and A x W_lo (M = 128, N = 128,
//     kind::tf32, A in TMEM) into the same accumulator (the A_lo x W_lo
//     product it also adds is ~2^-22 of the term); at a segment end it
//     commits the accumulator to the A set that ran the segment's last
//     chunk, which reads TMEM and writes planes 2 * segment + (A_lo rows).
// One "full" and one "done" barrier per chunk slot (kDnQ): full = A set +
// lo set + the W_hi bulk copy; done = the chunk's MMAs completed (frees its
// ring slot, lo buffer and TMEM A buffer at once).  Every waiter is at most
// one phase behind the barrier it waits on (a parity wait is exact only
// within one phase): see the per-wait notes.
// k_dense_reduce sums a tile's planes in ascending order in f64.
constexpr int kDnRing = 7;
constexpr int kDnLo = 3;
constexpr int kDnA = 4;    // TMEM A buffers (columns kDnAcol + 64 * b)
constexpr int kDnQ = 8;    // full / done barrier slots (> kDnRing: the TMA warp runs kDnRing chunks ahead)
constexpr int kDnTileTab = 512;  // k_dense_reduce: output tiles whose segment counts are tabulated
constexpr int kDnSeg = 8;  // accumulator-complete barriers (> segments an A set can run ahead: kDnA + 1)
constexpr int kDnBr = 8;   // bracket slots (>= kDnRing + 1)
constexpr int kDnT = kGmP + 64;       // A + lo warps, MMA warp, TMA warp
constexpr uint32_t kDnAcol = kGmN;    // TMEM: accumulator columns [0, 128), A buffers from 128

__host__ __device__ __forceinline__ long long dn_start(int c, long long T, int P) { return T * c / P; }
// the CTA whose chunk range holds flattened chunk x
__host__ __device__ __forceinline__ int dn_owner(long long x, long long T, int P) {
    return static_cast<int>(((x + 1) * P - 1) / T);
}
// With fewer units than CTAs some ranges are empty: a tile's segments are
// numbered densely over the NON-empty CTAs.  dn_rank = how many non-empty
// CTAs lie in [f, c) (c - f when every CTA has work).
__host__ __device__ __forceinline__ int dn_rank(long long T, int P, int f, int c) {
    if (T >= P) return c - f;
    int r = 0;
    for (int q = f; q < c; ++q) r += dn_start(q + 1, T, P) > dn_start(q, T, P);
    return r;
}
// segments of tile jt (units per tile u)
__host__ __device__ __forceinline__ int dn_nseg(int jt, int u, long long T, int P) {
    const int f = dn_owner(static_cast<long long>(jt) * u, T, P);
    return dn_rank(T, P, f, dn_owner(static_cast<long long>(jt + 1) * u - 1, T, P) + 1);
}

// debug stamps (skan_debug_gemm_timeline): CTA 0 of a wide layer, 4 roles
// x chunk u < 64 x phase < 8
__device__ __forceinline__ void dstamp(const FwdArgs& a, int role, int u, int ph) {
    if (a.dbg && u < 64 && blockIdx.x == 0 && a.L.out >= 1024) a.dbg[(role * 64 + u) * 8 + ph] = clock64();
}

// One chunk of a persistent dense kernel: for k < nb, A x W_hi then
// A x W_lo (TS form, A in TMEM at a_tmem + 8k, B descriptors advancing by
// `step` per K step: K = 8 for kind::tf32, 16 for kind::f16, both 8 TMEM
// columns of A and two core-matrix columns of B), all from ONE elect and one
// asm block.  acc_first = 0 starts a new accumulation with the first MMA.
template <bool F16>
__device__ __forceinline__ void mma_chunk_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t dh, uint64_t dl,
                                             uint32_t idesc, uint32_t acc_first, int nb, uint64_t step) {
    if constexpr (F16) {
        asm volatile(
            "{\n\t.reg .pred pe, q0, pt, p1, p2, p3, p4, p5;\n\t.reg .b32 ta;\n\t.reg .b64 bh, bl;\n\t"
            "elect.sync _|pe, 0xffffffff;\n\t"
            "setp.ne.b32 q0, %5, 0;\n\tsetp.eq.b32 pt, 0, 0;\n\t"
            "setp.gt.s32 p1, %6, 1;\n\tand.pred p1, p1, pe;\n\t"
            "setp.gt.s32 p2, %6, 2;\n\tand.pred p2, p2, pe;\n\t"
            "setp.gt.s32 p3, %6, 3;\n\tand.pred p3, p3, pe;\n\t"
            "setp.gt.s32 p4, %6, 4;\n\tand.pred p4, p4, pe;\n\t"
            "setp.gt.s32 p5, %6, 5;\n\tand.pred p5, p5, pe;\n\t"
            "mov.b32 ta, %1;\n\tmov.b64 bh, %2;\n\tmov.b64 bl, %3;\n\t"
            "@pe tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bh, %4, q0;\n\t"
            "@pe tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bl, %4, pt;\n\t"
            "add.u32 ta, ta, 8;\n\tadd.s64 bh, bh, %7;\n\tadd.s64 bl, bl, %7;\n\t"
            "@p1 tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bh, %4, pt;\n\t"
            "@p1 tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bl, %4, pt;\n\t"
            "add.u32 ta, ta, 8;\n\tadd.s64 bh, bh, %7;\n\tadd.s64 bl, bl, %7;\n\t"
            "@p2 tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bh, %4, pt;\n\t"
            "@p2 tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bl, %4, pt;\n\t"
            "add.u32 ta, ta, 8;\n\tadd.s64 bh, bh, %7;\n\tadd.s64 bl, bl, %7;\n\t"
            "@p3 tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bh, %4, pt;\n\t"
            "@p3 tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bl, %4, pt;\n\t"
            "add.u32 ta, ta, 8;\n\tadd.s64 bh, bh, %7;\n\tadd.s64 bl, bl, %7;\n\t"
            "@p4 tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bh, %4, pt;\n\t"
            "@p4 tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bl, %4, pt;\n\t"
            "add.u32 ta, ta, 8;\n\tadd.s64 bh, bh, %7;\n\tadd.s64 bl, bl, %7;\n\t"
            "@p5 tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bh, %4, pt;\n\t"
            "@p5 tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], bl, %4, pt;\n\t"
            "}\n"
            ::"r"(d_tmem), "r"(a_tmem), "l"(dh), "l"(dl), "r"(idesc), "r"(acc_first), "r"(nb), "l"(step)
            : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .pred pe, q0, pt, p1, p2, p3, p4, p5;\n\t.reg .b32 ta;\n\t.reg .b64 bh, bl;\n\t"
            "elect.sync _|pe, 0xffffffff;\n\t"
            "setp.ne.b32 q0, %5, 0;\n\tsetp.eq.b32 pt, 0, 0;\n\t"
            "setp.gt.s32 p1, %6, 1;\n\tand.pred p1, p1, pe;\n\t"
            "setp.gt.s32 p2, %6, 2;\n\tand.pred p2, p2, pe;\n\t"
            "setp.gt.s32 p3, %6, 3;\n\tand.pred p3, p3, pe;\n\t"
            "setp.gt.s32 p4, %6, 4;\n\tand.pred p4, p4, pe;\n\t"
            "setp.gt.s32 p5, %6, 5;\n\tand.pred p5, p5, pe;\n\t"
            "mov.b32 ta, %1;\n\tmov.b64 bh, %2;\n\tmov.b64 bl, %3;\n\t"
            "@pe tcgen05.mma.cta_group::1.kind::tf32 [%0], [ta], bh, %4, q0;\n\t"
            "@pe tcgen05.mma.cta_group::1.kind::tf32 [%0], [ta], bl, %4, pt;\n\t"
            "add.u32 ta, ta, 8;\n\tadd.s64 bh, bh, %7;\n\tadd.s64 bl, bl, %7;\n\t"
            "@p1 tcgen05.mma.cta_group::1.kind::tf32 [%0], [ta], bh, %4, pt;\n\t"
            "@p1 tcgen05.mma.cta_group::1.kind::tf32 [%0], [ta], bl, %4, pt;\n\t"
            "add.u32 ta, ta, 8;\n\tadd.s64 bh, bh, %7;\n\tadd.s64 bl, bl, %7;\n\t"
            "@p2 tcgen05.mma.cta_group::1.kind::tf32 [%0], [ta], bh, %4, pt;\n\t"
            "@p2 tcgen05.mma.cta_group::1.kind::tf32 [%0], [ta], bl, %4, pt;\n\t"
            "add.u32 ta, ta, 8;\n\tadd.s64 bh, bh, %7;\n\tadd.s64 bl, bl, %7;\n\t"
            "@p3 tcgen05.mma.cta_group::1.kind::tf32 [%0], [ta], bh, %4, pt;\n\t"
            "@p3 tcgen05.mma.cta_group::1.kind::tf32 [%0], [ta], bl, %4, pt;\n\t"
            "add.u32 ta, ta, 8;\n\tadd.s64 bh, bh, %7;\n\tadd.s64 bl, bl, %7;\n\t"
            "@p4 tcgen05.mma.cta_group::1.kind::tf32 [%0], [ta], bh, %4, pt;\n\t"
            "@p4 tcgen05.mma.cta_group::1.kind::tf32 [%0], [ta], bl, %4, pt;\n\t"
            "add.u32 ta, ta, 8;\n\tadd.s64 bh, bh, %7;\n\tadd.s64 bl, bl, %7;\n\t"
            "@p5 tcgen05.mma.cta_group::1.kind::tf32 [%0], [ta], bh, %4, pt;\n\t"
            "@p5 tcgen05.mma.cta_group::1.kind::tf32 [%0], [ta], bl, %4, pt;\n\t"
            "}\n"
            ::"r"(d_tmem), "r"(a_tmem), "l"(dh), "l"(dl), "r"(idesc), "r"(acc_first), "r"(nb), "l"(step)
            : "memory");
    }
}

template <int IC>
__global__ void __launch_bounds__(kDnT, 1) k_dense_persist(FwdArgs a, int nch) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t s_full[kDnQ];       // chunk u % kDnQ: A, W_lo written, W_hi landed
    __shared__ __align__(8) uint64_t s_done[kDnQ];       // chunk u % kDnQ: its MMAs completed
    __shared__ __align__(8) uint64_t s_accfull[kDnSeg];  // segment s % kDnSeg's accumulator complete
    __shared__ __align__(8) uint64_t s_accfree;          // ... and drained
    __shared__ __align__(8) uint64_t s_bfull[kDnBr];     // the chunk's brackets landed
    __shared__ uint32_t s_tmem;
    constexpr uint32_t kLbo = (kGmN / 8) * 128;  // one K group of a 128-row operand (2 KB)
    const DevLayer& L = a.L;
    const int KC = IC * L.G, nblk = KC / 8;
    const int P = gridDim.x, c = blockIdx.x;
    const int ntile = (L.out + kGmN - 1) / kGmN;
    const long long T = static_cast<long long>(ntile) * nch;
    const long long x0 = dn_start(c, T, P), x1 = dn_start(c + 1, T, P);
    const int n = static_cast<int>(x1 - x0);
    const uint32_t tile_t = kGmN * KC * 4;
    unsigned char* s_ring = smem;
    unsigned char* s_lo = smem + kDnRing * tile_t;
    // bracket slots: [IC][B] ints, then [IC][B] floats, of one chunk
    const uint32_t br_bytes = static_cast<uint32_t>(IC) * a.B * 4;
    unsigned char* s_br = s_lo + kDnLo * tile_t;
    // chunk x of the flattened schedule is tile x / nch, chunk x % nch; the
    // tiles of one output block are consecutive in wt (wt_nch == nch)
    auto tile_src = [&](int u) { return reinterpret_cast<const char*>(L.wt) + static_cast<size_t>(x0 + u) * tile_t; };
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    pdl_trigger();
    if (tid == 0) {
        for (int q = 0; q < kDnQ; ++q) {
            mbar_init(&s_full[q], kGmP / 2 + 1);
            mbar_init(&s_done[q], 1);
        }
        for (int q = 0; q < kDnSeg; ++q) mbar_init(&s_accfull[q], 1);
        mbar_init(&s_accfree, kGmP / 4);
        for (int q = 0; q < kDnBr; ++q) mbar_init(&s_bfull[q], 1);
    }
    if (warp == 0) tc::tmem_alloc<512>(&s_tmem);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = s_tmem;
    // the chunk slot of u, and the parity of u's phase on it
    auto qwait = [&](uint64_t* bar, int u) { mbar_wait_parity(&bar[u % kDnQ], (u / kDnQ) & 1); };
    if (warp == kGmP / 32 + 1) {
        // TMA warp
        if (lane == 0) {
            // W tiles do not depend on the previous kernel: the first ring's worth now
            for (int u = 0; u < kDnRing && u < n; ++u) {
                mbar_expect_tx(&s_full[u % kDnQ], tile_t);
                bulk_g2s(s_ring + u * tile_t, tile_src(u), tile_t, &s_full[u % kDnQ]);
            }
            pdl_wait();  // brackets come from the previous kernel
            int ch = static_cast<int>(x0 % nch);
#pragma unroll 1
            for (int u = 0; u < n; ++u, ch = ch + 1 == nch ? 0 : ch + 1) {
                if (u >= kDnRing) {
                    // ring slot u % kDnRing held chunk u - kDnRing.  Phase note: this
                    // warp waited for done(u - kDnRing - 1) last iteration
                    qwait(s_done, u - kDnRing);
                    dstamp(a, 2, u, 0);
                    mbar_expect_tx(&s_full[u % kDnQ], tile_t);
                    bulk_g2s(s_ring + (u % kDnRing) * tile_t, tile_src(u), tile_t, &s_full[u % kDnQ]);
                }
                // bracket slot u % kDnBr held chunk u - kDnBr, read before
                // done(u - kDnRing) (waited above; slots below kDnRing are fresh)
                const int bs = u % kDnBr;
                const int nin = min(IC, L.in - ch * IC);
                const uint32_t bytes = static_cast<uint32_t>(nin) * a.B * 4;
                mbar_expect_tx(&s_bfull[bs], 2 * bytes);
                bulk_g2s(s_br + bs * 2 * br_bytes, a.bm_in + static_cast<size_t>(ch) * IC * a.B, bytes, &s_bfull[bs]);
                bulk_g2s(s_br + bs * 2 * br_bytes + br_bytes, a.bt_in + static_cast<size_t>(ch) * IC * a.B, bytes,
                         &s_bfull[bs]);
                dstamp(a, 2, u, 1);
            }
        }
    } else if (warp == kGmP / 32) {
        // MMA warp
        const uint64_t dr0 = tc::make_desc(tc::smem_addr(s_ring), kLbo, 128);
        const uint64_t dl0 = tc::make_desc(tc::smem_addr(s_lo), kLbo, 128);
        constexpr uint64_t kStep = (2 * kLbo) >> 4;
        const uint32_t idesc = tc::idesc_tf32(kGmM, kGmN);
        int seg = 0;
        int ch = static_cast<int>(x0 % nch);
#pragma unroll 1
        for (int u = 0; u < n; ++u, ch = ch + 1 == nch ? 0 : ch + 1) {
            const bool first = u == 0 || ch == 0;
            const bool last = u == n - 1 || ch + 1 == nch;
            if (first && u > 0) mbar_wait_parity(&s_accfree, (seg - 1) & 1);  // previous segment drained
            qwait(s_full, u);
            tc::fence_after_sync();
            if (lane == 0) dstamp(a, 1, u, 0);
            const uint32_t ta = tmem + kDnAcol + (u % kDnA) * 64;
            const uint64_t dh = dr0 + (u % kDnRing) * (tile_t >> 4), dl = dl0 + (u % kDnLo) * (tile_t >> 4);
            mma_chunk_ts<false>(tmem, ta, dh, dl, idesc, first ? 0u : 1u, nblk, kStep);
            tc::mma_commit_warp(&s_done[u % kDnQ]);
            if (last) {
                tc::mma_commit_warp(&s_accfull[seg % kDnSeg]);
                ++seg;
            }
            if (lane == 0) dstamp(a, 1, u, 1);
        }
    } else if (warp < kGmP / 64) {
        // A warps.  Warp w owns TMEM lanes (w % 4) * 32.. (row r = its lane
        // there: sample r & 63, A_lo for r >= 64) and writes every 8-column
        // block of the chunk's K = IC * G columns (knot-major: column
        // k = m * IC + input).  The set that ran a segment's last chunk drains
        // the accumulator.
        const int q4 = warp & 3, set = warp >> 2;
        const int row = q4 * 32 + lane;
        const int smp = row & 63;
        const bool lo_row = row >= 64;
        const int nS = min(64, a.B);
        const bool aok = smp < nS;
        int seg = 0;
        int ch = static_cast<int>(x0 % nch), jt = static_cast<int>(x0 / nch);
#pragma unroll 1
        for (int u = 0; u < n; ++u) {
            const bool last = u == n - 1 || ch + 1 == nch;
            const int jt_u = jt;
            const int ch_u = ch;
            if (++ch == nch) {
                ch = 0;
                ++jt;
            }
            const bool mine = (a.gemm_skip & 1) ? set == 0 : (u & 1) == set;  // debug: bit 0 = one A set
            if (!mine) {
                seg += last;
                continue;
            }
            if (q4 == 0 && lane == 0) dstamp(a, set == 0 ? 0 : 3, u, 0);
            // brackets of (my sample, the chunk's inputs).  Phase note: this set
            // read chunk u - 2's slot, so u - kDnBr's phase is complete
            const int bs = u % kDnBr;
            mbar_wait_parity(&s_bfull[bs], (u / kDnBr) & 1);
            const int* sbm = reinterpret_cast<const int*>(s_br + bs * 2 * br_bytes);
            const float* sbt = reinterpret_cast<const float*>(s_br + bs * 2 * br_bytes + br_bytes);
            int m[IC];
            float w0[IC], w1[IC];
#pragma unroll
            for (int il = 0; il < IC; ++il) {
                const bool ok = aok && ch_u * IC + il < L.in;
                m[il] = ok ? sbm[il * a.B + smp] : -8;
                const float t = ok ? sbt[il * a.B + smp] : 0.f;
                w0[il] = lo_row ? tc::tf32_lo(1.f - t) : 1.f - t;
                w1[il] = lo_row ? tc::tf32_lo(t) : t;
            }
            // TMEM A buffer u % kDnA held chunk u - kDnA.  Phase note: at chunk
            // u - 2 this set waited for done(u - 2 - kDnA)
            if (u >= kDnA) qwait(s_done, u - kDnA);
            tc::fence_after_sync();
            if (q4 == 0 && lane == 0) dstamp(a, set == 0 ? 0 : 3, u, 1);
            const uint32_t ta = tmem + (static_cast<uint32_t>(q4 * 32) << 16) + kDnAcol + (u % kDnA) * 64;
            // every column's value in registers (fully unrolled, KC <= 48: two
            // compares and two selects each, knot and input compile-time), then
            // as few wide tcgen05.st as the width allows
            float v[48];
#pragma unroll
            for (int k = 0; k < 48; ++k) {
                const int mk = k / IC, il = k % IC;
                v[k] = mk == m[il] ? w0[il] : (mk == m[il] + 1 ? w1[il] : 0.f);
            }
            if (KC == 40 || KC == 48) {
                tc::tmem_st32(ta, v);
                if (KC == 40) tc::tmem_st8(ta + 32, *reinterpret_cast<const float(*)[8]>(v + 32));
                else tc::tmem_st16(ta + 32, v + 32);
            } else {
#pragma unroll
                for (int b = 0; b < 6; ++b) {
                    if (b >= nblk) break;
                    tc::tmem_st8(ta + 8 * b, *reinterpret_cast<const float(*)[8]>(v + 8 * b));
                }
            }
            tc::tmem_wait_st();
            tc::fence_before_sync();
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_addr(&s_full[u % kDnQ])) : "memory");
            if (q4 == 0 && lane == 0) dstamp(a, set == 0 ? 0 : 3, u, 2);
            if (!last) continue;
            // segment end: drain the accumulator into planes 2*seg' + (A_lo rows),
            // seg' = this CTA's index among the tile's CTAs
            mbar_wait_parity(&s_accfull[seg % kDnSeg], (seg / kDnSeg) & 1);
            tc::fence_after_sync();
            const int segi = dn_rank(T, P, dn_owner(static_cast<long long>(jt_u) * nch, T, P), c);
            const int as = (q4 & 1) * 32 + lane;
            const int j0 = jt_u * kGmN, nJ = min(kGmN, L.out - j0);
            const size_t plane = static_cast<size_t>(a.B) * L.out;
            float* dst = a.partial + (2 * segi + (q4 >> 1)) * plane + static_cast<size_t>(min(as, nS - 1)) * L.out + j0;
#pragma unroll 1
            for (int c8 = 0; c8 < kGmN; c8 += 8) {
                float v[8];
                tc::tmem_ld8(tmem + (static_cast<uint32_t>(q4 * 32) << 16) + c8, v);
                if (as < nS) {
                    if (c8 + 8 <= nJ && (L.out & 3) == 0) {
                        *reinterpret_cast<float4*>(dst + c8) = make_float4(v[0], v[1], v[2], v[3]);
                        *reinterpret_cast<float4*>(dst + c8 + 4) = make_float4(v[4], v[5], v[6], v[7]);
                    } else {
#pragma unroll
                        for (int e = 0; e < 8; ++e)
                            if (c8 + e < nJ) dst[c8 + e] = v[e];
                    }
                }
            }
            tc::fence_before_sync();
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_addr(&s_accfree)) : "memory");
            ++seg;
        }
    } else {
        // lo warps: W_lo of chunk u from the tile in L2 into lo buffer u % kDnLo
        const int set = (warp - kGmP / 64) >> 2;
        const int lt = tid - kGmP / 2 - set * (kGmP / 4);
        const int lstep = (a.gemm_skip & 2) ? 1 : 2;  // debug: bit 1 = one lo set
        constexpr int kPer = 16;                      // float4 per thread and chunk, at most (KC <= 64)
        const int nq = static_cast<int>(tile_t / 16);
#pragma unroll 1
        for (int u = lstep == 1 ? (set == 0 ? 0 : n) : set; u < n; u += lstep) {
            const float4* hi = reinterpret_cast<const float4*>(tile_src(u));
            float4 v[kPer];
#pragma unroll
            for (int r = 0; r < kPer; ++r) {
                const int q = lt + r * (kGmP / 4);
                if (q < nq) v[r] = __ldg(hi + q);
            }
            // lo buffer u % kDnLo held chunk u - kDnLo.  Phase note: at chunk
            // u - lstep this set waited for done(u - lstep - kDnLo)
            if (u >= kDnLo) qwait(s_done, u - kDnLo);
            if (lt == 0 && set == 0) dstamp(a, 2, u, 3);
            float4* lo = reinterpret_cast<float4*>(s_lo + (u % kDnLo) * tile_t);
#pragma unroll
            for (int r = 0; r < kPer; ++r) {
                const int q = lt + r * (kGmP / 4);
                if (q < nq)
                    lo[q] = make_float4(tc::tf32_lo(v[r].x), tc::tf32_lo(v[r].y), tc::tf32_lo(v[r].z), tc::tf32_lo(v[r].w));
            }
            tc::fence_proxy_async();
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_addr(&s_full[u % kDnQ])) : "memory");
            if (lt == 0 && set == 0) dstamp(a, 2, u, 4);
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_free<512>(tmem);
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
        reduce_finish(a, p, ordered_plane_sum(a.partial + p, plane, 0, 1, nsplit), add_bias);
    }
}

// The same reduction when a next layer needs brackets, through a 32 x 32
// (sample x output) tile: the partial loads and y stores run along the
// outputs, the input-major bracket stores ([j][B]) along the samples, both
// coalesced (one thread per entry wrote the brackets 4 bytes at a B-sample
// stride: ~12 us at bs256 for 360k entries).  One entry per thread, 1024
// threads per tile.  Same sums, same order as k_split_reduce.
__global__ void __launch_bounds__(1024) k_split_reduce_t(FwdArgs a, int nsplit, int add_bias) {
    __shared__ int s_m[32][33];
    __shared__ float s_t[32][33];
    pdl_trigger();
    pdl_wait();
    const DevLayer& L = a.L;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 32: one entry per thread
    const int j0 = blockIdx.x * 32, s0 = blockIdx.y * 32;
    const size_t plane = static_cast<size_t>(a.B) * L.out;
    const int j = j0 + tx, sm = s0 + ty;
    int m = 0;
    float t = 0.f;
    if (sm < a.B && j < L.out) {
        const size_t p = static_cast<size_t>(sm) * L.out + j;
        double w = ordered_plane_sum(a.partial + p, plane, 0, 1, nsplit);
        if (add_bias && L.bias_sum) w += L.bias_sum[j];
        a.y[p] = w;
        fast_locate(a.N, w, a.err, m, t);
    }
    s_m[ty][tx] = m;
    s_t[ty][tx] = t;
    __syncthreads();
    const int jj = j0 + ty, s2 = s0 + tx;
    if (jj < L.out && s2 < a.B) {
        a.bm_out[static_cast<size_t>(jj) * a.B + s2] = s_m[tx][ty];
        a.bt_out[static_cast<size_t>(jj) * a.B + s2] = s_t[tx][ty];
    }
}

// Many splits, few entries (narrow layers): one warp per entry, lane l sums
// splits l, l+32, ... in order, then a fixed butterfly.
// LP lanes per entry (32 / LP consecutive entries per warp): with fewer
// splits, 8 or 16 lanes each keep more loads in flight and a warp's loads
// cover LP planes x 32 / LP adjacent entries instead of 32 planes x 1.
template <int LP>
__global__ void k_split_reduce_warp(FwdArgs a, int nsplit, int add_bias) {
    pdl_trigger();
    pdl_wait();
    const size_t plane = static_cast<size_t>(a.B) * a.L.out;
    const int lane = threadIdx.x & (LP - 1);
    const size_t g = (blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x) / LP;
    const size_t gstep = static_cast<size_t>(gridDim.x) * blockDim.x / LP;
    // every lane of a warp runs the same number of iterations (the shuffles)
    const size_t iters = (plane + gstep - 1) / gstep;
    for (size_t it = 0; it < iters; ++it) {
        const size_t p = g + it * gstep;
        double v = p < plane ? ordered_plane_sum(a.partial + p, plane, lane, LP, nsplit) : 0.0;
#pragma unroll
        for (int o = LP >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
        if (lane == 0 && p < plane) reduce_finish(a, p, v, add_bias);
    }
}

void launch_split_reduce_warp(const FwdArgs& a, int nsplit, int add_bias, bool pdl, cudaStream_t s);

// ---------------------------------------------------------------------------
// The same persistent dense schedule in fp16 split precision (kind::f16: K =
// 16 per MMA at the tf32 instruction's cycles, so half the tensor time):
//     W * S = W_hi + W_lo,  t = t_hi + t_lo   (fp16 each, round to nearest)
// with S = 2^e the layer's scale (DevLayer::wsc) putting max|W| * S in
// [2^14, 2^15): both halves keep 11 significant bits like tf32's, and values
// the fp16 range cuts off are below 2^-40 of the layer's largest entry.  The
// MMAs add A_hi W_hi + A_lo W_hi (stacked A rows) + A W_lo; the epilogue
// multiplies by 1/S (exact).  A "pair chunk" is two consecutive IC = 4 tiles
// of the resident layout (K = 80 at G = 10): the TMA lands both f32 tiles in a
// ring slot, the conversion warps write the fp16 W_hi / W_lo operands (K order
// = tile a's columns, then tile b's), and the A warps write the hat weights in
// the same K order into TMEM as fp16 pairs.  The f32 tiles land by TMA in a
// ring (reading them from L2 in the conversion warps instead was measured
// latency-bound).
constexpr int kD16Ring = 5;   // pair slots (two f32 IC = 4 tiles each, converted in place to [W_hi | W_lo])
constexpr int kD16Br = kD16Ring + 1;  // bracket slots (8 inputs x B each): > the ring, see the TMA warp
constexpr int kD16Cv = 2;     // conversion warp sets (of four), taking pairs in turn
constexpr int kD16As = 3;     // A warp sets (of four), taking pairs in turn
constexpr int kD16T = kD16As * 128 + kD16Cv * 128 + 64;  // A sets + conversion sets + MMA warp + TMA warp
constexpr int kD16Mma = kD16T / 32 - 2, kD16Tma = kD16T / 32 - 1;

__host__ __device__ __forceinline__ int d16_nch2(int nch) { return (nch + 1) / 2; }

template <int KC>
__global__ void __launch_bounds__(kD16T, 1) k_dense_persist16(FwdArgs a, int nch) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t s_tfull[kD16Ring];  // pair u % kD16Ring: f32 tiles landed
    __shared__ __align__(8) uint64_t s_full[kDnQ];       // pair u % kDnQ: A and the fp16 W written
    __shared__ __align__(8) uint64_t s_done[kDnQ];       // pair u % kDnQ: its MMAs completed
    __shared__ __align__(8) uint64_t s_accfull[kDnSeg];
    __shared__ __align__(8) uint64_t s_accfree;
    __shared__ __align__(8) uint64_t s_bfull[kD16Br];
    __shared__ uint32_t s_tmem;
    constexpr int IC = 4;
    constexpr uint32_t kLbo = (kGmN / 8) * 128;  // one core-matrix column of a 128-row operand (2 KB)
    const DevLayer& L = a.L;
    constexpr int KC2 = 2 * KC, nstep = KC2 / 16;  // KC = IC * G (G = KC / 4, even)
    const int P = gridDim.x, c = blockIdx.x;
    const int ntile = (L.out + kGmN - 1) / kGmN;
    const int nch2 = d16_nch2(nch);
    const long long T = static_cast<long long>(ntile) * nch2;
    const long long x0 = dn_start(c, T, P), x1 = dn_start(c + 1, T, P);
    const int n = static_cast<int>(x1 - x0);
    const uint32_t tile_t = kGmN * KC * 4;         // one f32 IC = 4 tile
    const uint32_t half_t = kGmN * KC2 * 2;        // one fp16 operand (W_hi or W_lo) of a pair
    unsigned char* s_ring = smem;                                  // kD16Ring x 2 f32 tiles
    const uint32_t br_bytes = static_cast<uint32_t>(2 * IC) * a.B * 4;
    unsigned char* s_br = smem + kD16Ring * 2 * tile_t;            // kD16Br x [int m | float t] x 8 x B
    const float wsc = L.wsc, wsc_inv = 1.0f / L.wsc;
    // pair x = (tile jt = x / nch2, pair q = x % nch2): IC = 4 tiles 2q, 2q + 1 of block jt
    auto tile_src = [&](int jt, int ch) {
        return reinterpret_cast<const char*>(L.wt) + (static_cast<size_t>(jt) * nch + ch) * tile_t;
    };
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    pdl_trigger();
    if (tid == 0) {
        for (int q = 0; q < kD16Ring; ++q) {
            mbar_init(&s_tfull[q], 1);
        }
        for (int q = 0; q < kDnQ; ++q) {
            mbar_init(&s_full[q], kGmP / 4 + kD16Cv * 128);  // one A set + every conversion thread
            mbar_init(&s_done[q], 1);
        }
        for (int q = 0; q < kDnSeg; ++q) mbar_init(&s_accfull[q], 1);
        mbar_init(&s_accfree, kGmP / 4);
        for (int q = 0; q < kD16Br; ++q) mbar_init(&s_bfull[q], 1);
    }
    if (warp == 0) tc::tmem_alloc<512>(&s_tmem);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = s_tmem;
    auto qwait = [&](uint64_t* bar, int u) { mbar_wait_parity(&bar[u % kDnQ], (u / kDnQ) & 1); };
    if (warp == kD16Tma) {
        // TMA warp: the pair's f32 tiles into a ring slot, its brackets into a slot
        if (lane == 0) {
            int jt = static_cast<int>(x0 / nch2), q2 = static_cast<int>(x0 % nch2);
            auto issue = [&](int u, int jt_, int q_) {
                const int s = u % kD16Ring;
                const int nt = min(2, nch - 2 * q_);
                mbar_expect_tx(&s_tfull[s], nt * tile_t);
                for (int h = 0; h < nt; ++h)
                    bulk_g2s(s_ring + (s * 2 + h) * tile_t, tile_src(jt_, 2 * q_ + h), tile_t, &s_tfull[s]);
            };
            {  // the first ring's worth of W tiles before the previous kernel ends
                int jj = jt, qq = q2;
                for (int u = 0; u < kD16Ring && u < n; ++u) {
                    issue(u, jj, qq);
                    if (++qq == nch2) {
                        qq = 0;
                        ++jj;
                    }
                }
            }
            // optional HBM -> L2 prefetch running `dist` pairs past the ring
            // (a.gemm_ring = SKAN_DENSE_PREFETCH; 0 = off)
            const int dist = a.gemm_ring;
            int pu = kD16Ring, jp = jt, qp = q2;
            for (int r = 0; r < kD16Ring; ++r)
                if (++qp == nch2) {
                    qp = 0;
                    ++jp;
                }
            auto prefetch_to = [&](int lim) {
                for (; pu < lim && pu < n; ++pu) {
                    const int nt = min(2, nch - 2 * qp);
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(tile_src(jp, 2 * qp)),
                                 "r"(nt * tile_t)
                                 : "memory");
                    if (++qp == nch2) {
                        qp = 0;
                        ++jp;
                    }
                }
            };
            if (dist > 0) prefetch_to(kD16Ring + dist);
            pdl_wait();  // brackets come from the previous kernel
            int jr = jt, qr = q2;  // ring refill position: pair u
#pragma unroll 1
            for (int u = 0; u < n; ++u) {
                if (dist > 0) prefetch_to(u + kD16Ring + dist);
                if (u >= kD16Ring) {
                    // ring slot u % kD16Ring held pair u - kD16Ring (converted in place,
                    // then the MMAs' operand): free once those MMAs completed
                    qwait(s_done, u - kD16Ring);
                    dstamp(a, 2, u, 0);
                    issue(u, jr, qr);
                }
                if (++qr == nch2) {
                    qr = 0;
                    ++jr;
                }
                // brackets of pair u: 8 input rows of B; slot u % kD16Br held pair
                // u - kD16Br, read before done(u - kD16Ring) (waited above)
                const int bs = u % kD16Br;
                const int nin = min(2 * IC, L.in - q2 * 2 * IC);
                const uint32_t bytes = static_cast<uint32_t>(nin) * a.B * 4;
                mbar_expect_tx(&s_bfull[bs], 2 * bytes);
                bulk_g2s(s_br + bs * 2 * br_bytes, a.bm_in + static_cast<size_t>(q2) * 2 * IC * a.B, bytes, &s_bfull[bs]);
                bulk_g2s(s_br + bs * 2 * br_bytes + br_bytes, a.bt_in + static_cast<size_t>(q2) * 2 * IC * a.B, bytes,
                         &s_bfull[bs]);
                if (++q2 == nch2) {
                    q2 = 0;
                    ++jt;
                }
            }
        }
    } else if (warp == kD16Mma) {
        // MMA warp: per K = 16 step, A x W_hi and A x W_lo (M = 128, N = 128, kind::f16)
        const uint64_t dg0 = tc::make_desc(tc::smem_addr(s_ring), kLbo, 128);
        constexpr uint64_t kStep = (2 * kLbo) >> 4;
        const uint32_t idesc = tc::idesc_f16(kGmM, kGmN);
        int seg = 0;
        int q2 = static_cast<int>(x0 % nch2);
#pragma unroll 1
        for (int u = 0; u < n; ++u, q2 = q2 + 1 == nch2 ? 0 : q2 + 1) {
            const bool first = u == 0 || q2 == 0;
            const bool last = u == n - 1 || q2 + 1 == nch2;
            if (first && u > 0) mbar_wait_parity(&s_accfree, (seg - 1) & 1);
            qwait(s_full, u);
            tc::fence_after_sync();
            if (lane == 0) dstamp(a, 1, u, 0);
            const uint32_t ta = tmem + kDnAcol + (u % kDnA) * 64;
            const uint64_t dh = dg0 + (u % kD16Ring) * ((2 * half_t) >> 4), dl = dh + (half_t >> 4);
            mma_chunk_ts<true>(tmem, ta, dh, dl, idesc, first ? 0u : 1u, nstep, kStep);
            tc::mma_commit_warp(&s_done[u % kDnQ]);
            if (lane == 0) dstamp(a, 1, u, 1);
            if (last) {
                tc::mma_commit_warp(&s_accfull[seg % kDnSeg]);
                ++seg;
            }
        }
    } else if (warp < kD16As * 4) {
        // A warps, kD16As sets of four taking pairs in turn: lane row r (sample
        // r & 63, t_lo for r >= 64), every column k of the pair (k < KC: tile
        // a, knot k / 4, input k % 4; k >= KC: tile b), fp16 pairs in TMEM
        const int q4 = warp & 3, set = warp >> 2;
        const int row = q4 * 32 + lane;
        const int smp = row & 63;
        const bool lo_row = row >= 64;
        const int nS = min(64, a.B);
        const bool aok = smp < nS;
        int seg = 0;
        int q2 = static_cast<int>(x0 % nch2), jt = static_cast<int>(x0 / nch2);
#pragma unroll 1
        for (int u = 0; u < n; ++u) {
            const bool last = u == n - 1 || q2 + 1 == nch2;
            const int jt_u = jt, q2_u = q2;
            if (++q2 == nch2) {
                q2 = 0;
                ++jt;
            }
            if (u % kD16As != set) {
                seg += last;
                continue;
            }
            if (q4 == 0 && lane == 0) dstamp(a, set == 0 ? 0 : 3, u, 0);
            const int bs = u % kD16Br;
            mbar_wait_parity(&s_bfull[bs], (u / kD16Br) & 1);
            const int* sbm = reinterpret_cast<const int*>(s_br + bs * 2 * br_bytes);
            const float* sbt = reinterpret_cast<const float*>(s_br + bs * 2 * br_bytes + br_bytes);
            int m[2 * IC];
            __half w0[2 * IC], w1[2 * IC];
#pragma unroll
            for (int il = 0; il < 2 * IC; ++il) {
                const bool ok = aok && q2_u * 2 * IC + il < L.in;
                m[il] = ok ? sbm[il * a.B + smp] : -8;
                const float t = ok ? sbt[il * a.B + smp] : 0.f;
                const float u0 = 1.f - t;
                const __half h0 = __float2half_rn(u0), h1 = __float2half_rn(t);
                w0[il] = lo_row ? __float2half_rn(u0 - __half2float(h0)) : h0;
                w1[il] = lo_row ? __float2half_rn(t - __half2float(h1)) : h1;
            }
            // TMEM A buffer u % kDnA held pair u - kDnA (this set waited for
            // done(u - 2 - kDnA) at its previous pair)
            if (u >= kDnA) qwait(s_done, u - kDnA);
            tc::fence_after_sync();
            if (q4 == 0 && lane == 0) dstamp(a, set == 0 ? 0 : 3, u, 1);
            const uint32_t ta = tmem + (static_cast<uint32_t>(q4 * 32) << 16) + kDnAcol + (u % kDnA) * 64;
            // KC2 fp16 = KC columns of fp16 pairs (compile-time knot and input of each)
            float v[KC];
#pragma unroll
            for (int cc = 0; cc < KC; ++cc) {
                __half e2[2];
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const int k = 2 * cc + hh;
                    const int half = k >= KC ? 1 : 0, kk = k - KC * half;
                    const int mk = kk / IC, il = IC * half + kk % IC;
                    e2[hh] = mk == m[il] ? w0[il] : (mk == m[il] + 1 ? w1[il] : __float2half_rn(0.f));
                }
                v[cc] = __uint_as_float(static_cast<uint32_t>(__half_as_ushort(e2[0])) |
                                        static_cast<uint32_t>(__half_as_ushort(e2[1])) << 16);
            }
            if constexpr (KC == 40) {
                tc::tmem_st32(ta, v);
                tc::tmem_st8(ta + 32, *reinterpret_cast<const float(*)[8]>(v + 32));
            } else if constexpr (KC == 32) {
                tc::tmem_st32(ta, v);
            } else {
                static_assert(KC == 24, "fp16 dense: G in {6, 8, 10}");
                tc::tmem_st16(ta, v);
                tc::tmem_st8(ta + 16, *reinterpret_cast<const float(*)[8]>(v + 16));
            }
            tc::tmem_wait_st();
            tc::fence_before_sync();
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_addr(&s_full[u % kDnQ])) : "memory");
            if (q4 == 0 && lane == 0) dstamp(a, set == 0 ? 0 : 3, u, 2);
            if (!last) continue;
            mbar_wait_parity(&s_accfull[seg % kDnSeg], (seg / kDnSeg) & 1);
            tc::fence_after_sync();
            const int segi = dn_rank(T, P, dn_owner(static_cast<long long>(jt_u) * nch2, T, P), c);
            const int as = (q4 & 1) * 32 + lane;
            const int j0 = jt_u * kGmN, nJ = min(kGmN, L.out - j0);
            const size_t plane = static_cast<size_t>(a.B) * L.out;
            float* dst = a.partial + (2 * segi + (q4 >> 1)) * plane + static_cast<size_t>(min(as, nS - 1)) * L.out + j0;
#pragma unroll 1
            for (int c8 = 0; c8 < kGmN; c8 += 8) {
                float vv[8];
                tc::tmem_ld8(tmem + (static_cast<uint32_t>(q4 * 32) << 16) + c8, vv);
#pragma unroll
                for (int e = 0; e < 8; ++e) vv[e] *= wsc_inv;
                if (as < nS) {
                    if (c8 + 8 <= nJ && (L.out & 3) == 0) {
                        *reinterpret_cast<float4*>(dst + c8) = make_float4(vv[0], vv[1], vv[2], vv[3]);
                        *reinterpret_cast<float4*>(dst + c8 + 4) = make_float4(vv[4], vv[5], vv[6], vv[7]);
                    } else {
#pragma unroll
                        for (int e = 0; e < 8; ++e)
                            if (c8 + e < nJ) dst[c8 + e] = vv[e];
                    }
                }
            }
            tc::fence_before_sync();
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_addr(&s_accfree)) : "memory");
            ++seg;
        }
    } else {
        // conversion warps (kD16Cv sets of four), all on every pair, each
        // thread a share of it: the pair's f32 tiles -> fp16 W_hi and W_lo
        // (scaled), IN PLACE: every thread loads its share, the conversion
        // threads meet at a named barrier, then write the two fp16 operands
        // over the same 40 KB.  No separate operand stages, so the ring is
        // five pairs deep: the slots' TMA land latency (~5k cycles with all
        // SMs streaming) is what bounds this kernel.
        constexpr int kCvT = kD16Cv * 128;
        constexpr int kPer = (2 * 32 * KC + kCvT - 1) / kCvT;  // float4 per thread and pair (2 * nq / kCvT)
        const int lt = tid - kD16As * 128;
        const int nq = static_cast<int>(tile_t / 16);  // float4 per tile
        static_assert(32 * KC == kGmN * KC * 4 / 16 && (KC / 4) % 2 == 0, "nq; K groups come in pairs");
        int q2 = static_cast<int>(x0 % nch2);
#pragma unroll 1
        for (int u = 0; u < n; ++u) {
            const int nt = min(2, nch - 2 * q2);
            if (lt == 0) dstamp(a, 2, u, 2);
            mbar_wait_parity(&s_tfull[u % kD16Ring], (u / kD16Ring) & 1);
            if (lt == 0) dstamp(a, 2, u, 3);
            unsigned char* slot = s_ring + (u % kD16Ring) * 2 * tile_t;
            const float4* src = reinterpret_cast<const float4*>(slot);
            // share element e -> (tile h, K group g, row rr) so that a warp's 32
            // lanes are 16 rows x the two K groups of one 16-byte fp16 row
            // chunk: its fp16 stores are 256 contiguous bytes (no bank
            // conflicts) and its f32 loads two contiguous 256-byte runs.
            // float4 (g, rr) of an f32 tile = K 4g..4g+3 of row rr; fp16 K
            // index k = KC * h + 4g.
            auto share = [&](int e, int& h, int& g, int& rr) {
                h = e >= nq ? 1 : 0;
                const int i = e - h * nq, rem = i & 255;
                g = 2 * (i >> 8) + ((rem >> 4) & 1);
                rr = (rem >> 5) * 16 + (rem & 15);
            };
            float4 w[kPer];
#pragma unroll
            for (int r = 0; r < kPer; ++r) {
                const int qq = lt + r * kCvT;
                int h, g, rr;
                share(qq, h, g, rr);
                // a pair's missing second tile (odd chunk count) converts as zeros
                w[r] = qq < 2 * nq && (h == 0 || nt == 2) ? src[h * nq + g * 128 + rr] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            asm volatile("bar.sync 1, %0;" ::"n"(kCvT) : "memory");  // every share read before any write
#pragma unroll
            for (int r = 0; r < kPer; ++r) {
                const int qq = lt + r * kCvT;
                if (qq >= 2 * nq) break;
                int hsel, g, rr;
                share(qq, hsel, g, rr);
                const int k = KC * hsel + 4 * g;
                const uint32_t o = (k >> 3) * kLbo + (rr >> 3) * 128 + (rr & 7) * 16 + (k & 7) * 2;
                // packed: f32x2 scale, two-at-a-time fp16 rounding, f32x2 remainder
                const float2 sc = make_float2(wsc, wsc), neg = make_float2(-1.f, -1.f);
                const float2 a2 = __fmul2_rn(make_float2(w[r].x, w[r].y), sc), b2 = __fmul2_rn(make_float2(w[r].z, w[r].w), sc);
                const __half2 ha = __float22half2_rn(a2), hb = __float22half2_rn(b2);
                const __half2 la = __float22half2_rn(__ffma2_rn(__half22float2(ha), neg, a2));
                const __half2 lb = __float22half2_rn(__ffma2_rn(__half22float2(hb), neg, b2));
                *reinterpret_cast<uint2*>(slot + o) =
                    make_uint2(*reinterpret_cast<const uint32_t*>(&ha), *reinterpret_cast<const uint32_t*>(&hb));
                *reinterpret_cast<uint2*>(slot + half_t + o) =
                    make_uint2(*reinterpret_cast<const uint32_t*>(&la), *reinterpret_cast<const uint32_t*>(&lb));
            }
            tc::fence_proxy_async();
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_addr(&s_full[u % kDnQ])) : "memory");
            if (lt == 0) dstamp(a, 2, u, 4);
            q2 = q2 + 1 == nch2 ? 0 : q2 + 1;
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_free<512>(tmem);
}

void (*k_dense_persist16_ptr(int G))(FwdArgs, int) {
    return G == 10 ? k_dense_persist16<40> : (G == 8 ? k_dense_persist16<32> : k_dense_persist16<24>);
}

// Persistent dense layer: output j of tile jt has 2 * (CTAs holding part of
// the tile) planes, summed in ascending order in f64.
__global__ void k_dense_reduce(FwdArgs a, int nch, int P) {
    __shared__ int s_nz[kDnTileTab];  // planes per output tile (two per segment)
    const int ntile = (a.L.out + kGmN - 1) / kGmN;
    const long long T = static_cast<long long>(ntile) * nch;
    for (int jt = threadIdx.x; jt < min(ntile, kDnTileTab); jt += blockDim.x) s_nz[jt] = 2 * dn_nseg(jt, nch, T, P);
    __syncthreads();
    pdl_trigger();
    pdl_wait();
    const size_t plane = static_cast<size_t>(a.B) * a.L.out;
    for (size_t p = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; p < plane;
         p += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int jt = static_cast<int>(p % a.L.out) / kGmN;
        const int nz = jt < kDnTileTab ? s_nz[jt] : 2 * dn_nseg(jt, nch, T, P);
        reduce_finish(a, p, ordered_plane_sum(a.partial + p, plane, 0, 1, nz), 0);
    }
}

// ... one warp per output when a tile spans many CTAs (narrow layers): lane
// l sums planes l, l + 32, ... in order, then a fixed butterfly
__global__ void k_dense_reduce_warp(FwdArgs a, int nch, int P) {
    pdl_trigger();
    pdl_wait();
    const size_t plane = static_cast<size_t>(a.B) * a.L.out;
    const int ntile = (a.L.out + kGmN - 1) / kGmN;
    const long long T = static_cast<long long>(ntile) * nch;
    const int lane = threadIdx.x & 31;
    for (size_t p = (blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x) / 32; p < plane;
         p += static_cast<size_t>(gridDim.x) * blockDim.x / 32) {
        const int jt = static_cast<int>(p % a.L.out) / kGmN;
        const int nz = 2 * dn_nseg(jt, nch, T, P);
        double v = ordered_plane_sum(a.partial + p, plane, lane, 32, nz);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
        if (lane == 0) reduce_finish(a, p, v, 0);
    }
}

// ---------------------------------------------------------------------------
// Narrow dense layers (out <= 32, e.g. cfg4's 13664 -> 20 tail) at batch >= 3.
// A 128-output tensor-core tile would be 84% padding here (6.4x the grid's
// bytes streamed for a 20-wide layer), so the layer keeps its natural
// [in][out][G] grid and runs on the CUDA cores: CTA z owns a contiguous block
// of rows, stages their grid slice (one contiguous run: issued BEFORE the
// programmatic wait, so it streams while the previous kernel drains) and
// their brackets in shared memory, and each thread accumulates (sample,
// output) pairs over the rows in ascending order into split partials
// [z][B][out]; k_split_reduce(_warp) sums the splits in order in f64.
constexpr int kNarrowT = 256;

// n 4-byte words global -> shared by all threads, eight loads in flight each
__device__ __forceinline__ void stage_words(uint32_t* dst, const uint32_t* __restrict__ src, size_t n, int tid) {
    size_t e = tid;
    for (; e + 7 * kNarrowT < n; e += 8 * kNarrowT) {
        uint32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcg(src + e + u * kNarrowT);
#pragma unroll
        for (int u = 0; u < 8; ++u) dst[e + u * kNarrowT] = v[u];
    }
    for (; e < n; e += kNarrowT) dst[e] = __ldcg(src + e);
}
__device__ __forceinline__ bool bulk_ok(const void* p, size_t bytes) {
    return (reinterpret_cast<uintptr_t>(p) & 15) == 0 && (bytes & 15) == 0 && bytes > 0 && bytes < (1u << 20);
}

template <int FMT>
__global__ void __launch_bounds__(kNarrowT) k_dense_narrow(FwdArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t s_bar[2];  // [0] grid slice, [1] brackets
    const DevLayer& L = a.L;
    const int B = a.B, out = L.out, G = L.G;
    const int i0 = blockIdx.x * a.rows_per_cta, nr = min(a.rows_per_cta, L.in - i0);
    const int tid = threadIdx.x;
    float* s_grid = reinterpret_cast<float*>(smem);  // [nr][out][G]
    const size_t gfl = static_cast<size_t>(nr) * out * G;
    int* s_bm = reinterpret_cast<int*>(smem + ((gfl * 4 + 15) & ~static_cast<size_t>(15)));  // [nr][B]
    const size_t nb = static_cast<size_t>(nr) * B, boff = static_cast<size_t>(i0) * B;
    float* s_bt = reinterpret_cast<float*>(s_bm + ((nb + 3) & ~static_cast<size_t>(3)));
    const float* gsrc = FMT == FMT_DENSE ? L.cb32 + static_cast<size_t>(i0) * out * G : nullptr;
    const bool gbulk = FMT == FMT_DENSE && bulk_ok(gsrc, gfl * 4);
    const bool bbulk = bulk_ok(a.bm_in + boff, nb * 4) && bulk_ok(a.bt_in + boff, nb * 4);
    if (tid == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        if (gbulk) {  // the grid slice does not depend on the previous kernel
            mbar_expect_tx(&s_bar[0], static_cast<uint32_t>(gfl * 4));
            bulk_g2s(s_grid, gsrc, static_cast<uint32_t>(gfl * 4), &s_bar[0]);
        }
    }
    if constexpr (FMT == FMT_I8_R32) {
        // the rows' per-edge grids decoded from the records (g c[m]; the bias
        // sums are added by the reduction), before the programmatic wait
        const size_t ne = static_cast<size_t>(nr) * out;
        for (size_t e = tid; e < ne; e += kNarrowT) {
            const uint32_t r = __ldg(L.rec + static_cast<size_t>(i0) * out + e);
            const float g = __ldg(L.lutf + ((r >> 16) & 0xFFu));
            const uint4 row = __ldg(reinterpret_cast<const uint4*>(L.cb8 + static_cast<size_t>(r & 0xFFFFu) * L.rs));
            const uint32_t w[4] = {row.x, row.y, row.z, row.w};
#pragma unroll
            for (int m = 0; m < 16; ++m)
                if (m < G) s_grid[e * G + m] = g * static_cast<float>(static_cast<int8_t>((w[m >> 2] >> (8 * (m & 3))) & 0xFFu));
        }
    } else if (!gbulk) {
        stage_words(reinterpret_cast<uint32_t*>(s_grid), reinterpret_cast<const uint32_t*>(gsrc), gfl, tid);
    }
    pdl_trigger();
    pdl_wait();  // the brackets come from the previous kernel
    if (bbulk) {
        if (tid == 0) {
            mbar_expect_tx(&s_bar[1], static_cast<uint32_t>(nb * 8));
            bulk_g2s(s_bm, a.bm_in + boff, static_cast<uint32_t>(nb * 4), &s_bar[1]);
            bulk_g2s(s_bt, a.bt_in + boff, static_cast<uint32_t>(nb * 4), &s_bar[1]);
        }
    } else {
        stage_words(reinterpret_cast<uint32_t*>(s_bm), reinterpret_cast<const uint32_t*>(a.bm_in + boff), nb, tid);
        stage_words(reinterpret_cast<uint32_t*>(s_bt), reinterpret_cast<const uint32_t*>(a.bt_in + boff), nb, tid);
    }
    __syncthreads();  // the barrier inits and any word-staged data
    if (gbulk) mbar_wait(&s_bar[0], 0);
    if (bbulk) mbar_wait(&s_bar[1], 0);
    float* part = a.partial + static_cast<size_t>(blockIdx.x) * B * out;
    for (int p = tid; p < B * out; p += kNarrowT) {
        const int sm = p / out, j = p - sm * out;
        const float* g = s_grid + j * G;
        float acc = 0.f;
#pragma unroll 4
        for (int r = 0; r < nr; ++r) {
            const int m = s_bm[r * B + sm];
            const float t = s_bt[r * B + sm];
            const float c0 = g[r * out * G + m], c1 = g[r * out * G + m + 1];
            acc += fmaf(t, c1 - c0, c0);
        }
        part[p] = acc;
    }
}

// int8 narrow layers: the rows' per-edge grids decoded knot-major (see below)
template <int FMT>
__global__ void __launch_bounds__(kNarrowT) k_narrow_knot(FwdArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t s_bar;  // brackets
    const DevLayer& L = a.L;
    const int B = a.B, out = L.out, G = L.G, outp = (out + 3) & ~3;
    const int i0 = blockIdx.x * a.rows_per_cta, nr = min(a.rows_per_cta, L.in - i0);
    const int tid = threadIdx.x;
    // the rows' grid slice knot-major, [nr][G][outp]: a knot's outputs are
    // contiguous, so one 16-byte load serves four outputs of a sample
    float* s_grid = reinterpret_cast<float*>(smem);
    const size_t gfl = static_cast<size_t>(nr) * G * outp;
    int* s_bm = reinterpret_cast<int*>(smem + ((gfl * 4 + 15) & ~static_cast<size_t>(15)));  // [nr][B]
    const size_t nb = static_cast<size_t>(nr) * B, boff = static_cast<size_t>(i0) * B;
    float* s_bt = reinterpret_cast<float*>(s_bm + ((nb + 3) & ~static_cast<size_t>(3)));
    const bool bbulk = bulk_ok(a.bm_in + boff, nb * 4) && bulk_ok(a.bt_in + boff, nb * 4);
    if (tid == 0) mbar_init(&s_bar, 1);
    // the slice does not depend on the previous kernel: before the programmatic wait
    const size_t ne = static_cast<size_t>(nr) * out;
    if constexpr (FMT == FMT_I8_R32) {
        // per-edge grids decoded from the records (g c[m]; the bias sums are
        // added by the reduction)
        for (size_t e = tid; e < ne; e += kNarrowT) {
            const int r = static_cast<int>(e / out), j = static_cast<int>(e - static_cast<size_t>(r) * out);
            const uint32_t rec = __ldg(L.rec + static_cast<size_t>(i0) * out + e);
            const float g = __ldg(L.lutf + ((rec >> 16) & 0xFFu));
            const uint4 row = __ldg(reinterpret_cast<const uint4*>(L.cb8 + static_cast<size_t>(rec & 0xFFFFu) * L.rs));
            const uint32_t w[4] = {row.x, row.y, row.z, row.w};
#pragma unroll
            for (int m = 0; m < 16; ++m)
                if (m < G)
                    s_grid[(static_cast<size_t>(r) * G + m) * outp + j] =
                        g * static_cast<float>(static_cast<int8_t>((w[m >> 2] >> (8 * (m & 3))) & 0xFFu));
        }
    } else {
        // natural [i][out][G] rows, read coalesced and stored knot-major
        const float* src = L.cb32 + static_cast<size_t>(i0) * out * G;
        const size_t n = ne * G;
        size_t e = tid;
        for (; e + 7 * kNarrowT < n; e += 8 * kNarrowT) {
            float v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldg(src + e + u * kNarrowT);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const size_t q = e + u * kNarrowT, rj = q / G;
                const int m = static_cast<int>(q - rj * G), r = static_cast<int>(rj / out), j = static_cast<int>(rj - static_cast<size_t>(r) * out);
                s_grid[(static_cast<size_t>(r) * G + m) * outp + j] = v[u];
            }
        }
        for (; e < n; e += kNarrowT) {
            const size_t rj = e / G;
            const int m = static_cast<int>(e - rj * G), r = static_cast<int>(rj / out), j = static_cast<int>(rj - static_cast<size_t>(r) * out);
            s_grid[(static_cast<size_t>(r) * G + m) * outp + j] = __ldg(src + e);
        }
    }
    if (outp != out) {  // padding outputs read as zeros
        for (size_t e = tid; e < static_cast<size_t>(nr) * G * (outp - out); e += kNarrowT) {
            const size_t rm = e / (outp - out);
            s_grid[rm * outp + out + (e - rm * (outp - out))] = 0.f;
        }
    }
    pdl_trigger();
    pdl_wait();  // the brackets come from the previous kernel
    __syncthreads();  // the barrier init
    if (bbulk) {
        if (tid == 0) {
            mbar_expect_tx(&s_bar, static_cast<uint32_t>(nb * 8));
            bulk_g2s(s_bm, a.bm_in + boff, static_cast<uint32_t>(nb * 4), &s_bar);
            bulk_g2s(s_bt, a.bt_in + boff, static_cast<uint32_t>(nb * 4), &s_bar);
        }
    } else {
        stage_words(reinterpret_cast<uint32_t*>(s_bm), reinterpret_cast<const uint32_t*>(a.bm_in + boff), nb, tid);
        stage_words(reinterpret_cast<uint32_t*>(s_bt), reinterpret_cast<const uint32_t*>(a.bt_in + boff), nb, tid);
    }
    __syncthreads();  // the grid slice and any word-staged brackets
    if (bbulk) mbar_wait(&s_bar, 0);
    // work item: (sample, four consecutive outputs), rows in ascending order
    const int ng = outp >> 2;
    float* part = a.partial + static_cast<size_t>(blockIdx.x) * B * out;
    for (int q = tid; q < B * ng; q += kNarrowT) {
        const int sm = q / ng, j4 = (q - sm * ng) * 4;
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 2
        for (int r = 0; r < nr; ++r) {
            const int m = s_bm[r * B + sm];
            const float t = s_bt[r * B + sm];
            const float4 c0 = *reinterpret_cast<const float4*>(s_grid + (static_cast<size_t>(r) * G + m) * outp + j4);
            const float4 c1 = *reinterpret_cast<const float4*>(s_grid + (static_cast<size_t>(r) * G + m + 1) * outp + j4);
            acc[0] += fmaf(t, c1.x - c0.x, c0.x);
            acc[1] += fmaf(t, c1.y - c0.y, c0.y);
            acc[2] += fmaf(t, c1.z - c0.z, c0.z);
            acc[3] += fmaf(t, c1.w - c0.w, c0.w);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (j4 + u < out) part[static_cast<size_t>(sm) * out + j4 + u] = acc[u];
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
    cuda_check(cudaLaunchKernelEx(&cfg, kernel, args...), "kernel launch");
}

// k_split_reduce_warp launch: lanes per entry from the split count
void launch_split_reduce_warp(const FwdArgs& a, int nsplit, int add_bias, bool pdl, cudaStream_t s) {
    static const int lp_env = [] {
        const char* e = std::getenv("SKAN_REDUCE_LANES");  // A/B experiment: force 8, 16 or 32
        return e ? std::atoi(e) : 0;
    }();
    const int lp = lp_env == 8 || lp_env == 16 || lp_env == 32 ? lp_env : (nsplit <= 96 ? 8 : (nsplit <= 192 ? 16 : 32));
    const long long n = static_cast<long long>(a.B) * a.L.out;
    const int blocks = static_cast<int>(std::min<long long>((n * lp + 255) / 256, 148LL * 16));
    const dim3 g(blocks > 0 ? blocks : 1);
    if (lp == 8) launch_pdl(k_split_reduce_warp<8>, g, dim3(256), 0, pdl, s, a, nsplit, add_bias);
    else if (lp == 16) launch_pdl(k_split_reduce_warp<16>, g, dim3(256), 0, pdl, s, a, nsplit, add_bias);
    else launch_pdl(k_split_reduce_warp<32>, g, dim3(256), 0, pdl, s, a, nsplit, add_bias);
}

// k_split_reduce(_t) launch: the tiled form when a next layer takes brackets
// (SKAN_SPLIT_REDUCE_T=0: the one-thread-per-entry form, for A/B)
void launch_split_reduce(const FwdArgs& a, int nsplit, int add_bias, cudaStream_t s) {
    static const bool t_off = [] {
        const char* e = std::getenv("SKAN_SPLIT_REDUCE_T");
        return e && e[0] == '0';
    }();
    if (a.has_next && !t_off) {
        launch_pdl(k_split_reduce_t, dim3((a.L.out + 31) / 32, (a.B + 31) / 32), dim3(1024), 0, true, s, a, nsplit,
                   add_bias);
        return;
    }
    const long long n = static_cast<long long>(a.B) * a.L.out;
    const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, 148LL * 8));
    launch_pdl(k_split_reduce, dim3(blocks > 0 ? blocks : 1), dim3(256), 0, true, s, a, nsplit, add_bias);
}

}  // namespace

// Inputs per chunk: IC*G must be a multiple of the tf32 MMA K (8), and IC
// a multiple of 4 (16-byte W groups): 4 for even G, 8 for odd G.
int gemm_ic(int G) { return G % 2 == 0 ? 4 : 8; }

// Shared-memory plan of one configuration: two A buffers, `wst` W stages
// (3 where they fit, so the producers run two chunks ahead of the tensor
// core), and for dense layers the TMA ring (>= wst + 1 slots, up to 6).
struct GemmPlan {
    int wst, ring;
    size_t smem;
};
constexpr size_t kGemmSmemLimit = 220 * 1024;

bool gemm_plan(int G, int fmt, bool stack, GemmPlan* out) {
    const int kc = gemm_ic(G) * G;
    const size_t tile_a = static_cast<size_t>(kGmM) * kc * 4, tile_t = static_cast<size_t>(kGmN) * kc * 4;
    const size_t abuf = (stack ? 1 : 2) * tile_a, wstage = 2 * tile_t;
    static const int wst_env = [] {
        const char* e = std::getenv("SKAN_GEMM_WST");  // experiment: most W stages to try
        return e ? std::atoi(e) : 0;
    }();
    // two W stages by default: measured faster than three (the smaller
    // carve-out leaves the L1 ~90 KB instead of ~30 KB for the gathers)
    for (int wst = wst_env >= 2 && wst_env <= 4 ? wst_env : 2; wst >= 2; --wst) {
        size_t smem = 2 * abuf + wst * wstage;
        int ring = 0;
        if (fmt == FMT_DENSE) {
            if (smem >= kGemmSmemLimit) continue;
            ring = static_cast<int>(std::min<size_t>(6, (kGemmSmemLimit - smem) / tile_t));
            if (ring < 3) continue;
            smem += ring * tile_t;
        }
        if (smem > kGemmSmemLimit) continue;
        if (out) *out = GemmPlan{wst, ring, smem};
        return true;
    }
    return false;
}

bool gemm_supported(const DevLayer& L) {
    if (L.G > 16 || !gemm_plan(L.G, L.fmt, false, nullptr) || !gemm_plan(L.G, L.fmt, true, nullptr))
        return false;
    if (L.fmt == FMT_DENSE) return L.wt != nullptr;
    return L.fmt == FMT_I8_R32 || L.fmt == FMT_I8_WIDE || L.fmt == FMT_F32;
}

// Persistent dense schedule (k_dense_persist): batch <= 64, chunk tiles of
// at most 24 KB (KC <= 48) and kDnRing + kDnLo of them in shared memory.
size_t dense_persist_smem(int G) {
    const int kc = gemm_ic(G) * G;
    return (kDnRing + kDnLo) * static_cast<size_t>(kGmN) * kc * 4 + kDnBr * 2 * static_cast<size_t>(gemm_ic(G)) * 64 * 4;
}
// fp16 variant (k_dense_persist16): even G in {6, 8, 10} (IC = 4 tiles,
// pair chunks of K = 8G), a finite grid (DevLayer::wsc > 0)
bool dense_f16_ok(const DevLayer& L) {
    static const bool off = [] {
        const char* e = std::getenv("SKAN_DENSE_F16");  // A/B experiment: 0 = the tf32 persistent kernel
        return e && e[0] == '0';
    }();
    return !off && L.wsc > 0.f && (L.G == 6 || L.G == 8 || L.G == 10);
}
size_t dense_f16_smem(int G) {
    const size_t kc = 4 * static_cast<size_t>(G);
    return kD16Ring * 2 * kGmN * kc * 4 + kD16Br * 2 * 8 * 64 * 4;
}

bool dense_persist_ok(const DevLayer& L, int B) {
    static const bool off = [] {
        const char* e = std::getenv("SKAN_DENSE_PERSIST");  // A/B experiment: 0 = the split GEMM
        return e && e[0] == '0';
    }();
    return !off && L.fmt == FMT_DENSE && L.wt && B <= 64 && gemm_ic(L.G) * L.G <= 48 &&
           dense_persist_smem(L.G) <= kGemmSmemLimit;
}

// int8 layers in fp16 split precision (k_layer_gemm<..., F16>): even G with
// a finite scale; IC = 8 keeps K = 8G a multiple of the f16 MMA's 16
bool gemm_f16_ok(const DevLayer& L) {
    static const bool off = [] {
        const char* e = std::getenv("SKAN_GEMM_F16");  // A/B experiment: 0 = 3xTF32
        return e && e[0] == '0';
    }();
    return !off && (L.fmt == FMT_I8_R32 || L.fmt == FMT_I8_WIDE) && L.G % 2 == 0 && L.G <= 12 && L.wsc > 0.f;
}

LaunchCfg gemm_cfg(const DevLayer& L, int B, int num_sms) {
    LaunchCfg c{};
    if (dense_persist_ok(L, B)) {
        const int sms = num_sms > 0 ? num_sms : 148;
        c.kind = 4;
        c.persist = 1;
        c.ic = gemm_ic(L.G);
        c.spt = 64;
        c.tj = kGmN;
        c.dn_nch = (L.in + c.ic - 1) / c.ic;
        c.persist = dense_f16_ok(L) ? 2 : 1;
        const int ntile = (L.out + kGmN - 1) / kGmN;
        const int units = c.persist == 2 ? d16_nch2(c.dn_nch) : c.dn_nch;  // schedule units per tile
        const long long T = static_cast<long long>(ntile) * units;
        c.jt = sms;  // grid
        c.st = (ntile + sms - 1) / sms;  // so that jt * st >= ntile: the per-tile arrival counters fit
        int maxseg = 1;
        for (int jt = 0; jt < ntile; ++jt)
            maxseg = std::max(maxseg, dn_nseg(jt, units, T, sms));
        c.nsplit = 2 * maxseg;
        c.ichunk = L.in;
        c.smem = c.persist == 2 ? dense_f16_smem(L.G) : dense_persist_smem(L.G);
        return c;
    }
    c.kind = 4;
    c.ic = gemm_ic(L.G);
    if (gemm_f16_ok(L)) {
        c.persist = 3;
        c.ic = 8;  // the same shared-memory bytes per chunk as tf32 at IC = 4
    }
    c.spt = B <= 64 ? 64 : kGmM;  // samples per tile: 64 = A_hi / A_lo stacked in the 128 rows
    static const bool dual_off = [] {
        const char* e = std::getenv("SKAN_GEMM_DUAL");  // A/B experiment: 0 = one CTA per 128 samples
        return e && e[0] == '0';
    }();
    if (c.persist == 3 && B > kGmM && !dual_off) c.spt = 2 * kGmM;  // 256 samples per CTA, W decoded once
    const bool stack = c.spt == 64;
    c.tj = kGmN;
    GemmPlan gp{};
    gemm_plan(L.G, L.fmt, stack, &gp);
    if (c.spt == 2 * kGmM) {  // one A buffer of two [A_hi | A_lo] pairs + two W stages
        const size_t kc = static_cast<size_t>(gemm_ic(L.G)) * L.G;  // fp16 at IC = 8: the bytes of f32 at IC = 4
        gp.wst = 2;
        gp.ring = 0;
        gp.smem = 4 * kGmM * kc * 4 + 2 * 2 * kGmN * kc * 4;
    }
    // the epilogue stages the output tile in shared memory: [rows][128 + 4] f32
    if (!stack) gp.smem = std::max(gp.smem, static_cast<size_t>(c.spt == 2 * kGmM ? 2 * kGmM : kGmM) * (kGmN + 4) * 4);
    c.vj = gp.wst;
    c.rw = gp.ring;
    c.jt = (L.out + c.tj - 1) / c.tj;
    c.st = (B + c.spt - 1) / c.spt;
    const int sms = num_sms > 0 ? num_sms : 148;
    // one CTA per SM: the fewest input splits whose waves are >= 90% full
    const long long base = static_cast<long long>(c.jt) * c.st;
    const long long maxns = std::max<long long>(1, std::min<long long>(148, (L.in + c.ic - 1) / c.ic));
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
    // partial planes: one per input split, two when A_hi / A_lo are stacked
    c.nsplit = (L.in + c.ichunk - 1) / c.ichunk * (stack ? 2 : 1);
    c.smem = gp.smem;
    return c;
}

template <bool STACK>
void (*gemm_kernel(int fmt, int ic, bool f16 = false, bool dual = false))(FwdArgs) {
    const bool i4 = ic == 4;
    if constexpr (!STACK) {
        if (f16 && dual)
            return fmt == FMT_I8_R32 ? k_layer_gemm<FMT_I8_R32, 8, false, true, true>
                                     : k_layer_gemm<FMT_I8_WIDE, 8, false, true, true>;
    }
    if (f16) return fmt == FMT_I8_R32 ? k_layer_gemm<FMT_I8_R32, 8, STACK, true> : k_layer_gemm<FMT_I8_WIDE, 8, STACK, true>;
    switch (fmt) {
        case FMT_I8_R32: return i4 ? k_layer_gemm<FMT_I8_R32, 4, STACK> : k_layer_gemm<FMT_I8_R32, 8, STACK>;
        case FMT_I8_WIDE: return i4 ? k_layer_gemm<FMT_I8_WIDE, 4, STACK> : k_layer_gemm<FMT_I8_WIDE, 8, STACK>;
        case FMT_F32: return i4 ? k_layer_gemm<FMT_F32, 4, STACK> : k_layer_gemm<FMT_F32, 8, STACK>;
        default: return i4 ? k_layer_gemm<FMT_DENSE, 4, STACK> : k_layer_gemm<FMT_DENSE, 8, STACK>;
    }
}

double gemm_issued_flops(const DevLayer& L, const LaunchCfg& c, int B) {
    if (c.persist == 1 || c.persist == 2)  // one M=128 x N=256 x K=8 MMA per K step of every (tile, chunk)
        return static_cast<double>((L.out + kGmN - 1) / kGmN) * c.dn_nch * (c.ic * L.G / 8) * 2.0 * kGmM * 8 *
               (2 * kGmN);
    // per 128-sample half and K = 8 step: one M=128 x N=256 MMA, plus (not
    // stacked) one N=128; dual-half tiles run two halves per CTA
    const double ksteps = static_cast<double>((L.in + c.ic - 1) / c.ic) * c.ic * L.G / 8.0;
    const double per_step = 2.0 * kGmM * 8 * (2 * kGmN + (c.spt == 64 ? 0 : kGmN));
    const double halves = c.spt == 2 * kGmM ? 2.0 : 1.0;
    (void)B;
    return ksteps * per_step * halves * c.jt * c.st;
}

unsigned long long* g_gemm_dbg = nullptr;
int g_gemm_min_batch = kGemmMinBatch;

int launch_layer_gemm(const FwdArgs& a0, const LaunchCfg& c, bool pdl, cudaStream_t s, bool with_reduce) {
    FwdArgs a = a0;
    a.dbg = g_gemm_dbg;
    a.gemm_wst = c.vj;
    a.gemm_ring = c.rw;
    static const int skip_env = [] {
        const char* e = std::getenv("SKAN_GEMM_SKIP");
        return e ? std::atoi(e) : 0;
    }();
    a.gemm_skip = skip_env;
    if (c.persist == 1 || c.persist == 2) {  // dense persistent (tf32 / fp16)
        static const int dist_env = [] {
            const char* e = std::getenv("SKAN_DENSE_PREFETCH");  // experiment: L2 prefetch distance in chunks
            return e ? std::atoi(e) : 0;
        }();
        a.gemm_ring = dist_env;
        void (*kp)(FwdArgs, int) = c.ic == 4 ? k_dense_persist<4> : k_dense_persist<8>;
        if (c.persist == 2) ensure_smem(k_dense_persist16_ptr(a.L.G), c.smem);
        else ensure_smem(kp, c.smem);
        // (fusing the reduction into the kernel — the CTA that drains a
        // tile's last segment reduces it — measured slower: 311 -> 421 us at
        // cfg4, the reducing CTA's stream stalls behind ~8k outputs)
        if (c.persist == 2) {
            launch_pdl(k_dense_persist16_ptr(a.L.G), dim3(c.jt), dim3(kD16T), c.smem, pdl, s, a, c.dn_nch);
            if (!with_reduce) return 1;
        } else {
            launch_pdl(kp, dim3(c.jt), dim3(kDnT), c.smem, pdl, s, a, c.dn_nch);
            if (!with_reduce) return 1;
        }
        const int units = c.persist == 2 ? d16_nch2(c.dn_nch) : c.dn_nch;  // the reduction's schedule unit
        const long long n = static_cast<long long>(a.B) * a.L.out;
        if (c.nsplit >= 32) {
            const int blocks = static_cast<int>(std::min<long long>((n * 32 + 255) / 256, 148LL * 16));
            launch_pdl(k_dense_reduce_warp, dim3(blocks > 0 ? blocks : 1), dim3(256), 0, true, s, a, units, c.jt);
        } else {
            static const long long cap = [] {
                const char* e = std::getenv("SKAN_DENSE_REDUCE_BLOCKS");  // experiment: grid cap per SM
                return e ? std::max(1, std::atoi(e)) : 64;  // one output per thread at cfg4
            }();
            // (a tiled form with coalesced bracket stores, as k_split_reduce_t,
            // measured no faster here: cfg4's reduction overlaps the narrow tail)
            const int blocks = static_cast<int>(std::min<long long>((n + 255) / 256, 148LL * cap));
            launch_pdl(k_dense_reduce, dim3(blocks > 0 ? blocks : 1), dim3(256), 0, true, s, a, units, c.jt);
        }
        return 2;
    }
    const bool stack = c.spt == 64;
    const bool f16 = c.persist == 3;  // int8 layer GEMM in fp16 split precision
    const bool dual = c.spt == 2 * kGmM;  // 256 samples per CTA (two halves share W)
    void (*k)(FwdArgs) =
        stack ? gemm_kernel<true>(a.L.fmt, c.ic, f16) : gemm_kernel<false>(a.L.fmt, c.ic, f16, dual);
    ensure_smem(k, c.smem);
    static const int carve_env = [] {
        const char* e = std::getenv("SKAN_GEMM_CARVEOUT");  // experiment: shared-memory carve-out percent
        return e ? std::atoi(e) : -1;
    }();
    if (carve_env >= 0) cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carve_env);
    const int splits = (a.L.in + c.ichunk - 1) / c.ichunk;
    launch_pdl(k, dim3(c.jt, splits, c.st), dim3(kGmT), c.smem, pdl, s, a);
    if (!with_reduce) return 1;
    // bias: folded into W for compressed layers; dense layers have none
    const long long n = static_cast<long long>(a.B) * a.L.out;
    if (c.nsplit >= 16 && n < 148LL * 256) {
        launch_split_reduce_warp(a, c.nsplit, 0, true, s);
    } else {
        launch_split_reduce(a, c.nsplit, 0, s);
    }
    return 2;
}

static bool narrow_i8_on() {
    static const bool on = [] {
        const char* e = std::getenv("SKAN_NARROW_I8");  // A/B experiment: 0 = narrow int8 layers on the GEMM
        return !(e && e[0] == '0');
    }();
    return on;
}

bool dense_narrow_ok(const DevLayer& L) {
    // one input row of the grid plus the brackets of 512 samples must fit the
    // staging; int8 layers (records decoded in the kernel) with 16-byte rows
    const bool fmt_ok = (L.fmt == FMT_DENSE && !L.wt) || (L.fmt == FMT_I8_R32 && L.G <= 16 && narrow_i8_on());
    return fmt_ok && L.out <= 32 && L.G >= 2 && static_cast<size_t>(L.out + 3) * L.G * 4 + 16 + 512 * 8 <= 100 * 1024;
}

size_t dense_narrow_smem(const DevLayer& L, int B, int rows) {
    const size_t nb = (static_cast<size_t>(rows) * B + 3) & ~static_cast<size_t>(3);
    const size_t outp = L.fmt == FMT_DENSE ? static_cast<size_t>(L.out)
                                           : (static_cast<size_t>(L.out) + 3) & ~static_cast<size_t>(3);
    return ((static_cast<size_t>(rows) * outp * L.G * 4 + 15) & ~static_cast<size_t>(15)) + nb * 8;
}

LaunchCfg dense_narrow_cfg(const DevLayer& L, int B, int num_sms) {
    LaunchCfg c{};
    const int sms = num_sms > 0 ? num_sms : 148;
    c.kind = 5;
    // about two CTAs per SM, fewer rows per CTA while the staging exceeds ~100 KB
    static const int per_sm = [] {
        const char* e = std::getenv("SKAN_NARROW_PER_SM");  // experiment: CTAs per SM
        return e ? std::max(1, std::atoi(e)) : 2;
    }();
    // (int8: one CTA per SM, fewer partial planes; its staging is small)
    int splits = std::min(L.in, (L.fmt == FMT_DENSE ? per_sm : 1) * sms);
    int rows = (L.in + splits - 1) / splits;
    while (rows > 1 && dense_narrow_smem(L, B, rows) > 100 * 1024) rows = (rows + 1) / 2;
    c.ichunk = rows;
    c.nsplit = (L.in + rows - 1) / rows;
    c.jt = 1;
    c.st = 1;
    c.smem = dense_narrow_smem(L, B, rows);
    return c;
}

int launch_dense_narrow(const FwdArgs& a0, const LaunchCfg& c, bool pdl, cudaStream_t s) {
    FwdArgs a = a0;
    a.rows_per_cta = c.ichunk;
    // dense: natural [i][out][G] slice bulk-copied (cfg4's tail measured faster
    // that way); int8: knot-major decoded slice, four outputs per 16-byte load
    void (*k)(FwdArgs) = a.L.fmt == FMT_DENSE ? k_dense_narrow<FMT_DENSE> : k_narrow_knot<FMT_I8_R32>;
    ensure_smem(k, c.smem);
    launch_pdl(k, dim3(c.nsplit), dim3(kNarrowT), c.smem, pdl, s, a);
    // int8 partials exclude the edges' biases: their per-output sums are added
    // here (dense layers have none)
    const int add_bias = a.L.fmt == FMT_DENSE ? 0 : 1;
    const long long n = static_cast<long long>(a.B) * a.L.out;
    if (c.nsplit >= 16 && n < 148LL * 256) {
        launch_split_reduce_warp(a, c.nsplit, add_bias, true, s);
    } else {
        launch_split_reduce(a, c.nsplit, add_bias, s);
    }
    return 2;
}

// Dense layers the GEMM takes keep their grid ONLY in its pre-tiled layout
// (DevLayer::wt; every other kernel reads it through dense_at): number of
// floats, and the device-side build of input chunks [ch0, ch1) from a natural
// layout source (rows from input ch0 * IC).
uint64_t dense_tile_floats(int in, int out, int G) {
    const int ic = gemm_ic(G);
    return static_cast<uint64_t>((out + kGmN - 1) / kGmN) * ((in + ic - 1) / ic) * kGmN * ic * G;
}

// max |v| as float bits (non-negative floats order like their bits; NaN
// sorts above +inf)
__global__ void k_absmax_bits(const float* __restrict__ p, size_t n, unsigned* out) {
    unsigned m = 0;
    for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; q < n;
         q += static_cast<size_t>(gridDim.x) * blockDim.x)
        m = max(m, __float_as_uint(p[q]) & 0x7FFFFFFFu);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// The fp16 GEMM's power-of-two scale of a tiled dense grid: max|W| * S in
// [2^14, 2^15); 0 when the grid holds a non-finite value (no fp16 path).
float dense_fp16_scale(const float* wt, uint64_t n, cudaStream_t s) {
    unsigned* d = nullptr;
    cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(unsigned), s), "cudaMallocAsync");
    cuda_check(cudaMemsetAsync(d, 0, sizeof(unsigned), s), "cudaMemsetAsync");
    const int blocks = static_cast<int>(std::min<uint64_t>((n + 255) / 256, 148ull * 16));
    k_absmax_bits<<<blocks > 0 ? blocks : 1, 256, 0, s>>>(wt, n, d);
    unsigned bits = 0;
    cuda_check(cudaMemcpyAsync(&bits, d, sizeof(unsigned), cudaMemcpyDeviceToHost, s), "absmax");
    cuda_check(cudaFreeAsync(d, s), "cudaFreeAsync");
    cuda_check(cudaStreamSynchronize(s), "absmax");
    float mx;
    std::memcpy(&mx, &bits, 4);
    if (!std::isfinite(mx)) return 0.f;
    if (mx == 0.f) return 1.f;
    int ex = 0;
    std::frexp(mx, &ex);  // mx = f * 2^ex, f in [0.5, 1)
    return std::ldexp(1.0f, 15 - ex);
}

void build_dense_tiles(const DevLayer& L, float* wt, const float* src, int ch0, int ch1, cudaStream_t s) {
    const int ic = gemm_ic(L.G);
    const int nch = (L.in + ic - 1) / ic;
    const uint64_t total = static_cast<uint64_t>((L.out + kGmN - 1) / kGmN) * (ch1 - ch0) * kGmN * ic * L.G;
    const int blocks = static_cast<int>(std::min<uint64_t>((total + 255) / 256, 148ull * 32));
    k_dense_tiles<<<blocks > 0 ? blocks : 1, 256, 0, s>>>(src, wt, L.in, L.out, L.G, ic, nch, ch0, ch1, total);
}

}  // namespace skan

extern "C" skan_status skan_debug_gemm_timeline(unsigned long long* d_stamps) {
    skan::g_gemm_dbg = d_stamps;
    return SKAN_OK;
}

extern "C" int skan_debug_set_gemm_min_batch(int batch) {
    const int prev = skan::g_gemm_min_batch;
    skan::g_gemm_min_batch = batch > 0 ? batch : skan::kGemmMinBatch;
    return prev;
}
