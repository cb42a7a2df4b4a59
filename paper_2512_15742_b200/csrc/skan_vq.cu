// GSB-VQ nearest-row assignment on the GPU:
// holoquant::assign_indices, gsb.cpp:275-286, with nearest_row (62-73) and
// dist2 (23-30).  For every shape the codebook row of least squared
// distance, ties to the lowest row -- bit-identical to the reference:
//   * the distance is accumulated in f64 in dim order, s = s + (a-b)*(a-b),
//     each operation rounded on its own (__dsub_rn/__dmul_rn/__dadd_rn: the
//     reference build has no FMA contraction, -ffp-contract=off);
//   * rows are scanned in ascending order with a strict <, and the K range
//     is split across CTAs only into ascending row ranges, merged in range
//     order with the same strict < (so the lowest row wins every tie);
//   * NaN distances never win; k == 0 leaves row 0, as nearest_row does.
// Layout: shapes [n][dim], codebook [k][dim], row-major f64.  A CTA owns 512
// shapes (two per thread, in registers) and one K range, streamed through
// shared memory in tiles of rows that every thread reads by broadcast.
// Bound: FP64 issue (3·dim DADD/DMUL per shape-row pair; ~64 lane-ops per
// cycle per SM measured, profiles/r1/mb_fp64.txt).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>

#include "skan.h"
#include "skan_internal.hpp"

namespace skan {
namespace {

constexpr int kVqThreads = 256;
constexpr int kVqShapes = 2 * kVqThreads;  // shapes per CTA
constexpr int kVqTileBytes = 40 * 1024;    // codebook rows staged per tile

__device__ __forceinline__ double dist_step(double s, double a, double b) {
    const double d = __dsub_rn(a, b);
    return __dadd_rn(s, __dmul_rn(d, d));
}

// D > 0: compile-time dim (shapes in registers); D == 0: runtime dim <= 64.
template <int D>
__global__ void __launch_bounds__(kVqThreads) k_assign(const double* __restrict__ shapes, uint64_t n, int dim,
                                                       const double* __restrict__ cb, int k, int rows_per_split,
                                                       double* __restrict__ part_d, uint32_t* __restrict__ part_r,
                                                       uint32_t* __restrict__ out) {
    extern __shared__ __align__(16) double s_rows[];
    constexpr int kMaxD = D > 0 ? D : 64;
    const int dm = D > 0 ? D : dim;
    const uint64_t i0 = blockIdx.x * static_cast<uint64_t>(kVqShapes) + threadIdx.x;
    const uint64_t i1 = i0 + kVqThreads;
    double a0[kMaxD], a1[kMaxD];
#pragma unroll
    for (int c = 0; c < kMaxD; ++c) {
        if (c < dm) {
            a0[c] = i0 < n ? shapes[i0 * dm + c] : 0.0;
            a1[c] = i1 < n ? shapes[i1 * dm + c] : 0.0;
        }
    }
    const int r_begin = blockIdx.y * rows_per_split, r_end = min(k, r_begin + rows_per_split);
    const int tile_rows = kVqTileBytes / (8 * dm);
    double b0 = INFINITY, b1 = INFINITY;
    int best0 = r_begin, best1 = r_begin;
    for (int t0 = r_begin; t0 < r_end; t0 += tile_rows) {
        const int nr = min(tile_rows, r_end - t0);
        __syncthreads();
        for (int q = threadIdx.x; q < nr * dm; q += kVqThreads) s_rows[q] = cb[static_cast<uint64_t>(t0) * dm + q];
        __syncthreads();
#pragma unroll 2
        for (int r = 0; r < nr; ++r) {
            const double* row = s_rows + r * dm;
            double d0 = 0.0, d1 = 0.0;
#pragma unroll
            for (int c = 0; c < kMaxD; ++c) {
                if (c < dm) {
                    const double v = row[c];
                    d0 = dist_step(d0, a0[c], v);
                    d1 = dist_step(d1, a1[c], v);
                }
            }
            if (d0 < b0) {  // strict: ties keep the lowest row
                b0 = d0;
                best0 = t0 + r;
            }
            if (d1 < b1) {
                b1 = d1;
                best1 = t0 + r;
            }
        }
    }
    if (gridDim.y == 1) {
        if (i0 < n) out[i0] = static_cast<uint32_t>(best0);
        if (i1 < n) out[i1] = static_cast<uint32_t>(best1);
    } else {
        const uint64_t base = blockIdx.y * n;
        if (i0 < n) {
            part_d[base + i0] = b0;
            part_r[base + i0] = static_cast<uint32_t>(best0);
        }
        if (i1 < n) {
            part_d[base + i1] = b1;
            part_r[base + i1] = static_cast<uint32_t>(best1);
        }
    }
}

// Merge the K-range winners in ascending range order (strict <): the result
// is the first minimum over rows 0..k-1, as nearest_row returns.
__global__ void k_assign_merge(const double* __restrict__ part_d, const uint32_t* __restrict__ part_r, uint64_t n,
                               int nsplit, uint32_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        double b = INFINITY;
        uint32_t r = part_r[i];  // every range NaN/inf: the first range's start (row 0)
        for (int z = 0; z < nsplit; ++z) {
            const double d = part_d[z * n + i];
            if (d < b) {
                b = d;
                r = part_r[z * n + i];
            }
        }
        out[i] = r;
    }
}

using AssignKernel = void (*)(const double*, uint64_t, int, const double*, int, int, double*, uint32_t*, uint32_t*);

AssignKernel assign_kernel(int dim) {
    switch (dim) {
        case 2: return k_assign<2>;
        case 3: return k_assign<3>;
        case 4: return k_assign<4>;
        case 5: return k_assign<5>;
        case 6: return k_assign<6>;
        case 7: return k_assign<7>;
        case 8: return k_assign<8>;
        case 9: return k_assign<9>;
        case 10: return k_assign<10>;
        case 11: return k_assign<11>;
        case 12: return k_assign<12>;
        case 13: return k_assign<13>;
        case 14: return k_assign<14>;
        case 15: return k_assign<15>;
        case 16: return k_assign<16>;
        default: return k_assign<0>;
    }
}

skan_status cuda_fail(cudaError_t e, const char* what) {
    return set_error(SKAN_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e), 0, SKAN_FAULT_NONE);
}

}  // namespace
}  // namespace skan

extern "C" skan_status skan_assign_indices(const double* shapes, uint64_t n, int dim, const double* codebook, int k,
                                           uint32_t* indices, unsigned ptr_flags, void* stream) {
    using namespace skan;
    if (dim < 1 || dim > 64)
        return set_error(SKAN_SHAPE_ERROR, "assign_indices: shape dimension must be in [1, 64]", 0, SKAN_FAULT_NONE);
    if (k < 0) return set_error(SKAN_CONTRACT_ERROR, "assign_indices: negative codebook size", 0, SKAN_FAULT_NONE);
    if (n == 0) return SKAN_OK;
    if (!shapes || !indices || (k > 0 && !codebook))
        return set_error(SKAN_CONTRACT_ERROR, "assign_indices: null buffer", 0, SKAN_FAULT_NONE);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool host = ptr_flags == SKAN_PTR_HOST;
    const size_t sbytes = n * static_cast<size_t>(dim) * 8, cbytes = static_cast<size_t>(k) * dim * 8;
    const double* d_s = shapes;
    const double* d_c = codebook;
    uint32_t* d_out = indices;
    void* own = nullptr;
    cudaError_t e = cudaSuccess;
    if (host) {
        e = cudaMallocAsync(&own, sbytes + cbytes + n * 4 + 16, s);
        if (e != cudaSuccess) return cuda_fail(e, "assign_indices: device buffers");
        double* ds = static_cast<double*>(own);
        double* dc = ds + n * dim;
        d_out = reinterpret_cast<uint32_t*>(dc + static_cast<size_t>(k) * dim);
        cudaMemcpyAsync(ds, shapes, sbytes, cudaMemcpyHostToDevice, s);
        if (k > 0) cudaMemcpyAsync(dc, codebook, cbytes, cudaMemcpyHostToDevice, s);
        d_s = ds;
        d_c = dc;
    }
    if (k == 0) {
        cudaMemsetAsync(d_out, 0, n * 4, s);  // nearest_row over no rows returns 0
    } else {
        // K split into ascending row ranges until there are ~2 CTAs per SM
        const uint64_t bx = (n + kVqShapes - 1) / kVqShapes;
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int tile_rows = kVqTileBytes / (8 * dim);
        int nsplit = static_cast<int>(std::min<uint64_t>((2ull * sms + bx - 1) / bx, (k + tile_rows - 1) / tile_rows));
        nsplit = std::max(1, std::min(nsplit, 1024));
        const int per = (k + nsplit - 1) / nsplit;
        nsplit = (k + per - 1) / per;
        void* part = nullptr;
        if (nsplit > 1) {
            e = cudaMallocAsync(&part, n * nsplit * 12, s);
            if (e != cudaSuccess) {
                if (own) cudaFreeAsync(own, s);
                return cuda_fail(e, "assign_indices: split scratch");
            }
        }
        double* pd = static_cast<double*>(part);
        uint32_t* pr = part ? reinterpret_cast<uint32_t*>(pd + n * nsplit) : nullptr;
        const size_t smem = static_cast<size_t>(tile_rows) * dim * 8;
        assign_kernel(dim)<<<dim3(static_cast<unsigned>(bx), nsplit), kVqThreads, smem, s>>>(d_s, n, dim, d_c, k, per,
                                                                                             pd, pr, d_out);
        if (nsplit > 1) {
            const int mb = static_cast<int>(std::min<uint64_t>((n + 255) / 256, 4096));
            k_assign_merge<<<mb, 256, 0, s>>>(pd, pr, n, nsplit, d_out);
            cudaFreeAsync(part, s);
        }
    }
    e = cudaGetLastError();
    if (host) {
        if (e == cudaSuccess) e = cudaMemcpyAsync(indices, d_out, n * 4, cudaMemcpyDeviceToHost, s);
        cudaFreeAsync(own, s);
        const cudaError_t e2 = cudaStreamSynchronize(s);
        if (e == cudaSuccess) e = e2;
    }
    if (e != cudaSuccess) return cuda_fail(e, "assign_indices");
    return SKAN_OK;
}
