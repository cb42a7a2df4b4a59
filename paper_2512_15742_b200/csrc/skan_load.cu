// SKAN v1 direct-to-device load: the file's sections
// are copied to HBM as they are and every per-edge step runs here, on the
// device -- the LSB-first index unpack with its range check (lutham.cpp:
// 114-137, 669-676), the resident records, the codebook tables and the bias
// sums.  The host keeps only what is O(layers): the header checks, the
// section walk and the 256-entry gain tables.
#include <cuda_runtime.h>

#include <cstdint>

#include "skan_internal.hpp"

namespace skan {
namespace {

// index n of the LSB-first stream (lutham.cpp:114-137); bytes past the
// packed length read as zero, as k_unpack_indices
__device__ __forceinline__ uint32_t unpack_at(const uint8_t* __restrict__ bytes, uint64_t nbytes, uint64_t n,
                                              int bits) {
    if (bits == 0) return 0u;
    const uint64_t bit = n * static_cast<uint64_t>(bits);
    const uint64_t byte0 = bit >> 3;
    const int shift = static_cast<int>(bit & 7);
    uint64_t acc = 0;
    const int need = (shift + bits + 7) / 8;  // <= 5
    for (int q = 0; q < need; ++q) {
        const uint64_t at = byte0 + q;
        if (at < nbytes) acc |= static_cast<uint64_t>(bytes[at]) << (8 * q);
    }
    return static_cast<uint32_t>((acc >> shift) & ((static_cast<uint64_t>(1) << bits) - 1));
}

// The range check of lutham.cpp:669-676 over a packed index section: the
// first edge (lowest n) whose row is >= K is recorded (atomicMin); the
// reference throws IndexOutOfRange for that edge.
__global__ void k_check_indices(const uint8_t* __restrict__ index, uint64_t index_bytes, int bits, uint32_t K,
                                uint64_t E, unsigned long long* bad) {
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < E;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        if (unpack_at(index, index_bytes, e, bits) >= K) atomicMin(bad, static_cast<unsigned long long>(e));
}

// Per edge (indices already range-checked): the codebook row from the packed
// index section, then the resident record of the layer's format.
template <int FMT>
__global__ void k_load_edges(DevLayer d, const uint8_t* __restrict__ index, uint64_t index_bytes, int bits,
                             const uint8_t* __restrict__ gain, const uint8_t* __restrict__ bias, uint64_t E) {
    for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < E;
         e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t v = unpack_at(index, index_bytes, e, bits);
        if constexpr (FMT == FMT_I8_R32) {
            const_cast<uint32_t*>(d.rec)[e] = (v & 0xFFFFu) | static_cast<uint32_t>(gain[e]) << 16 |
                                              static_cast<uint32_t>(bias[e]) << 24;
        } else if constexpr (FMT == FMT_I8_WIDE) {
            const_cast<uint32_t*>(d.idx)[e] = v;
            const_cast<uint16_t*>(d.gb)[e] = static_cast<uint16_t>(gain[e] | static_cast<uint16_t>(bias[e]) << 8);
        } else {  // FMT_F32: the sections are 64-byte aligned f32 arrays
            if (d.idx) const_cast<uint32_t*>(d.idx)[e] = v;
            const_cast<float*>(d.gain)[e] = reinterpret_cast<const float*>(gain)[e];
            const_cast<float*>(d.bias)[e] = reinterpret_cast<const float*>(bias)[e];
        }
    }
}

// sum_i b_ij in ascending i per output j, in f64: the host staging's order
// (skan_api.cpp fill_bias_sum), so the sums are bitwise the same
__global__ void k_bias_sums(DevLayer d, const uint8_t* __restrict__ bias, int int8) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= d.out) return;
    double s = 0.0;
    for (int i = 0; i < d.in; ++i) {
        const size_t e = static_cast<size_t>(i) * d.out + j;
        const double b = int8 ? __dmul_rn(static_cast<double>(static_cast<int8_t>(bias[e])), d.bs)
                              : static_cast<double>(reinterpret_cast<const float*>(bias)[e]);
        s = __dadd_rn(s, b);
    }
    const_cast<double*>(d.bias_sum)[j] = s;
}

// int8 codebook tables from the K x G section: rows padded to rs bytes
// (zeros), the biased copy (every byte ^ 0x80, padding included) and the
// pair planes P[m][k] = c[k][m] | c[k][m+1] << 8
__global__ void k_codebook_tables(DevLayer d, const int8_t* __restrict__ cb) {
    const int G = d.G, rs = d.rs;
    const size_t total = static_cast<size_t>(d.K) * rs;
    for (size_t q = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; q < total;
         q += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t k = q / rs;
        const int m = static_cast<int>(q - k * rs);
        const uint8_t c = m < G ? static_cast<uint8_t>(cb[k * G + m]) : 0u;
        const_cast<int8_t*>(d.cb8)[q] = static_cast<int8_t>(c);
        const_cast<uint8_t*>(d.cb8u)[q] = c ^ 0x80u;
        if (m + 1 < G)
            const_cast<uint16_t*>(d.pair8)[static_cast<size_t>(m) * d.K + k] =
                static_cast<uint16_t>(c | static_cast<uint16_t>(static_cast<uint8_t>(cb[k * G + m + 1])) << 8);
    }
}

int grid_of(uint64_t n) {
    const uint64_t b = (n + 255) / 256;
    return static_cast<int>(b < 148ull * 16 ? (b > 0 ? b : 1) : 148ull * 16);
}

}  // namespace

void check_index_section(const uint8_t* index, uint64_t index_bytes, int bits, uint32_t K, uint64_t E,
                         unsigned long long* bad, cudaStream_t s) {
    if (bits == 0 || E == 0) return;
    k_check_indices<<<grid_of(E), 256, 0, s>>>(index, index_bytes, bits, K, E, bad);
    cuda_check(cudaGetLastError(), "index check");
}

void build_layer_from_sections(const DevLayer& d, const LayerSrc& src, int bits, cudaStream_t s) {
    const uint64_t E = static_cast<uint64_t>(d.in) * d.out;
    if (d.fmt == FMT_DENSE) {
        if (d.wt) {  // the GEMM's tiled layout is the only resident copy: tiled straight from the section
            build_dense_tiles(d, const_cast<float*>(d.wt), reinterpret_cast<const float*>(src.codebook), 0, d.wt_nch, s);
            cuda_check(cudaGetLastError(), "dense tiles");
        } else {
            cuda_check(cudaMemcpyAsync(const_cast<float*>(d.cb32), src.codebook, E * d.G * sizeof(float),
                                       cudaMemcpyDeviceToDevice, s), "dense coefficients");
        }
        return;
    }
    switch (d.fmt) {
        case FMT_I8_R32:
            k_load_edges<FMT_I8_R32><<<grid_of(E), 256, 0, s>>>(d, src.index, src.index_bytes, bits, src.gain, src.bias, E);
            break;
        case FMT_I8_WIDE:
            k_load_edges<FMT_I8_WIDE><<<grid_of(E), 256, 0, s>>>(d, src.index, src.index_bytes, bits, src.gain, src.bias, E);
            break;
        default:
            k_load_edges<FMT_F32><<<grid_of(E), 256, 0, s>>>(d, src.index, src.index_bytes, bits, src.gain, src.bias, E);
            break;
    }
    const bool int8 = d.fmt != FMT_F32;
    if (int8) {
        k_codebook_tables<<<grid_of(static_cast<uint64_t>(d.K) * d.rs), 256, 0, s>>>(
            d, reinterpret_cast<const int8_t*>(src.codebook));
    } else {
        cuda_check(cudaMemcpyAsync(const_cast<float*>(d.cb32), src.codebook,
                                   static_cast<size_t>(d.K) * d.G * sizeof(float), cudaMemcpyDeviceToDevice, s),
                   "f32 codebook");
    }
    k_bias_sums<<<(d.out + 127) / 128, 128, 0, s>>>(d, src.bias, int8 ? 1 : 0);
    cuda_check(cudaGetLastError(), "load kernels");
}

}  // namespace skan
