// SKAN v1 container loader -> device head.
//
// Follows the normative layout in /root/reference/proj/docs/FORMAT.md and the
// fault contract of deserialize (src/lutham.cpp:532-704): the same fault
// kinds, byte offsets and message fragments, checked in the same order, so
// a caller switching from holoquant::deserialize sees identical errors.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "skan.h"
#include "skan_internal.hpp"

namespace {

constexpr uint64_t kPrelude = 16;      // magic, version, endian tag, layer count
constexpr uint64_t kHeaderBytes = 72;  // per-layer header
constexpr uint64_t kSectionAlign = 64;
constexpr uint32_t kVersion = 1;
constexpr uint32_t kEndianTag = 0x01020304u;
constexpr uint32_t kMaxLayers = 1u << 20;

struct Cursor {
    const uint8_t* p;
    uint64_t n;
    void need(uint64_t end, uint64_t at, const std::string& what) const {
        if (n < end) skan::raise_format(SKAN_FAULT_TRUNCATED, at, what + " is truncated");
    }
    uint32_t u32(uint64_t at) const {
        uint32_t v;
        std::memcpy(&v, p + at, 4);
        return v;
    }
    double f64(uint64_t at) const {
        double v;
        std::memcpy(&v, p + at, 8);
        return v;
    }
};

int bit_width_minus1(uint32_t k) {
    if (k <= 1) return 0;
    int b = 0;
    for (uint32_t v = k - 1; v; v >>= 1) ++b;
    return b;
}

}  // namespace

namespace {

void parse_headers(const uint8_t* bytes, uint64_t n, std::vector<skan_layer_header>& hs,
                   std::vector<skan_layer_plan>& lp) {
    Cursor r{bytes, n};
    r.need(4, 0, "magic");
    if (std::memcmp(bytes, "SKAN", 4) != 0)
        skan::raise_format(SKAN_FAULT_BAD_MAGIC, 0, "bad magic, expected 'SKAN'");
    r.need(8, 4, "version field");
    const uint32_t version = r.u32(4);
    if (version != kVersion)
        skan::raise_format(SKAN_FAULT_BAD_VERSION, 4, "unsupported format version " + std::to_string(version));
    r.need(12, 8, "endianness tag");
    if (r.u32(8) != kEndianTag) skan::raise_format(SKAN_FAULT_BAD_ENDIANNESS, 8, "endianness tag mismatch");
    r.need(16, 12, "layer count");
    const uint32_t count = r.u32(12);
    if (count == 0 || count > kMaxLayers) skan::raise_format(SKAN_FAULT_BAD_HEADER, 12, "implausible layer count");

    hs.resize(count);
    for (uint32_t l = 0; l < count; ++l) {
        const uint64_t at = kPrelude + uint64_t{l} * kHeaderBytes;
        const std::string where = "layer " + std::to_string(l);
        r.need(at + kHeaderBytes, at, where + " header");
        skan_layer_header& h = hs[l];
        h.in_dim = r.u32(at + 0);
        h.out_dim = r.u32(at + 4);
        h.grid_size = r.u32(at + 8);
        h.k = r.u32(at + 12);
        h.domain_lo = r.f64(at + 16);
        h.domain_hi = r.f64(at + 24);
        h.flags = r.u32(at + 32);
        h.reserved = r.u32(at + 36);
        h.codebook_scale = r.f64(at + 40);
        h.gain_log_min = r.f64(at + 48);
        h.gain_log_step = r.f64(at + 56);
        h.bias_scale = r.f64(at + 64);
        const bool int8 = (h.flags & SKAN_FLAG_INT8) != 0;
        if (h.in_dim == 0 || h.out_dim == 0)
            skan::raise_format(SKAN_FAULT_BAD_HEADER, at, where + " has a zero dimension");
        if (h.grid_size < 2)
            skan::raise_format(SKAN_FAULT_BAD_HEADER, at + 8, where + " grid size must be at least 2");
        if (!(h.domain_lo < h.domain_hi) || !std::isfinite(h.domain_lo) || !std::isfinite(h.domain_hi))
            skan::raise_format(SKAN_FAULT_BAD_HEADER, at + 16, where + " has an invalid domain");
        if ((h.flags & ~SKAN_FLAG_INT8) != 0)
            skan::raise_format(SKAN_FAULT_BAD_HEADER, at + 32, where + " has unknown flags");
        if (h.reserved != 0)
            skan::raise_format(SKAN_FAULT_BAD_HEADER, at + 36, where + " reserved field must be zero");
        if (h.k == 0 && int8)
            skan::raise_format(SKAN_FAULT_BAD_HEADER, at + 32, where + " is dense but flagged int8");
        if (l > 0 && hs[l - 1].out_dim != h.in_dim)
            skan::raise_format(SKAN_FAULT_BAD_HEADER, at, where + " input width does not chain");
        if (int8) {
            if (!(h.codebook_scale > 0.0) || !std::isfinite(h.codebook_scale))
                skan::raise_format(SKAN_FAULT_BAD_QUANT_PARAM, at + 40,
                                   where + " codebook scale must be positive and finite");
            if (!std::isfinite(h.gain_log_min))
                skan::raise_format(SKAN_FAULT_BAD_QUANT_PARAM, at + 48, where + " gain log minimum must be finite");
            if (!(h.gain_log_step > 0.0) || !std::isfinite(h.gain_log_step))
                skan::raise_format(SKAN_FAULT_BAD_QUANT_PARAM, at + 56,
                                   where + " gain log step must be positive and finite");
            if (!(h.bias_scale > 0.0) || !std::isfinite(h.bias_scale))
                skan::raise_format(SKAN_FAULT_BAD_QUANT_PARAM, at + 64,
                                   where + " bias scale must be positive and finite");
        }
    }

    lp.resize(count);
    skan_memory_plan tot{};
    if (skan_plan_memory(hs.data(), static_cast<int>(count), lp.data(), &tot) != SKAN_OK) {
        char msg[256];
        skan_last_error(msg, sizeof msg, nullptr, nullptr);
        skan::raise_format(SKAN_FAULT_BAD_HEADER, kPrelude, msg);
    }
}

// Section offsets of every layer, walked in deserialize's order
// (lutham.cpp:642-704; FORMAT.md:41-53: 64-byte aligned); the walk stops at
// the first truncated section, whose fault is raised only after the index
// range checks of the sections before it (the reference's check order).
struct Sections {
    uint64_t at[4] = {};  // codebook (or dense coefficients), index, gain, bias
};
struct Walk {
    std::vector<Sections> sec;
    int trunc_layer = -1, trunc_sec = -1;  // first truncated section (0 codebook, 1 index, 2 gain, 3 bias)
    uint64_t trunc_at = 0;
    std::string trunc_msg;
    uint64_t end = 0;  // bytes the file must hold
};

Walk walk_sections(uint64_t n, const std::vector<skan_layer_header>& hs, const std::vector<skan_layer_plan>& lp) {
    Walk w;
    w.sec.resize(hs.size());
    uint64_t cursor = kPrelude + uint64_t{hs.size()} * kHeaderBytes;
    for (size_t l = 0; l < hs.size() && w.trunc_layer < 0; ++l) {
        const skan_layer_header& h = hs[l];
        const std::string where = "layer " + std::to_string(l);
        const uint64_t sizes[4] = {lp[l].codebook_bytes, lp[l].index_bytes, lp[l].gain_bytes, lp[l].bias_bytes};
        static const char* names[4] = {"codebook", "index", "gain", "bias"};
        const int nsec = h.k == 0 ? 1 : 4;
        for (int q = 0; q < nsec; ++q) {
            cursor = (cursor + kSectionAlign - 1) / kSectionAlign * kSectionAlign;
            w.sec[l].at[q] = cursor;
            if (n < cursor + sizes[q]) {
                w.trunc_layer = static_cast<int>(l);
                w.trunc_sec = q;
                w.trunc_at = cursor;
                w.trunc_msg = where + " " + (h.k == 0 ? "coefficient" : names[q]) + " section is truncated";
                break;
            }
            cursor += sizes[q];
        }
    }
    w.end = cursor;
    return w;
}

// index n of an LSB-first packed stream (one value: the fault message)
uint32_t unpack_one(const uint8_t* p, uint64_t n, int bits) {
    const uint64_t bit = n * static_cast<uint64_t>(bits), b0 = bit >> 3, b1 = (bit + bits + 7) / 8;
    uint64_t acc = 0;
    for (uint64_t q = b0; q < b1; ++q) acc |= uint64_t{p[q]} << (8 * (q - b0));
    return static_cast<uint32_t>((acc >> (bit & 7)) & ((uint64_t{1} << bits) - 1));
}

// Parse, copy the file to the device, range-check every complete index
// section there, raise the first fault in deserialize's order, then build
// the head (or refill `swap_into`) from the device copy.
skan_head* load_to_device(const uint8_t* bytes, uint64_t n, int device, skan_head* swap_into, cudaStream_t stream) {
    std::vector<skan_layer_header> hs;
    std::vector<skan_layer_plan> lp;
    parse_headers(bytes, n, hs, lp);
    const Walk w = walk_sections(n, hs, lp);
    const size_t nl = hs.size();
    // a truncation with no index section before it is the first fault: no
    // device work is needed to know it
    bool checks_first = false;
    for (size_t l = 0; l < nl && w.trunc_layer >= 0; ++l)
        if (hs[l].k != 0 && hs[l].k > 1 && (static_cast<int>(l) < w.trunc_layer ||
                                             (static_cast<int>(l) == w.trunc_layer && w.trunc_sec > 1)))
            checks_first = true;
    if (w.trunc_layer >= 0 && !checks_first) skan::raise_format(SKAN_FAULT_TRUNCATED, w.trunc_at, w.trunc_msg);
    int ndev = 0;
    skan::cuda_check(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) skan::raise(SKAN_CONTRACT_ERROR, "no such CUDA device");
    int prev = -1;
    skan::cuda_check(cudaGetDevice(&prev), "cudaGetDevice");
    if (prev != device) skan::cuda_check(cudaSetDevice(device), "cudaSetDevice");
    struct Restore {
        int prev, cur;
        ~Restore() {
            if (prev != cur && prev >= 0) cudaSetDevice(prev);
        }
    } restore{prev, device};
    // the file (as far as it goes) in HBM; index checks of complete sections
    struct Buf {
        void* p = nullptr;
        ~Buf() {
            if (p) cudaFree(p);
        }
    } file, bad;
    const uint64_t have = std::min<uint64_t>(n, std::max<uint64_t>(w.end, 1));
    skan::cuda_check(cudaMalloc(&file.p, std::max<uint64_t>(have, 256)), "cudaMalloc(file)");
    skan::cuda_check(cudaMalloc(&bad.p, nl * sizeof(unsigned long long)), "cudaMalloc(check)");
    skan::cuda_check(cudaMemcpyAsync(file.p, bytes, have, cudaMemcpyHostToDevice, stream), "file to device");
    skan::cuda_check(cudaMemsetAsync(bad.p, 0xFF, nl * sizeof(unsigned long long), stream), "memset");
    const uint8_t* d = static_cast<const uint8_t*>(file.p);
    auto* dbad = static_cast<unsigned long long*>(bad.p);
    for (size_t l = 0; l < nl; ++l) {
        if (hs[l].k == 0) continue;
        if (w.trunc_layer >= 0 && (static_cast<int>(l) > w.trunc_layer ||
                                   (static_cast<int>(l) == w.trunc_layer && w.trunc_sec <= 1)))
            break;
        skan::check_index_section(d + w.sec[l].at[1], lp[l].index_bytes, bit_width_minus1(hs[l].k), hs[l].k,
                                  uint64_t{hs[l].in_dim} * hs[l].out_dim, dbad + l, stream);
    }
    std::vector<unsigned long long> first(nl);
    skan::cuda_check(cudaMemcpyAsync(first.data(), dbad, nl * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                     stream), "check result");
    skan::cuda_check(cudaStreamSynchronize(stream), "index check");
    for (size_t l = 0; l < nl; ++l) {
        const bool trunc_here = static_cast<int>(l) == w.trunc_layer;
        if (trunc_here && w.trunc_sec <= 1) skan::raise_format(SKAN_FAULT_TRUNCATED, w.trunc_at, w.trunc_msg);
        if (first[l] != ~0ull) {
            const uint64_t q = first[l];
            const uint32_t v = unpack_one(bytes + w.sec[l].at[1], q, bit_width_minus1(hs[l].k));
            skan::raise_format(SKAN_FAULT_INDEX_OUT_OF_RANGE, w.sec[l].at[1],
                               "layer " + std::to_string(l) + " edge " + std::to_string(q) + " index " +
                                   std::to_string(v) + " is outside K=" + std::to_string(hs[l].k));
        }
        if (trunc_here) skan::raise_format(SKAN_FAULT_TRUNCATED, w.trunc_at, w.trunc_msg);
    }
    std::vector<skan::SectionLayer> L(nl);
    for (size_t l = 0; l < nl; ++l) {
        L[l].h = hs[l];
        L[l].bits = bit_width_minus1(hs[l].k);
        L[l].src.codebook = d + w.sec[l].at[0];
        L[l].src.index = d + w.sec[l].at[1];
        L[l].src.index_bytes = lp[l].index_bytes;
        L[l].src.gain = d + w.sec[l].at[2];
        L[l].src.bias = d + w.sec[l].at[3];
    }
    if (swap_into) {
        skan::swap_head_from_sections(swap_into, L.data(), static_cast<int>(nl), stream);
        return swap_into;
    }
    return skan::create_head_from_sections(L.data(), static_cast<int>(nl), device);  // synchronizes
}

}  // namespace

extern "C" {

skan_status skan_head_load(const uint8_t* bytes, size_t n, int device, skan_head** out) {
    try {
        if (!bytes && n) skan::raise(SKAN_CONTRACT_ERROR, "null buffer");
        if (!out) skan::raise(SKAN_CONTRACT_ERROR, "null output handle");
        *out = load_to_device(bytes, n, device, nullptr, nullptr);
        return SKAN_OK;
    } catch (const skan::Error& e) {
        return skan::set_error(e.status, e.what(), e.offset, e.fault);
    } catch (const std::exception& e) {
        return skan::set_error(SKAN_CONTRACT_ERROR, e.what(), 0, SKAN_FAULT_NONE);
    }
}

skan_status skan_head_swap_bytes(skan_head* head, const uint8_t* bytes, size_t n, void* stream) {
    try {
        if (!head) skan::raise(SKAN_CONTRACT_ERROR, "null head");
        if (!bytes && n) skan::raise(SKAN_CONTRACT_ERROR, "null buffer");
        load_to_device(bytes, n, skan_head_device(head), head, static_cast<cudaStream_t>(stream));
        return SKAN_OK;
    } catch (const skan::Error& e) {
        return skan::set_error(e.status, e.what(), e.offset, e.fault);
    } catch (const std::exception& e) {
        return skan::set_error(SKAN_CONTRACT_ERROR, e.what(), 0, SKAN_FAULT_NONE);
    }
}

skan_status skan_head_load_file(const char* path, int device, skan_head** out) {
    std::ifstream in(path ? path : "", std::ios::binary | std::ios::ate);
    if (!in) {
        const std::string m = std::string("cannot open '") + (path ? path : "") + "'";
        return skan::set_error(SKAN_VALUE_ERROR, m, 0, SKAN_FAULT_NONE);
    }
    const std::streamsize size = in.tellg();
    in.seekg(0);
    std::vector<uint8_t> bytes(static_cast<size_t>(size));
    in.read(reinterpret_cast<char*>(bytes.data()), size);
    if (!in) {
        const std::string m = std::string("short read from '") + path + "'";
        return skan::set_error(SKAN_VALUE_ERROR, m, 0, SKAN_FAULT_NONE);
    }
    return skan_head_load(bytes.data(), bytes.size(), device, out);
}

}  // extern "C"
