// SKAN v1 container loader -> device head.
//
// Follows the normative layout in /root/reference/proj/docs/FORMAT.md and the
// fault contract of deserialize (src/lutham.cpp:532-704): the same fault
// kinds, byte offsets and message fragments, checked in the same order, so
// a caller switching from holoquant::deserialize sees identical errors.
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

// Owned copies of one layer's sections (file offsets are only 64-B aligned
// relative to the buffer start, which itself may be unaligned).
struct LayerTables {
    std::vector<float> f32;
    std::vector<int8_t> i8;
    std::vector<uint16_t> idx16;
    std::vector<uint32_t> idx32;
    std::vector<float> gains, biases;
    std::vector<int8_t> gcodes, bcodes;
};

}  // namespace

namespace {

void parse(const uint8_t* bytes, uint64_t n, std::vector<skan_layer_header>& hs,
           std::vector<LayerTables>& tabs) {
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

    std::vector<skan_layer_plan> lp(count);
    skan_memory_plan tot{};
    if (skan_plan_memory(hs.data(), static_cast<int>(count), lp.data(), &tot) != SKAN_OK) {
        char msg[256];
        skan_last_error(msg, sizeof msg, nullptr, nullptr);
        skan::raise_format(SKAN_FAULT_BAD_HEADER, kPrelude, msg);
    }

    tabs.resize(count);
    uint64_t cursor = kPrelude + uint64_t{count} * kHeaderBytes;
    for (uint32_t l = 0; l < count; ++l) {
        const skan_layer_header& h = hs[l];
        LayerTables& t = tabs[l];
        const std::string where = "layer " + std::to_string(l);
        const uint64_t e = uint64_t{h.in_dim} * h.out_dim;
        const bool int8 = (h.flags & SKAN_FLAG_INT8) != 0;
        auto section = [&](uint64_t size, const char* name, uint64_t* at_out = nullptr) {
            cursor = (cursor + kSectionAlign - 1) / kSectionAlign * kSectionAlign;
            r.need(cursor + size, cursor, where + " " + name + " section");
            const uint8_t* p = bytes + cursor;
            if (at_out) *at_out = cursor;
            cursor += size;
            return p;
        };
        if (h.k == 0) {
            const uint8_t* p = section(lp[l].codebook_bytes, "coefficient");
            t.f32.resize(e * h.grid_size);
            std::memcpy(t.f32.data(), p, lp[l].codebook_bytes);
            continue;
        }
        const uint8_t* cb = section(lp[l].codebook_bytes, "codebook");
        const uint64_t kg = uint64_t{h.k} * h.grid_size;
        if (int8) {
            t.i8.resize(kg);
            std::memcpy(t.i8.data(), cb, lp[l].codebook_bytes);
        } else {
            t.f32.resize(kg);
            std::memcpy(t.f32.data(), cb, lp[l].codebook_bytes);
        }
        uint64_t index_at = 0;
        const uint8_t* ix = section(lp[l].index_bytes, "index", &index_at);
        const int bits = bit_width_minus1(h.k);
        if (bits > 0) {
            // LSB-first unpack (lutham.cpp:114-137) with the range check of
            // lutham.cpp:669-676.
            const uint64_t mask = (uint64_t{1} << bits) - 1;
            uint64_t acc = 0;
            int filled = 0;
            uint64_t pos = 0;
            if (h.k <= 65536) t.idx16.resize(e); else t.idx32.resize(e);
            for (uint64_t q = 0; q < e; ++q) {
                while (filled < bits) {
                    acc |= uint64_t{ix[pos++]} << filled;
                    filled += 8;
                }
                const uint32_t v = static_cast<uint32_t>(acc & mask);
                acc >>= bits;
                filled -= bits;
                if (v >= h.k)
                    skan::raise_format(SKAN_FAULT_INDEX_OUT_OF_RANGE, index_at,
                                       where + " edge " + std::to_string(q) + " index " + std::to_string(v) +
                                           " is outside K=" + std::to_string(h.k));
                if (h.k <= 65536) t.idx16[q] = static_cast<uint16_t>(v); else t.idx32[q] = v;
            }
        }
        const uint8_t* g = section(lp[l].gain_bytes, "gain");
        const uint8_t* b = section(lp[l].bias_bytes, "bias");
        if (int8) {
            t.gcodes.assign(reinterpret_cast<const int8_t*>(g), reinterpret_cast<const int8_t*>(g) + e);
            t.bcodes.assign(reinterpret_cast<const int8_t*>(b), reinterpret_cast<const int8_t*>(b) + e);
        } else {
            t.gains.resize(e);
            t.biases.resize(e);
            std::memcpy(t.gains.data(), g, e * 4);
            std::memcpy(t.biases.data(), b, e * 4);
        }
    }
}

}  // namespace

extern "C" {

skan_status skan_head_load(const uint8_t* bytes, size_t n, int device, skan_head** out) {
    std::vector<skan_layer_header> hs;
    std::vector<LayerTables> tabs;
    try {
        if (!bytes && n) skan::raise(SKAN_CONTRACT_ERROR, "null buffer");
        parse(bytes, n, hs, tabs);
    } catch (const skan::Error& e) {
        return skan::set_error(e.status, e.what(), e.offset, e.fault);
    }
    std::vector<skan_layer_desc> d(hs.size());
    for (size_t l = 0; l < hs.size(); ++l) {
        skan_layer_desc& x = d[l];
        std::memset(&x, 0, sizeof x);
        x.kind = SKAN_LAYER_RUNTIME;
        x.header = hs[l];
        const LayerTables& t = tabs[l];
        x.table_f32 = t.f32.empty() ? nullptr : t.f32.data();
        x.table_i8 = t.i8.empty() ? nullptr : t.i8.data();
        x.idx16 = t.idx16.empty() ? nullptr : t.idx16.data();
        x.idx32 = t.idx32.empty() ? nullptr : t.idx32.data();
        x.gains_f32 = t.gains.empty() ? nullptr : t.gains.data();
        x.biases_f32 = t.biases.empty() ? nullptr : t.biases.data();
        x.rt_gain_codes = t.gcodes.empty() ? nullptr : t.gcodes.data();
        x.rt_bias_codes = t.bcodes.empty() ? nullptr : t.bcodes.data();
        // An empty vector means a zero-edge section; supply a non-null
        // pointer so the runtime staging accepts it.
        static const int8_t kNone[1] = {0};
        if ((hs[l].flags & SKAN_FLAG_INT8) && hs[l].k) {
            if (!x.table_i8) x.table_i8 = kNone;
        }
    }
    return skan_head_create(d.data(), static_cast<int>(d.size()), device, out);
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
