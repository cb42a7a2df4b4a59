// C-ABI implementation: validation, static planner, resident upload, and the
// per-call launch sequence.  Host C++ only; kernels live in skan_kernels.cu.
//
// Reference interfaces replaced (paths under /root/reference/proj):
//   plan_memory        src/lutham.cpp:52-86       -> skan_plan_memory
//   build_model        src/lutham.cpp:214-271     -> skan_head_create (COMPRESSED)
//   build_dense_model  src/lutham.cpp:177-195     -> skan_head_create (DENSE)
//   make_workspace     src/lutham.cpp:757-763     -> skan_workspace_create
//   compressed_forward src/lutham.cpp:819-850     -> skan_forward
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <shared_mutex>
#include <string>
#include <vector>

#include "skan.h"
#include "skan_internal.hpp"

using skan::DevLayer;
using skan::Error;
using skan::raise;

namespace {

// ---------------------------------------------------------------------------
// thread-local last error (no exceptions cross the ABI)

struct LastError {
    skan_status status = SKAN_OK;
    std::string msg;
    uint64_t offset = 0;
    int fault = SKAN_FAULT_NONE;
};
thread_local LastError g_err;

template <class F>
skan_status guarded(F&& f) {
    try {
        f();
        return SKAN_OK;
    } catch (const Error& e) {
        g_err = {e.status, e.what(), e.offset, e.fault};
        return e.status;
    } catch (const std::bad_alloc&) {
        g_err = {SKAN_CONTRACT_ERROR, "host allocation failed", 0, SKAN_FAULT_NONE};
        return SKAN_CONTRACT_ERROR;
    } catch (const std::exception& e) {
        g_err = {SKAN_CONTRACT_ERROR, e.what(), 0, SKAN_FAULT_NONE};
        return SKAN_CONTRACT_ERROR;
    }
}

// Restores the caller's current device on scope exit.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        skan::cuda_check(cudaGetDevice(&prev), "cudaGetDevice");
        if (prev != dev) skan::cuda_check(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~DeviceGuard() {
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
    }
};

// ---------------------------------------------------------------------------
// planner arithmetic (overflow-checked like lutham.cpp:27-39)

uint64_t mul_checked(uint64_t a, uint64_t b) {
    if (a != 0 && b > std::numeric_limits<uint64_t>::max() / a)
        raise(SKAN_PLAN_ERROR, "size arithmetic overflows 64 bits");
    return a * b;
}
uint64_t add_checked(uint64_t a, uint64_t b) {
    if (b > std::numeric_limits<uint64_t>::max() - a)
        raise(SKAN_PLAN_ERROR, "size arithmetic overflows 64 bits");
    return a + b;
}

int index_bits(uint32_t k) {
    if (k <= 1) return 0;
    int b = 0;
    for (uint32_t v = k - 1; v; v >>= 1) ++b;
    return b;
}

bool is_int8(const skan_layer_header& h) { return (h.flags & SKAN_FLAG_INT8) != 0; }

// Bytes of the B200 resident form (layout of upload_layer below).
constexpr uint64_t kAlign = 256;
uint64_t align_up(uint64_t v) { return add_checked(v, kAlign - 1) / kAlign * kAlign; }

uint64_t int8_row_stride(uint64_t G) { return (G + 15) / 16 * 16; }

int device_format(const skan_layer_header& h) {
    if (h.k == 0) return skan::FMT_DENSE;
    if (is_int8(h)) return h.k <= 65536 ? skan::FMT_I8_R32 : skan::FMT_I8_WIDE;
    return skan::FMT_F32;
}

// Dense layers wide enough for the tensor-core layer GEMM also keep their
// grid pre-tiled in its shared-memory layout (DevLayer::wt): the GEMM then
// streams each chunk with one TMA bulk copy.  Built on the device at upload.
bool dense_tiled(const skan_layer_header& h) {
    // (out <= 32: a 128-output tile would be mostly padding; those layers keep
    // the natural layout for the CUDA-core narrow kernel, LaunchCfg kind 5)
    return h.k == 0 && h.out_dim > 32 && h.grid_size >= 2 && h.grid_size <= 16 &&
           skan::gemm_ic(static_cast<int>(h.grid_size)) * static_cast<int>(h.grid_size) <= 88;
}

uint64_t device_bytes(const skan_layer_header& h) {
    const uint64_t e = mul_checked(h.in_dim, h.out_dim);
    const int fmt = device_format(h);
    // node positions + their integer keys (fast knot selection), every format
    uint64_t b = 2 * align_up(mul_checked(h.grid_size, 8));
    if (fmt == skan::FMT_DENSE) {  // one copy of the grid: the GEMM's tiled layout, or the natural one
        if (dense_tiled(h))
            return add_checked(b, align_up(mul_checked(skan::dense_tile_floats(h.in_dim, h.out_dim, h.grid_size), 4)));
        return add_checked(b, align_up(mul_checked(mul_checked(e, h.grid_size), 4)));
    }
    const uint64_t kg = mul_checked(h.k, h.grid_size);
    // int8 codebook: rows padded to 16 B (one 128-bit load per row) plus the
    // (c[m], c[m+1]) pair table (one 2-byte gather per edge-sample)
    const uint64_t cb8 = mul_checked(h.k, int8_row_stride(h.grid_size));
    const uint64_t pairs = mul_checked(mul_checked(h.k, h.grid_size - 1), 2);
    if (fmt == skan::FMT_I8_R32) {
        b = add_checked(b, align_up(mul_checked(e, 4)));        // records
        b = add_checked(b, align_up(cb8));
        b = add_checked(b, align_up(cb8));                      // biased copy (tensor-core GEMM)
        b = add_checked(b, align_up(pairs));
    } else if (fmt == skan::FMT_I8_WIDE) {
        b = add_checked(b, align_up(mul_checked(e, 4)));        // u32 index
        b = add_checked(b, align_up(mul_checked(e, 2)));        // gain|bias codes
        b = add_checked(b, align_up(cb8));
        b = add_checked(b, align_up(cb8));                      // biased copy (tensor-core GEMM)
        b = add_checked(b, align_up(pairs));
    } else {
        if (h.k > 1) b = add_checked(b, align_up(mul_checked(e, 4)));  // u32 index
        b = add_checked(b, align_up(mul_checked(e, 4)));        // gains
        b = add_checked(b, align_up(mul_checked(e, 4)));        // biases
        b = add_checked(b, align_up(mul_checked(kg, 4)));       // f32 codebook
    }
    b = add_checked(b, align_up(256 * 4) + align_up(256 * 8));  // gain LUTs
    b = add_checked(b, align_up(mul_checked(h.out_dim, 8)));     // bias sums
    return b;
}

// plan_memory, lutham.cpp:52-86 (plus device bytes).
skan_memory_plan plan(const skan_layer_header* hs, int n, skan_layer_plan* per) {
    skan_memory_plan tot{};
    uint64_t max_width = 0;
    for (int l = 0; l < n; ++l) {
        const skan_layer_header& h = hs[l];
        if (h.in_dim == 0 || h.out_dim == 0 || h.grid_size < 2)
            raise(SKAN_PLAN_ERROR, "layer header has degenerate dimensions");
        const uint64_t e = mul_checked(h.in_dim, h.out_dim);
        skan_layer_plan lp{};
        if (h.k == 0) {
            lp.codebook_bytes = mul_checked(mul_checked(e, h.grid_size), 4);
        } else {
            const uint64_t w = is_int8(h) ? 1 : 4;
            lp.codebook_bytes = mul_checked(mul_checked(h.k, h.grid_size), w);
            const int bits = index_bits(h.k);
            lp.index_bytes = add_checked(mul_checked(e, static_cast<uint64_t>(bits)), 7) / 8;
            if (bits > 0) lp.unpacked_index_bytes = mul_checked(e, h.k <= 65536 ? 2 : 4);
            lp.gain_bytes = mul_checked(e, w);
            lp.bias_bytes = mul_checked(e, w);
        }
        lp.device_bytes = device_bytes(h);
        const uint64_t payload = add_checked(add_checked(lp.codebook_bytes, lp.index_bytes),
                                             add_checked(lp.gain_bytes, lp.bias_bytes));
        const uint64_t working = add_checked(add_checked(lp.codebook_bytes, lp.unpacked_index_bytes),
                                             add_checked(lp.gain_bytes, lp.bias_bytes));
        tot.payload_total = add_checked(tot.payload_total, payload);
        tot.working_set_total = add_checked(tot.working_set_total, working);
        tot.device_total = add_checked(tot.device_total, lp.device_bytes);
        max_width = std::max<uint64_t>({max_width, h.in_dim, h.out_dim});
        if (per) per[l] = lp;
    }
    tot.scratch_bytes = mul_checked(mul_checked(max_width, 2), sizeof(double));
    tot.working_set_total = add_checked(tot.working_set_total, tot.scratch_bytes);
    return tot;
}

// dequantize_gain_code, quant.cpp:88-91.  The LUT holds exactly the doubles
// the reference produces per edge (same libm exp2, same expression), so the
// exact kernel's gains are bitwise the reference's.
double gain_of_code(int8_t code, double log_min, double log_step) {
    if (code == 127) return 0.0;
    return std::exp2(log_min + static_cast<double>(code) * log_step);
}

}  // namespace

skan_status skan::set_error(skan_status s, const std::string& msg, uint64_t offset, int fault) {
    g_err = {s, msg, offset, fault};
    return s;
}

// ---------------------------------------------------------------------------
// resident objects

struct skan_head {
    int device = 0;
    int num_sms = 148;
    std::vector<skan_layer_header> headers;
    std::vector<DevLayer> dl;
    std::vector<skan_layer_plan> lplan;
    skan_memory_plan totals{};
    void* dmem = nullptr;
    uint64_t dbytes = 0;
    uint64_t edges = 0;
    int in_dim = 0, out_dim = 0, max_width = 0;
    // batch-1 persistent kernel plan (skan_head_b1.cu)
    bool b1_ok = false;
    int b1_grid = 0;
    size_t b1_smem = 0;
    skan::HeadB1Args b1_plan{};  // layers + shared-memory plan; per-call pointers filled at launch
    void* b1_rows = nullptr;     // v2: layer 1's per-edge codebook rows (derived from the head's tables)
    // Forwards hold it shared while they read the layer views and enqueue
    // (host-buffer calls: until they return); skan_head_swap holds it
    // exclusively, so a swap never races a forward's reads of dl/b1_plan.
    mutable std::shared_mutex swap_mu;
    // persisting-L2 fraction requested by skan_head_set_l2_persist (0: off);
    // skan_forward_multi applies it to the side stream that runs this head
    mutable float l2_frac = 0.f;
    uint64_t gen = 1;  // bumped whenever the resident tables (and so kernel parameters) change
};

struct skan_workspace {
    const skan_head* head = nullptr;
    int device = 0;
    int max_batch = 0;
    int width = 0;
    uint64_t interp_ops = 0;
    skan::DevScratch d{};
    double* xin = nullptr;   // staging for host inputs
    double* yout = nullptr;  // staging for host outputs
    uint64_t partial_floats = 0;
    // Non-finite-input flag (ValueError, kan.cpp:29): page-locked host memory
    // mapped into the device, written by a kernel only when it meets a
    // non-finite input.  Sticky: a synchronizing call (host-buffer forward,
    // skan_workspace_check) reads it after its stream sync, clears it and
    // raises.  No per-call memset or device->host copy of a device flag: on
    // the batch-1 path those two copy-engine operations cost more than the
    // kernel itself.
    int* zc_err_h = nullptr; // host view
    int* zc_err_d = nullptr; // device alias (DevScratch::err)
    cudaStream_t last_stream = nullptr;
    int last_launches = 0;
    const double* last_x = nullptr;  // device inputs of the last fast forward (profiling hook)
    float* b1_part = nullptr;        // 2 x [grid][max_width] partials of the batch-1 kernel
    unsigned* b1_done = nullptr;     // its arrival / grid-barrier counters (0 between launches)
    // Host-buffer batch-1 forwards replay a CUDA graph [H2D of x from a pinned
    // staging buffer -> the persistent kernel writing y into mapped pinned
    // memory]: one launch call instead of a copy plus a cooperative launch
    // with a 2 KB parameter block.  Rebuilt when the head's tables change.
    double* pin_in = nullptr;        // page-locked staging of one sample's inputs
    double* pin_out = nullptr;       // page-locked (mapped) outputs of one sample
    double* pin_out_d = nullptr;     // its device alias
    cudaGraphExec_t b1_graph = nullptr;
    uint64_t b1_graph_gen = 0;       // skan_head::gen the graph was built for
    bool b1_graph_failed = false;    // capture unsupported: keep the copy + launch path
    unsigned long long* b1_timeline = nullptr;  // optional phase stamps (profiling hook)
    double* ex_terms = nullptr;      // exact mode, batch <= kExactSplitMaxBatch: the per-edge terms
    size_t ex_doubles = 0;           // ... its size (>= one input's terms for the workspace's batch)
    double* ex_acc = nullptr;        // ... and the running in-order sums [kExactSplitMaxBatch * width]
    // Fast-path launch plans for every batch 1..max_batch, [B-1][layer],
    // built at creation (forward allocates nothing); rebuilt in place if the
    // GEMM routing threshold changes (skan_debug_set_gemm_min_batch).
    std::vector<skan::LaunchCfg> plans;
    int plans_gemm_min = -1;
    std::vector<void*> allocs;
};

namespace {

// ---------------------------------------------------------------------------
// head construction

// Host-side staging of one layer's resident form before upload.
struct Staged {
    skan_layer_header h{};
    std::vector<uint32_t> rec;    // FMT_I8_R32 records
    std::vector<uint32_t> idx;    // u32 indices (WIDE / F32)
    std::vector<uint16_t> gb;     // WIDE gain|bias codes
    std::vector<float> gain, bias;
    std::vector<int8_t> cb8;      // K x G codes (as given)
    std::vector<float> cb32;      // codebook or dense grid
    double lutd[256] = {};
    float lutf[256] = {};
    std::vector<double> bias_sum;
    // SKAN v1 direct-to-device load: the per-edge regions (records, codebook
    // tables, bias sums) are built on the device from the file's sections
    bool dev = false;
    skan::LayerSrc src{};
    int bits = 0;
};

void check_domain(const skan_layer_header& h, int l) {
    if (!(h.domain_lo < h.domain_hi) || !std::isfinite(h.domain_lo) || !std::isfinite(h.domain_hi))
        raise(SKAN_CONTRACT_ERROR, "layer " + std::to_string(l) + " has an invalid domain");
}

void fill_int8_luts(Staged& s) {
    for (int c = 0; c < 256; ++c) {
        const int8_t code = static_cast<int8_t>(c);
        const double g = gain_of_code(code, s.h.gain_log_min, s.h.gain_log_step);
        s.lutd[c] = g;
        s.lutf[c] = static_cast<float>(g * s.h.codebook_scale);
    }
}

// Σ_i b_ij in ascending i, per output j (fast path bias term; valid because
// (1-t)+t == 1 in double, SURVEY.md §7 "hard parts").
template <class BiasAt>
void fill_bias_sum(Staged& s, BiasAt bias_at) {
    const uint32_t in = s.h.in_dim, out = s.h.out_dim;
    s.bias_sum.assign(out, 0.0);
    for (uint32_t i = 0; i < in; ++i)
        for (uint32_t j = 0; j < out; ++j)
            s.bias_sum[j] += bias_at(static_cast<uint64_t>(i) * out + j);
}

void pack_int8_edges(Staged& s, const uint32_t* idx32, const uint16_t* idx16, const int8_t* gcodes,
                     const int8_t* bcodes) {
    const uint64_t e = static_cast<uint64_t>(s.h.in_dim) * s.h.out_dim;
    auto index_at = [&](uint64_t n) -> uint32_t {
        if (idx16) return idx16[n];
        if (idx32) return idx32[n];
        return 0u;
    };
    if (s.h.k <= 65536) {
        s.rec.resize(e);
        for (uint64_t n = 0; n < e; ++n)
            s.rec[n] = (index_at(n) & 0xFFFFu) | (static_cast<uint32_t>(static_cast<uint8_t>(gcodes[n])) << 16) |
                       (static_cast<uint32_t>(static_cast<uint8_t>(bcodes[n])) << 24);
    } else {
        s.idx.resize(e);
        s.gb.resize(e);
        for (uint64_t n = 0; n < e; ++n) {
            s.idx[n] = index_at(n);
            s.gb[n] = static_cast<uint16_t>(static_cast<uint8_t>(gcodes[n]) |
                                            (static_cast<uint16_t>(static_cast<uint8_t>(bcodes[n])) << 8));
        }
    }
    fill_int8_luts(s);
    const double bs = s.h.bias_scale;
    fill_bias_sum(s, [&](uint64_t n) { return static_cast<double>(bcodes[n]) * bs; });
}

// build_model semantics (lutham.cpp:214-271) for one CompressedLayer.
Staged stage_compressed(const skan_layer_desc& d, int l) {
    const std::string where = "layer " + std::to_string(l);
    const skan_layer_header& hd = d.header;
    if (hd.in_dim == 0 || hd.out_dim == 0) raise(SKAN_SHAPE_ERROR, where + " has a zero dimension");
    const uint64_t e = static_cast<uint64_t>(hd.in_dim) * hd.out_dim;
    const int k = static_cast<int>(hd.k);
    if (hd.k < 1 || k < 1) raise(SKAN_CONTRACT_ERROR, "compressed layer has an empty codebook");
    if (d.n_indices != e || d.n_gains != e || d.n_biases != e)
        raise(SKAN_CONTRACT_ERROR, "compressed layer tables disagree on edge count");
    const uint64_t kg = static_cast<uint64_t>(hd.k) * hd.grid_size;
    if (d.n_codebook != kg) raise(SKAN_CONTRACT_ERROR, "codebook does not match layer grid size");
    if (e && (!d.indices || !d.gains || !d.biases)) raise(SKAN_CONTRACT_ERROR, where + " is missing tables");
    if (kg && !d.codebook) raise(SKAN_CONTRACT_ERROR, where + " is missing its codebook");
    for (uint64_t n = 0; n < e; ++n)
        if (d.indices[n] >= hd.k) raise(SKAN_CONTRACT_ERROR, "edge index exceeds codebook size");
    for (uint64_t n = 0; n < e; ++n)
        if (!(d.gains[n] >= 0.0)) raise(SKAN_CONTRACT_ERROR, "edge gains must be nonnegative");
    Staged s;
    s.h = hd;
    s.h.reserved = 0;
    if (d.has_int8) {
        if (d.n_codebook_codes != kg || d.n_gain_codes != e || d.n_bias_codes != e ||
            (kg && !d.codebook_codes) || (e && (!d.gain_codes || !d.bias_codes)))
            raise(SKAN_CONTRACT_ERROR, "int8 tables disagree with layer dimensions");
        s.h.flags = SKAN_FLAG_INT8;
        s.h.codebook_scale = d.codebook_scale;
        s.h.gain_log_min = d.gain_log_min;
        s.h.gain_log_step = d.gain_log_step;
        s.h.bias_scale = d.bias_scale;
        s.cb8.assign(d.codebook_codes, d.codebook_codes + kg);
        pack_int8_edges(s, d.indices, nullptr, d.gain_codes, d.bias_codes);
    } else {
        s.h.flags = 0;
        s.h.codebook_scale = 0.0;
        s.h.gain_log_min = 0.0;
        s.h.gain_log_step = 1.0;
        s.h.bias_scale = 0.0;
        s.cb32.resize(kg);
        for (uint64_t n = 0; n < kg; ++n) s.cb32[n] = static_cast<float>(d.codebook[n]);
        if (hd.k > 1) s.idx.assign(d.indices, d.indices + e);
        s.gain.resize(e);
        s.bias.resize(e);
        for (uint64_t n = 0; n < e; ++n) {
            s.gain[n] = static_cast<float>(d.gains[n]);
            s.bias[n] = static_cast<float>(d.biases[n]);
        }
        fill_bias_sum(s, [&](uint64_t n) { return static_cast<double>(s.bias[n]); });
    }
    return s;
}

// build_dense_model semantics (lutham.cpp:177-195)
Staged stage_dense(const skan_layer_desc& d, int l) {
    const skan_layer_header& hd = d.header;
    if (hd.in_dim == 0 || hd.out_dim == 0) raise(SKAN_SHAPE_ERROR, "layer dimensions must be positive");
    if (hd.grid_size < 2) raise(SKAN_SHAPE_ERROR, "grid size must be at least 2");
    const uint64_t eg = static_cast<uint64_t>(hd.in_dim) * hd.out_dim * hd.grid_size;
    if (d.n_coefficients != eg || (eg && !d.coefficients))
        raise(SKAN_SHAPE_ERROR, "layer " + std::to_string(l) + " coefficient table has the wrong size");
    Staged s;
    s.h = hd;
    s.h.k = 0;
    s.h.flags = 0;
    s.h.reserved = 0;
    s.cb32.resize(eg);
    for (uint64_t n = 0; n < eg; ++n) s.cb32[n] = static_cast<float>(d.coefficients[n]);
    return s;
}

// RuntimeLayer resident tables (lutham.hpp:91-109), e.g. from deserialize.
Staged stage_runtime(const skan_layer_desc& d, int l) {
    const std::string where = "layer " + std::to_string(l);
    const skan_layer_header& hd = d.header;
    if (hd.in_dim == 0 || hd.out_dim == 0 || hd.grid_size < 2)
        raise(SKAN_CONTRACT_ERROR, where + " has degenerate dimensions");
    const uint64_t e = static_cast<uint64_t>(hd.in_dim) * hd.out_dim;
    Staged s;
    s.h = hd;
    if (hd.k == 0) {
        if (is_int8(hd)) raise(SKAN_CONTRACT_ERROR, where + ": dense layers are float only");
        if (!d.table_f32) raise(SKAN_CONTRACT_ERROR, where + " coefficient table is missing");
        s.cb32.assign(d.table_f32, d.table_f32 + e * hd.grid_size);
        return s;
    }
    const uint64_t kg = static_cast<uint64_t>(hd.k) * hd.grid_size;
    const int bits = index_bits(hd.k);
    const uint16_t* i16 = bits > 0 && hd.k <= 65536 ? d.idx16 : nullptr;
    const uint32_t* i32 = bits > 0 && hd.k > 65536 ? d.idx32 : nullptr;
    if (bits > 0 && !i16 && !i32) raise(SKAN_CONTRACT_ERROR, where + " index table has the wrong size");
    for (uint64_t n = 0; n < e && bits > 0; ++n) {
        const uint32_t v = i16 ? i16[n] : i32[n];
        if (v >= hd.k) raise(SKAN_CONTRACT_ERROR, where + " edge " + std::to_string(n) + " indexes past the codebook");
    }
    if (is_int8(hd)) {
        if (!d.table_i8 || !d.rt_gain_codes || !d.rt_bias_codes)
            raise(SKAN_CONTRACT_ERROR, where + " int8 tables have the wrong size");
        s.cb8.assign(d.table_i8, d.table_i8 + kg);
        pack_int8_edges(s, i32, i16, d.rt_gain_codes, d.rt_bias_codes);
    } else {
        if (!d.table_f32 || !d.gains_f32 || !d.biases_f32)
            raise(SKAN_CONTRACT_ERROR, where + " float tables have the wrong size");
        s.cb32.assign(d.table_f32, d.table_f32 + kg);
        if (hd.k > 1) {
            s.idx.resize(e);
            for (uint64_t n = 0; n < e; ++n) s.idx[n] = i16 ? i16[n] : i32[n];
        }
        s.gain.assign(d.gains_f32, d.gains_f32 + e);
        s.bias.assign(d.biases_f32, d.biases_f32 + e);
        fill_bias_sum(s, [&](uint64_t n) { return static_cast<double>(s.bias[n]); });
    }
    return s;
}

// Copy the staged layers into one device allocation (sub-buffers 256-B
// aligned) and fill the kernel-side DevLayer views.
// With `swap` the head's existing allocation is refilled (hot swap: same
// plan), ordered on `stream`; otherwise it is allocated here.
void upload(skan_head* h, std::vector<Staged>& st, bool swap = false, cudaStream_t stream = nullptr) {
    uint64_t total = 0;
    for (const auto& lp : h->lplan) total = add_checked(total, lp.device_bytes);
    // the new layer views are built off to the side and published at the end
    std::vector<DevLayer> new_dl;
    std::vector<skan_layer_header> new_headers;
    if (swap) {
        if (total != h->dbytes) raise(SKAN_CONTRACT_ERROR, "hot swap needs a head with the same memory plan");
    } else {
        h->dbytes = total;
        skan::cuda_check(cudaMalloc(&h->dmem, std::max<uint64_t>(total, 256)), "cudaMalloc(head)");
    }
    // host image of everything but the holes (device-built regions, never touched here)
    std::unique_ptr<uint8_t[]> host(new uint8_t[std::max<uint64_t>(total, 1)]);
    std::vector<std::pair<uint64_t, uint64_t>> holes;
    uint64_t cur = 0;
    auto put = [&](const void* src, uint64_t bytes) -> void* {
        if (add_checked(cur, bytes) > total) raise(SKAN_PLAN_ERROR, "resident layout overruns the plan");
        void* dst = static_cast<uint8_t*>(h->dmem) + cur;
        if (bytes) std::memcpy(host.get() + cur, src, bytes);
        const uint64_t next = std::min(align_up(add_checked(cur, bytes)), total);
        std::memset(host.get() + cur + bytes, 0, next - cur - bytes);
        cur = next;
        return dst;
    };
    auto reserve = [&](uint64_t bytes) -> void* {
        if (add_checked(cur, bytes) > total) raise(SKAN_PLAN_ERROR, "resident layout overruns the plan");
        void* dst = static_cast<uint8_t*>(h->dmem) + cur;
        const uint64_t next = std::min(align_up(add_checked(cur, bytes)), total);
        holes.emplace_back(cur, next);
        cur = next;
        return dst;
    };
    for (size_t l = 0; l < st.size(); ++l) {
        Staged& s = st[l];
        DevLayer d{};
        d.in = static_cast<int>(s.h.in_dim);
        d.out = static_cast<int>(s.h.out_dim);
        d.G = static_cast<int>(s.h.grid_size);
        d.K = static_cast<int>(s.h.k);
        d.fmt = device_format(s.h);
        d.lo = s.h.domain_lo;
        d.hi = s.h.domain_hi;
        d.dx = (s.h.domain_hi - s.h.domain_lo) / static_cast<double>(static_cast<int>(s.h.grid_size) - 1);
        d.cs = s.h.codebook_scale;
        d.bs = s.h.bias_scale;
        const uint64_t begin = cur;
        {  // node positions exactly as node_position (kan.cpp:21-26) + integer keys
            const int G = d.G;
            std::vector<double> node(G);
            std::vector<long long> key(G);
            for (int i = 0; i < G; ++i) {
                node[i] = i == 0 ? d.lo : (i == G - 1 ? d.hi : d.lo + static_cast<double>(i) * d.dx);
                long long bits;
                std::memcpy(&bits, &node[i], 8);
                if (bits == static_cast<long long>(0x8000000000000000ULL)) bits = 0;
                key[i] = bits ^ ((bits >> 63) & 0x7FFFFFFFFFFFFFFFLL);
            }
            d.node = static_cast<const double*>(put(node.data(), node.size() * 8));
            d.nkey = static_cast<const long long*>(put(key.data(), key.size() * 8));
            d.lo_f = static_cast<float>(d.lo);
            d.inv_dx = 1.0 / d.dx;
            d.inv_dx_f = static_cast<float>(d.inv_dx);
            // |q - exact position| <= u*(|lo| + |hi|)/dx from the node roundings
            // plus ~3u*(G-1) from computing q; 16x margin, floor 1e-9
            const double u = 0x1.0p-53;
            d.q_eps = 1e-9 + 16.0 * u * ((std::fabs(d.lo) + std::fabs(d.hi)) / d.dx + 5.0 * G);
            if (!(d.q_eps < 0.25)) d.q_eps = -1.0;  // pathological domain: always search the nodes
            // fp32 bracket estimate (bracket_f32): |qf - (x-lo)/dx| <= 2^-24 * ((2 max|lo|,|hi| +
            // (hi-lo))/dx + 2(G-1)) from rounding x, lo, 1/dx and two fp32 ops; 4x margin on top of q_eps
            d.hi_f = static_cast<float>(d.hi);
            const double uf = 0x1.0p-24;
            const double amax = std::max(std::fabs(d.lo), std::fabs(d.hi));
            const double qf_eps = 4.0 * uf * ((2.0 * amax + (d.hi - d.lo)) / d.dx + 2.0 * (G - 1)) + d.q_eps;
            d.qf_eps = (d.q_eps >= 0.0 && qf_eps < 0.25 && G - 1 < (1 << 21)) ? static_cast<float>(qf_eps) : -1.f;
            // exp2-form of the int8 gain LUT (fast path): log2(cs) folded into the base
            d.g_base = static_cast<float>(s.h.gain_log_min + std::log2(s.h.codebook_scale));
            d.g_step = static_cast<float>(s.h.gain_log_step);
        }
        const uint64_t E = static_cast<uint64_t>(d.in) * d.out;
        // host-built regions go into the image; a directly loaded layer's
        // per-edge regions are holes its build kernels fill
        auto region = [&](const void* src, uint64_t bytes) { return s.dev ? reserve(bytes) : put(src, bytes); };
        switch (d.fmt) {
            case skan::FMT_DENSE:
                if (dense_tiled(s.h)) {  // built on the device from the natural grid (below)
                    d.wt = static_cast<const float*>(reserve(skan::dense_tile_floats(d.in, d.out, d.G) * 4));
                    d.wt_nch = (d.in + skan::gemm_ic(d.G) - 1) / skan::gemm_ic(d.G);
                } else {
                    d.cb32 = static_cast<const float*>(region(s.cb32.data(), E * d.G * 4));
                }
                break;
            case skan::FMT_I8_R32:
            case skan::FMT_I8_WIDE: {
                if (d.fmt == skan::FMT_I8_R32) {
                    d.rec = static_cast<const uint32_t*>(region(s.rec.data(), E * 4));
                } else {
                    d.idx = static_cast<const uint32_t*>(region(s.idx.data(), E * 4));
                    d.gb = static_cast<const uint16_t*>(region(s.gb.data(), E * 2));
                }
                const uint64_t G = s.h.grid_size, K = s.h.k, rs = int8_row_stride(G);
                d.rs = static_cast<int>(rs);
                if (s.dev) {
                    d.cb8 = static_cast<const int8_t*>(reserve(K * rs));
                    d.cb8u = static_cast<const uint8_t*>(reserve(K * rs));
                    d.pair8 = static_cast<const uint16_t*>(reserve(K * (G - 1) * 2));
                    break;
                }
                std::vector<int8_t> padded(K * rs, 0);
                std::vector<uint16_t> pairs(K * (G - 1));
                // pair planes, bracket-major: pairs[m][k] = c[k][m] | c[k][m+1] << 8
                for (uint64_t k = 0; k < K; ++k) {
                    const int8_t* row = s.cb8.data() + k * G;
                    std::memcpy(padded.data() + k * rs, row, G);
                    for (uint64_t m = 0; m + 1 < G; ++m)
                        pairs[m * K + k] = static_cast<uint16_t>(static_cast<uint8_t>(row[m]) |
                                                                 (static_cast<uint8_t>(row[m + 1]) << 8));
                }
                d.cb8 = static_cast<const int8_t*>(put(padded.data(), padded.size()));
                // the same rows with every code biased to u = c ^ 0x80: the GEMM
                // builds 2^23 + u with one byte permute (no XOR per element)
                std::vector<uint8_t> biased(padded.size());
                for (size_t q = 0; q < padded.size(); ++q) biased[q] = static_cast<uint8_t>(padded[q]) ^ 0x80u;
                d.cb8u = static_cast<const uint8_t*>(put(biased.data(), biased.size()));
                d.pair8 = static_cast<const uint16_t*>(put(pairs.data(), pairs.size() * 2));
                break;
            }
            default:
                if (s.h.k > 1) d.idx = static_cast<const uint32_t*>(region(s.idx.data(), E * 4));
                d.gain = static_cast<const float*>(region(s.gain.data(), E * 4));
                d.bias = static_cast<const float*>(region(s.bias.data(), E * 4));
                d.cb32 = static_cast<const float*>(region(s.cb32.data(), static_cast<uint64_t>(d.K) * d.G * 4));
                break;
        }
        if (d.fmt == skan::FMT_I8_R32 || d.fmt == skan::FMT_I8_WIDE) {
            // fp16 layer GEMM scale: |W| = |g c + b| <= max|g| * 128 + 128 |bias scale|
            float gmax = 0.f;
            for (float g : s.lutf) gmax = std::max(gmax, std::fabs(g));
            const double bound = static_cast<double>(gmax) * 128.0 + 128.0 * std::fabs(d.bs);
            d.wsc = 0.f;
            if (std::isfinite(bound) && bound < 1e30) {
                int ex = 0;
                std::frexp(bound > 0.0 ? bound : 1.0, &ex);
                d.wsc = static_cast<float>(std::ldexp(1.0, 15 - ex));
            }
        }
        if (d.fmt != skan::FMT_DENSE) {
            d.lutf = static_cast<const float*>(put(s.lutf, sizeof s.lutf));
            d.lutd = static_cast<const double*>(put(s.lutd, sizeof s.lutd));
            d.bias_sum = static_cast<const double*>(region(s.bias_sum.data(), static_cast<uint64_t>(d.out) * 8));
        }
        if (cur - begin != h->lplan[l].device_bytes)
            raise(SKAN_PLAN_ERROR, "resident layout of layer " + std::to_string(l) + " disagrees with the plan");
        new_dl.push_back(d);
        new_headers.push_back(s.h);
    }
    // copy the image around the holes, then build the device-side regions
    const cudaStream_t cs = swap ? stream : nullptr;
    uint64_t from = 0;
    holes.emplace_back(total, total);
    for (const auto& hole : holes) {
        if (hole.first > from)
            skan::cuda_check(cudaMemcpyAsync(static_cast<uint8_t*>(h->dmem) + from, host.get() + from, hole.first - from,
                                             cudaMemcpyHostToDevice, cs),
                             swap ? "swap head" : "upload head");
        from = hole.second;
    }
    for (size_t l = 0; l < st.size(); ++l)
        if (st[l].dev) skan::build_layer_from_sections(new_dl[l], st[l].src, st[l].bits, cs);
    // host-staged tiled dense layers: the natural grid goes up in slices of
    // whole input chunks through a bounded staging buffer and is tiled there
    for (size_t l = 0; l < st.size(); ++l) {
        const DevLayer& d = new_dl[l];
        if (!d.wt || st[l].dev) continue;
        const int ic = skan::gemm_ic(d.G);
        const uint64_t chunk_bytes = static_cast<uint64_t>(ic) * d.out * d.G * 4;
        const int per = static_cast<int>(std::max<uint64_t>(1, (64ull << 20) / chunk_bytes));
        void* tmp = nullptr;
        skan::cuda_check(cudaMalloc(&tmp, std::min<uint64_t>(static_cast<uint64_t>(per), d.wt_nch) * chunk_bytes),
                         "cudaMalloc (dense staging)");
        for (int ch0 = 0; ch0 < d.wt_nch; ch0 += per) {
            const int ch1 = std::min(d.wt_nch, ch0 + per);
            const uint64_t i0 = static_cast<uint64_t>(ch0) * ic, i1 = std::min<uint64_t>(d.in, static_cast<uint64_t>(ch1) * ic);
            skan::cuda_check(cudaMemcpyAsync(tmp, st[l].cb32.data() + i0 * d.out * d.G, (i1 - i0) * d.out * d.G * 4,
                                             cudaMemcpyHostToDevice, cs),
                             "dense grid slice");
            skan::build_dense_tiles(d, const_cast<float*>(d.wt), static_cast<const float*>(tmp), ch0, ch1, cs);
            skan::cuda_check(cudaStreamSynchronize(cs), "dense tiles");  // the slice buffer is reused
        }
        cudaFree(tmp);
    }
    skan::cuda_check(cudaGetLastError(), "dense tiles");
    for (DevLayer& d : new_dl)  // the fp16 dense GEMM's per-layer scale
        if (d.wt) d.wsc = skan::dense_fp16_scale(d.wt, skan::dense_tile_floats(d.in, d.out, d.G), cs);
    skan::cuda_check(cudaStreamSynchronize(cs), swap ? "swap head" : "upload head");  // host image is freed on return
    h->dl = std::move(new_dl);
    h->headers = std::move(new_headers);
}

std::vector<Staged> stage_all(const skan_layer_desc* layers, int n) {
    std::vector<Staged> st;
    st.reserve(n);
    for (int l = 0; l < n; ++l) {
        switch (layers[l].kind) {
            case SKAN_LAYER_COMPRESSED: st.push_back(stage_compressed(layers[l], l)); break;
            case SKAN_LAYER_DENSE: st.push_back(stage_dense(layers[l], l)); break;
            case SKAN_LAYER_RUNTIME: st.push_back(stage_runtime(layers[l], l)); break;
            default: raise(SKAN_CONTRACT_ERROR, "unknown layer descriptor kind");
        }
        check_domain(st.back().h, l);
        if (l > 0 && st[l].h.in_dim != st[l - 1].h.out_dim)
            raise(SKAN_SHAPE_ERROR, "layer " + std::to_string(l - 1) + " out_dim does not match layer " +
                                        std::to_string(l) + " in_dim");
    }
    return st;
}

// Kernel-side copies of the layer views for the persistent batch-1 plan.
void refresh_b1_layers(skan_head* h, cudaStream_t stream = nullptr) {
    const int nl = static_cast<int>(h->dl.size());
    for (int l = 0; l < nl && l < skan::kMaxHeadLayers; ++l) h->b1_plan.L[l] = h->dl[l];
    const DevLayer& L0 = h->dl[0];
    for (int i = 0; i < L0.G && i < 33; ++i)  // node_position, kan.cpp:21-26
        h->b1_plan.node0[i] = i == 0 ? L0.lo : (i == L0.G - 1 ? L0.hi : L0.lo + static_cast<double>(i) * L0.dx);
    const size_t rb = skan::head_b1_rows_bytes(h->b1_plan);
    if (rb) {  // rebuilt from the current tables (creation, hot swap)
        if (!h->b1_rows) skan::cuda_check(cudaMalloc(&h->b1_rows, rb), "cudaMalloc (batch-1 layer-1 rows)");
        h->b1_plan.l1rows = static_cast<const uint4*>(h->b1_rows);
        skan::cuda_check(skan::head_b1_build_rows(h->b1_plan, static_cast<uint4*>(h->b1_rows), stream),
                         "batch-1 layer-1 rows");
        skan::cuda_check(cudaStreamSynchronize(stream), "batch-1 layer-1 rows");
    }
}

skan_head* create_head_staged(std::vector<Staged>& st, int device);

skan_head* create_head(const skan_layer_desc* layers, int n, int device) {
    if (n <= 0 || !layers) raise(SKAN_SHAPE_ERROR, "model has no layers");
    int ndev = 0;
    skan::cuda_check(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) raise(SKAN_CONTRACT_ERROR, "no such CUDA device");
    std::vector<Staged> st = stage_all(layers, n);
    return create_head_staged(st, device);
}

skan_head* create_head_staged(std::vector<Staged>& st, int device) {
    const int n = static_cast<int>(st.size());
    auto h = std::make_unique<skan_head>();
    h->device = device;
    std::vector<skan_layer_header> hs;
    for (auto& s : st) hs.push_back(s.h);
    h->lplan.resize(n);
    h->totals = plan(hs.data(), n, h->lplan.data());
    DeviceGuard g(device);
    skan::cuda_check(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device), "sm count");
    upload(h.get(), st);
    h->in_dim = static_cast<int>(hs.front().in_dim);
    h->out_dim = static_cast<int>(hs.back().out_dim);
    uint32_t w = 0;
    for (auto& x : hs) {
        w = std::max({w, x.in_dim, x.out_dim});
        h->edges += static_cast<uint64_t>(x.in_dim) * x.out_dim;
    }
    h->max_width = static_cast<int>(w);
    // batch-1 persistent kernel: eligible heads get one CTA per SM, all
    // co-resident (checked against the occupancy calculator at its smem size)
    const int nl = static_cast<int>(h->dl.size());
    if (skan::head_b1_supported(h->dl.data(), nl)) {
        h->b1_smem = skan::head_b1_smem(h->dl.data(), nl, h->num_sms, &h->b1_plan);
        h->b1_plan.nl = nl;
        refresh_b1_layers(h.get());
        h->b1_grid = skan::head_b1_max_grid(h->b1_smem, h->num_sms);
        // the persistent kernel pays for its cooperative launch and grid
        // barriers only on heads whose first layer is wide enough for the
        // pair-plane scheme; small heads take the multi-kernel path
        if (h->b1_grid > 0 && h->b1_plan.planes0) {
            h->b1_ok = true;
        }
    }
    return h.release();
}

// ---------------------------------------------------------------------------
// forward

// Fast-path kernel choice for every layer at batch B.  A layer may use the
// pair-plane kernel only if it has a successor and its predecessor did not
// (the successor reduces its partials while locating).
void plan_head_into(const skan_head* h, int B, skan::LaunchCfg* cfg) {
    const int nl = static_cast<int>(h->dl.size());
    for (int l = 0; l < nl; ++l) {
        const bool allow = l + 1 < nl && !(l > 0 && cfg[l - 1].kind == 2);
        cfg[l] = skan::choose_cfg(h->dl[l], B, false, h->num_sms, allow);
    }
}

std::vector<skan::LaunchCfg> plan_head(const skan_head* h, int B) {
    std::vector<skan::LaunchCfg> cfg(h->dl.size());
    plan_head_into(h, B, cfg.data());
    return cfg;
}

// Largest split-partial buffer (floats) and per-layer counter count any
// batch up to max_batch needs on the fast path.
void scratch_needs(const skan_head* h, int max_batch, uint64_t* partial_floats, uint64_t* counters,
                   std::vector<skan::LaunchCfg>* plans) {
    uint64_t best = 0, cnt = 1;
    const size_t nl = h->dl.size();
    plans->assign(static_cast<size_t>(max_batch) * nl, skan::LaunchCfg{});
    for (int b = 1; b <= max_batch; ++b) {
        skan::LaunchCfg* cfg = plans->data() + static_cast<size_t>(b - 1) * nl;
        plan_head_into(h, b, cfg);
        for (size_t l = 0; l < nl; ++l) {
            const skan::LaunchCfg& c = cfg[l];
            best = std::max<uint64_t>(best, static_cast<uint64_t>(c.nsplit) * b * h->dl[l].out);
            cnt = std::max<uint64_t>(cnt, static_cast<uint64_t>(c.jt) * c.st);
        }
    }
    *partial_floats = best;
    *counters = cnt;
}

// The workspace's plan of batch B: no allocation, the table is sized at
// workspace creation for every batch up to max_batch.
const skan::LaunchCfg* ws_plan(const skan_head* h, skan_workspace* ws, int B) {
    const size_t nl = h->dl.size();
    if (ws->plans_gemm_min != skan::g_gemm_min_batch) {
        for (int b = 1; b <= ws->max_batch; ++b) plan_head_into(h, b, ws->plans.data() + (b - 1) * nl);
        ws->plans_gemm_min = skan::g_gemm_min_batch;
    }
    return ws->plans.data() + static_cast<size_t>(B - 1) * nl;
}

// One fused fast-path layer launch (plus the standalone locate in front of
// layer 0 when that kernel does not locate inline).  Layer l reads brackets
// bm[l&1] and its finisher writes layer l+1's into bm[(l+1)&1]; split
// partials ping-pong between two buffers so a layer can reduce its
// predecessor's partials while writing its own.
// Small-batch fused split reduction (below): on unless SKAN_GEMM_FUSE_REDUCE=0
// or skan_debug_set_fuse_reduce(0).
std::atomic<bool> g_fuse_reduce{[] {
    const char* e = std::getenv("SKAN_GEMM_FUSE_REDUCE");
    return !(e && e[0] == '0');
}()};

int launch_layer_fast(const skan_head* h, skan_workspace* ws, const skan::LaunchCfg* cfg, int l,
                      const double* x, int B, double* out, bool chained, cudaStream_t s) {
    auto& d = ws->d;
    const int nl = static_cast<int>(h->dl.size());
    const size_t plane = static_cast<size_t>(ws->max_batch) * h->max_width;
    int* bm[2] = {d.bm, d.bm + plane};
    float* bt[2] = {d.btf, d.btf + plane};
    float* part[2] = {d.partial, d.partial + ws->partial_floats};
    const DevLayer& L = h->dl[l];
    const DevLayer* next = l + 1 < nl ? &h->dl[l + 1] : nullptr;
    const skan::LaunchCfg& c = cfg[l];
    const bool prev_planes = l > 0 && cfg[l - 1].kind == 2;
    // at small batch a layer GEMM followed by a one-tile-wide layer GEMM
    // leaves its split partials to that GEMM, which reduces and brackets them
    // in its prologue (measured: batch 16 59.4 -> 55.3 us; from batch 64 the
    // separate 1184-block reduction is faster than ~90 CTAs doing it)
    auto fuses = [&](const skan::LaunchCfg& p, const skan::LaunchCfg& n) {
        return g_fuse_reduce.load(std::memory_order_relaxed) && B <= 32 && p.kind == 4 && (p.persist == 0 || p.persist == 3) && n.kind == 4 &&
               (n.persist == 0 || n.persist == 3) && n.jt == 1;
    };
    const bool prev_fused = l > 0 && fuses(cfg[l - 1], c);
    const bool next_fused = next != nullptr && fuses(c, cfg[l + 1]);
    int launches = 0;
    skan::FwdArgs a{};
    a.L = L;
    a.B = B;
    a.rows_per_cta = c.ichunk;
    if (l == 0) {
        if (c.kind == 0) {
            a.x = x;  // small batch: knot selection inline in each CTA
        } else {
            skan::launch_locate_input(x, B, L.in, L, bm[0], bt[0], nullptr, d.err, s, /*input_major=*/true);
            ++launches;
            chained = true;
        }
    }
    a.bm_in = bm[l & 1];
    a.bt_in = bt[l & 1];
    if (prev_planes) {
        a.prev_partial = part[(l - 1) & 1];
        a.prev_nsplit = cfg[l - 1].nsplit;
        a.prev_bias_sum = h->dl[l - 1].bias_sum;
    }
    if (prev_fused) {  // bias folded into the previous GEMM's W: partials only
        a.prev_partial = part[(l - 1) & 1];
        a.prev_nsplit = cfg[l - 1].nsplit;
    }
    a.partial = part[l & 1];
    a.counters = d.counters + static_cast<size_t>(l) * d.counter_stride;
    a.y = out;
    a.has_next = next != nullptr;
    if (next) {
        a.N = *next;
        a.bm_out = bm[(l + 1) & 1];
        a.bt_out = bt[(l + 1) & 1];
    }
    a.err = d.err;
    if (next_fused) return launches + skan::launch_layer_gemm(a, c, chained, s, /*with_reduce=*/false);
    return launches + skan::launch_fwd_fast(a, c, chained, s);  // the GEMM's split reduction counted inside
}
// batches at or below this take the two-pass exact path (SKAN_EXACT_SPLIT_MAX
// overrides it, for measurement; 0 = always the one-pass kernel)
static int exact_split_max() {
    static const int v = [] {
        const char* e = std::getenv("SKAN_EXACT_SPLIT_MAX");
        return e ? std::atoi(e) : skan::kExactSplitMaxBatch;
    }();
    return std::min(v, skan::kExactSplitMaxBatch);
}


// Enqueue one chunk (B <= ws->max_batch) on `s`; x/y are device pointers.
//   fast:  [locate] -> fused layer 0 -> fused layer 1 -> ...  (PDL-chained;
//          each layer's last CTAs write the next layer's brackets)
//   exact: locate -> gather_exact -> locate -> gather_exact ...
int enqueue_chunk(const skan_head* h, skan_workspace* ws, const double* x, int B, double* y,
                  bool exact, cudaStream_t s, int* err_flag = nullptr) {
    const int nl = static_cast<int>(h->dl.size());
    auto& d = ws->d;
    int launches = 0;
    if (exact) {
        // each layer brackets its own input (layer l: x or layer l-1's output)
        const double* xin = x;
        for (int l = 0; l < nl; ++l) {
            const DevLayer& L = h->dl[l];
            const DevLayer* next = l + 1 < nl ? &h->dl[l + 1] : nullptr;
            double* out = next ? d.act[l & 1] : y;
            const int b1 = B == 1 && exact_split_max() >= 1 && ws->ex_terms
                               ? skan::launch_exact_b1(L, xin, d.bm, d.btf, d.btd, d.err, out, ws->ex_terms,
                                                       ws->ex_doubles, ws->ex_acc, s)
                               : 0;
            xin = out;
            if (b1) {
                launches += b1;
                continue;
            }
            skan::launch_locate_input(l == 0 ? x : d.act[(l - 1) & 1], B, L.in, L, d.bm, d.btf, d.btd, d.err, s);
            ++launches;
            if (B <= exact_split_max() && ws->ex_terms) {
                launches += skan::launch_exact_split(L, B, d.bm, d.btd, out, ws->ex_terms, ws->ex_doubles,
                                                     ws->ex_acc, s);
            } else {
                const skan::LaunchCfg c = skan::choose_cfg(L, B, true, h->num_sms);
                skan::launch_gather_exact(L, c, B, d.bm, d.btd, out, s);
                ++launches;
            }
        }
    } else {
        ws->last_x = x;
        if (B <= skan::kB1MaxBatch && h->b1_ok && ws->b1_part) {
            // the whole head in one persistent cooperative kernel per sample
            // (B = 2: two back-to-back launches beat the multi-kernel path)
            for (int b = 0; b < B; ++b) {
                skan::HeadB1Args a = h->b1_plan;
                a.x = x + static_cast<size_t>(b) * h->in_dim;
                a.y = y + static_cast<size_t>(b) * h->out_dim;
                const size_t n = h->b1_plan.part_floats;
                a.part[0] = ws->b1_part;
                a.part[1] = ws->b1_part + n;
                a.x_tma = (reinterpret_cast<uintptr_t>(a.x) % 16 == 0) && (h->in_dim % 2 == 0);
                a.done = ws->b1_done;
                a.epoch = 0;  // the kernel's last CTA resets the counters
                a.err = err_flag ? err_flag : d.err;
                a.timeline = ws->b1_timeline;
                skan::cuda_check(skan::launch_head_b1(a, h->b1_grid, h->b1_smem, s), "kernel launch");
            }
            skan::cuda_check(cudaGetLastError(), "kernel launch");
            return B;
        }
        const skan::LaunchCfg* cfg = ws_plan(h, ws, B);
        bool chained = false;
        for (int l = 0; l < nl; ++l) {
            launches += launch_layer_fast(h, ws, cfg, l, x, B, l + 1 < nl ? d.act[l & 1] : y, chained, s);
            chained = true;
        }
    }
    skan::cuda_check(cudaGetLastError(), "kernel launch");
    return launches;
}

// Validation in compressed_forward's order (lutham.cpp:821-834): model,
// batch, spans (checked by the caller in between), then the workspace.
void check_head_batch(const skan_head* h, int batch) {
    if (!h) raise(SKAN_SHAPE_ERROR, "model has no layers");
    if (batch < 0) raise(SKAN_SHAPE_ERROR, "batch must be nonnegative");
}

// A workspace's buffers are sized for the head it was made for (staging,
// split partials, arrival counters, the batch-1 partials).  Another head may
// use it only if every layer has the same shape, grid, codebook size and
// format, which fixes all of those sizes (e.g. the same-architecture heads
// of a multi-head server).  The reference checks only the width
// (lutham.cpp:833); a wider check is needed here because the device scratch
// is planned per head.
bool same_layout(const skan_head* a, const skan_head* b) {
    if (a == b) return true;
    if (!a || !b) return false;
    if (a->dl.size() != b->dl.size() || a->b1_ok != b->b1_ok || a->b1_grid != b->b1_grid) return false;
    for (size_t l = 0; l < a->dl.size(); ++l) {
        const DevLayer &x = a->dl[l], &y = b->dl[l];
        if (x.in != y.in || x.out != y.out || x.G != y.G || x.K != y.K || x.fmt != y.fmt) return false;
    }
    return true;
}

void check_workspace_for(const skan_head* h, const skan_workspace* ws) {
    if (!ws) raise(SKAN_CONTRACT_ERROR, "workspace is null");
    if (ws->width < h->max_width)
        raise(SKAN_CONTRACT_ERROR, "workspace is smaller than the model's widest layer");
    if (ws->device != h->device) raise(SKAN_CONTRACT_ERROR, "workspace lives on another device");
    if (!same_layout(h, ws->head))
        raise(SKAN_CONTRACT_ERROR, "workspace was made for a head with a different layer layout");
}

void check_forward_args(const skan_head* h, const skan_workspace* ws, int batch) {
    check_head_batch(h, batch);
    check_workspace_for(h, ws);
}

// Persisting-L2 carve-out per device: the sum of the resident bytes of the
// heads that asked for persistence, capped at the device maximum.
void update_persist_limit(int device, int64_t delta) {
    static std::mutex mu;
    static std::map<int, int64_t> bytes;
    std::lock_guard<std::mutex> lock(mu);
    int64_t& b = bytes[device];
    b = std::max<int64_t>(0, b + delta);
    int max_persist = 0;
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, device);
    skan::cuda_check(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize,
                                        static_cast<size_t>(std::min<int64_t>(b, max_persist))),
                     "persisting L2 limit");
}

// The access-policy window of a head (empty when it has none).
cudaStreamAttrValue l2_window(const skan_head* h) {
    cudaStreamAttrValue v{};
    if (h->l2_frac > 0.f) {
        int max_window = 0;
        cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, h->device);
        v.accessPolicyWindow.base_ptr = h->dmem;
        v.accessPolicyWindow.num_bytes = std::min<size_t>(h->dbytes, static_cast<size_t>(max_window));
        v.accessPolicyWindow.hitRatio = std::min(1.f, h->l2_frac);
        v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    }
    return v;
}

// Refill a resident head in place (same shapes, grids, K and formats, so
// the same memory plan).  Forwards are excluded by the swap lock and
// in-flight ones drained first: a forward sees the old tables or the new.
void swap_staged(skan_head* h, std::vector<Staged>& st, cudaStream_t stream) {
    const int n = static_cast<int>(st.size());
    if (n != static_cast<int>(h->headers.size())) raise(SKAN_CONTRACT_ERROR, "hot swap needs the same number of layers");
    for (int l = 0; l < n; ++l) {
        const skan_layer_header &a = st[l].h, &b = h->headers[l];
        if (a.in_dim != b.in_dim || a.out_dim != b.out_dim || a.grid_size != b.grid_size || a.k != b.k ||
            (a.flags & SKAN_FLAG_INT8) != (b.flags & SKAN_FLAG_INT8))
            raise(SKAN_CONTRACT_ERROR, "hot swap needs the same layer shapes, grid sizes, K and formats");
    }
    std::vector<skan_layer_header> hs;
    for (auto& x : st) hs.push_back(x.h);
    std::vector<skan_layer_plan> lp(n);
    const skan_memory_plan tot = plan(hs.data(), n, lp.data());
    DeviceGuard g(h->device);
    std::unique_lock<std::shared_mutex> lock(h->swap_mu);
    skan::cuda_check(cudaDeviceSynchronize(), "drain in-flight forwards before a swap");
    h->lplan = lp;
    h->totals = tot;
    upload(h, st, /*swap=*/true, stream);
    if (h->b1_ok) refresh_b1_layers(h, stream);
    ++h->gen;  // captured launches (workspace graphs) are rebuilt
}

// Staging of directly loaded layers: headers (already checked by the SKAN
// parser) and the device addresses of their sections; the gain tables are
// the only per-layer host work.
std::vector<Staged> stage_sections(const skan::SectionLayer* L, int n) {
    std::vector<Staged> st(n);
    for (int l = 0; l < n; ++l) {
        Staged& s = st[l];
        s.h = L[l].h;
        s.dev = true;
        s.src = L[l].src;
        s.bits = L[l].bits;
        if (s.h.k != 0 && is_int8(s.h)) fill_int8_luts(s);
        check_domain(s.h, l);
    }
    return st;
}

}  // namespace

// ===========================================================================
extern "C" {

skan_status skan_last_error(char* msg, size_t cap, uint64_t* off, int* fault) {
    if (msg && cap) {
        std::strncpy(msg, g_err.msg.c_str(), cap - 1);
        msg[cap - 1] = 0;
    }
    if (off) *off = g_err.offset;
    if (fault) *fault = g_err.fault;
    return g_err.status;
}

const char* skan_status_name(skan_status s) {
    switch (s) {
        case SKAN_OK: return "OK";
        case SKAN_SHAPE_ERROR: return "ShapeError";
        case SKAN_VALUE_ERROR: return "ValueError";
        case SKAN_CONTRACT_ERROR: return "ContractError";
        case SKAN_FORMAT_ERROR: return "FormatError";
        case SKAN_PLAN_ERROR: return "PlanError";
        case SKAN_CUDA_ERROR: return "CudaError";
    }
    return "Unknown";
}

int skan_abi_version(void) { return SKAN_ABI_VERSION; }

int skan_index_bits(uint32_t k) { return index_bits(k); }

skan_status skan_plan_memory(const skan_layer_header* hs, int n, skan_layer_plan* per,
                             skan_memory_plan* totals) {
    return guarded([&] {
        if (n < 0 || (n > 0 && !hs)) raise(SKAN_SHAPE_ERROR, "bad header list");
        const skan_memory_plan t = plan(hs, n, per);
        if (totals) *totals = t;
    });
}

skan_status skan_head_create(const skan_layer_desc* layers, int n, int device, skan_head** out) {
    return guarded([&] {
        if (!out) raise(SKAN_CONTRACT_ERROR, "null output handle");
        *out = create_head(layers, n, device);
    });
}

skan_status skan_head_swap(skan_head* h, const skan_layer_desc* layers, int n, void* stream) {
    return guarded([&] {
        if (!h) raise(SKAN_CONTRACT_ERROR, "null head");
        if (n != static_cast<int>(h->headers.size()) || !layers)
            raise(SKAN_CONTRACT_ERROR, "hot swap needs the same number of layers");
        std::vector<Staged> st = stage_all(layers, n);
        swap_staged(h, st, static_cast<cudaStream_t>(stream));
    });
}

skan_status skan_head_destroy(skan_head* h) {
    return guarded([&] {
        if (!h) return;
        if (h->dmem) {
            DeviceGuard g(h->device);
            if (h->l2_frac > 0.f) update_persist_limit(h->device, -static_cast<int64_t>(h->dbytes));
            cudaFree(h->dmem);
            if (h->b1_rows) cudaFree(h->b1_rows);
        }
        delete h;
    });
}

int skan_head_num_layers(const skan_head* h) { return h ? static_cast<int>(h->dl.size()) : 0; }
int skan_head_input_dim(const skan_head* h) { return h ? h->in_dim : 0; }
int skan_head_output_dim(const skan_head* h) { return h ? h->out_dim : 0; }
int skan_head_max_width(const skan_head* h) { return h ? h->max_width : 0; }
int skan_head_device(const skan_head* h) { return h ? h->device : -1; }
uint64_t skan_head_edges(const skan_head* h) { return h ? h->edges : 0; }

skan_status skan_head_layer_header(const skan_head* h, int l, skan_layer_header* out) {
    return guarded([&] {
        if (!h || l < 0 || l >= static_cast<int>(h->headers.size()))
            raise(SKAN_SHAPE_ERROR, "layer index out of range");
        *out = h->headers[l];
    });
}

skan_status skan_head_plan(const skan_head* h, skan_layer_plan* per, skan_memory_plan* totals) {
    return guarded([&] {
        if (!h) raise(SKAN_CONTRACT_ERROR, "null head");
        if (per) std::copy(h->lplan.begin(), h->lplan.end(), per);
        if (totals) *totals = h->totals;
    });
}

skan_status skan_head_set_l2_persist(const skan_head* h, void* stream, float fraction) {
    return guarded([&] {
        if (!h) raise(SKAN_CONTRACT_ERROR, "null head");
        DeviceGuard g(h->device);
        const float f = fraction > 0.f ? std::min(1.f, fraction) : 0.f;
        if ((f > 0.f) != (h->l2_frac > 0.f))
            update_persist_limit(h->device, f > 0.f ? static_cast<int64_t>(h->dbytes) : -static_cast<int64_t>(h->dbytes));
        h->l2_frac = f;
        const cudaStreamAttrValue v = l2_window(h);
        skan::cuda_check(cudaStreamSetAttribute(static_cast<cudaStream_t>(stream),
                                                cudaStreamAttributeAccessPolicyWindow, &v),
                         "access policy window");
    });
}

skan_status skan_workspace_create(const skan_head* h, int max_batch, skan_workspace** out) {
    return guarded([&] {
        if (!h || !out) raise(SKAN_CONTRACT_ERROR, "null head or output handle");
        if (max_batch < 1) raise(SKAN_SHAPE_ERROR, "workspace needs max_batch >= 1");
        DeviceGuard g(h->device);
        auto ws = std::make_unique<skan_workspace>();
        ws->head = h;
        ws->device = h->device;
        ws->max_batch = max_batch;
        ws->width = h->max_width;
        const size_t act = static_cast<size_t>(max_batch) * h->max_width;
        auto alloc = [&](size_t bytes) {
            void* p = nullptr;
            skan::cuda_check(cudaMalloc(&p, std::max<size_t>(bytes, 256)), "cudaMalloc(workspace)");
            ws->allocs.push_back(p);
            return p;
        };
        ws->d.act[0] = static_cast<double*>(alloc(act * 8));
        ws->d.act[1] = static_cast<double*>(alloc(act * 8));
        ws->d.bm = static_cast<int*>(alloc(2 * act * 4));      // ping-pong: layer l reads [l&1]
        ws->d.btf = static_cast<float*>(alloc(2 * act * 4));
        ws->d.btd = static_cast<double*>(alloc(act * 8));
        uint64_t ncnt = 0;
        scratch_needs(h, max_batch, &ws->partial_floats, &ncnt, &ws->plans);
        ws->plans_gemm_min = skan::g_gemm_min_batch;
        ws->d.partial = static_cast<float*>(alloc(2 * ws->partial_floats * 4));  // ping-pong
        ws->d.counter_stride = ncnt;
        const size_t cbytes = ncnt * h->dl.size() * sizeof(unsigned);
        ws->d.counters = static_cast<unsigned*>(alloc(cbytes));
        skan::cuda_check(cudaMemset(ws->d.counters, 0, std::max<size_t>(cbytes, 256)), "cudaMemset");
        if (h->b1_ok) {
            const size_t n = h->b1_plan.part_floats;
            ws->b1_part = static_cast<float*>(alloc(2 * n * sizeof(float)));
            // [0] last-layer arrivals, [1] the v2 kernel's grid barrier (0 between launches)
            ws->b1_done = static_cast<unsigned*>(alloc(2 * sizeof(unsigned)));
            skan::cuda_check(cudaMemset(ws->b1_done, 0, 2 * sizeof(unsigned)), "cudaMemset");
            skan::cuda_check(cudaHostAlloc(&ws->pin_in, static_cast<size_t>(h->in_dim) * 8, cudaHostAllocDefault),
                             "cudaHostAlloc");
            skan::cuda_check(cudaHostAlloc(&ws->pin_out, static_cast<size_t>(h->out_dim) * 8, cudaHostAllocMapped),
                             "cudaHostAlloc");
            skan::cuda_check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ws->pin_out_d), ws->pin_out, 0),
                             "cudaHostGetDevicePointer");
        }
        {  // exact-mode scratch: the largest layer's terms at this workspace's batch, capped
            const size_t bx = static_cast<size_t>(std::min<uint32_t>(max_batch, skan::kExactSplitMaxBatch));
            size_t need = 0;
            for (const auto& L : h->dl) need = std::max(need, bx * ((L.out + 31) / 32 * 32) * L.in);
            ws->ex_doubles = std::min(need, skan::kExactTermBytes / sizeof(double));
            ws->ex_terms = static_cast<double*>(alloc(ws->ex_doubles * sizeof(double)));
            ws->ex_acc = static_cast<double*>(alloc(bx * ws->width * 8));
        }
        ws->xin = static_cast<double*>(alloc(static_cast<size_t>(max_batch) * h->in_dim * 8));
        ws->yout = static_cast<double*>(alloc(static_cast<size_t>(max_batch) * h->out_dim * 8));
        skan::cuda_check(cudaHostAlloc(&ws->zc_err_h, sizeof(int), cudaHostAllocMapped), "cudaHostAlloc");
        *ws->zc_err_h = 0;
        skan::cuda_check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&ws->zc_err_d), ws->zc_err_h, 0),
                         "cudaHostGetDevicePointer");
        ws->d.err = ws->zc_err_d;
        *out = ws.release();
    });
}

skan_status skan_workspace_destroy(skan_workspace* ws) {
    return guarded([&] {
        if (!ws) return;
        DeviceGuard g(ws->device);
        if (ws->b1_graph) cudaGraphExecDestroy(ws->b1_graph);
        for (void* p : ws->allocs) cudaFree(p);
        if (ws->zc_err_h) cudaFreeHost(ws->zc_err_h);
        if (ws->pin_in) cudaFreeHost(ws->pin_in);
        if (ws->pin_out) cudaFreeHost(ws->pin_out);
        delete ws;
    });
}

uint64_t skan_workspace_interp_ops(const skan_workspace* ws) { return ws ? ws->interp_ops : 0; }
int skan_workspace_max_batch(const skan_workspace* ws) { return ws ? ws->max_batch : 0; }
int skan_workspace_width(const skan_workspace* ws) { return ws ? ws->width : 0; }
int skan_workspace_last_launches(const skan_workspace* ws) { return ws ? ws->last_launches : 0; }

// After a stream sync: a non-finite input met by any forward on this
// workspace since the last check raises ValueError (and clears the flag).
void raise_if_flagged(skan_workspace* ws) {
    volatile int* f = ws->zc_err_h;
    if (*f) {
        *f = 0;
        raise(SKAN_VALUE_ERROR, "spline evaluated at non-finite x");
    }
}

// Device alias of a page-locked, mapped host buffer (cudaHostAlloc /
// cudaMallocHost / cudaHostRegister'd memory, e.g. torch pin_memory), or
// null for pageable memory.
const double* mapped_alias(const double* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();  // clear the sticky-free error of an unknown pointer
        return nullptr;
    }
    if (at.type != cudaMemoryTypeHost || !at.devicePointer) return nullptr;
    return static_cast<const double*>(at.devicePointer);
}

// The workspace's batch-1 host-path graph: [H2D pin_in -> xin, the
// persistent kernel (y -> mapped pin_out)], captured on a private stream;
// null when capture is not possible (the caller falls back).
cudaGraphExec_t b1_host_graph(const skan_head* h, skan_workspace* ws) {
    if (ws->b1_graph && ws->b1_graph_gen == h->gen) return ws->b1_graph;
    if (ws->b1_graph_failed) return nullptr;
    if (ws->b1_graph) {
        cudaGraphExecDestroy(ws->b1_graph);
        ws->b1_graph = nullptr;
    }
    cudaStream_t cs = nullptr;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ex = nullptr;
    bool ok = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) == cudaSuccess;
    ok = ok && cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (ok) {
        cudaMemcpyAsync(ws->xin, ws->pin_in, static_cast<size_t>(h->in_dim) * 8, cudaMemcpyHostToDevice, cs);
        skan::HeadB1Args a = h->b1_plan;
        const size_t n = h->b1_plan.part_floats;
        a.x = ws->xin;
        a.y = ws->pin_out_d;
        a.part[0] = ws->b1_part;
        a.part[1] = ws->b1_part + n;
        a.x_tma = (reinterpret_cast<uintptr_t>(a.x) % 16 == 0) && (h->in_dim % 2 == 0);
        a.done = ws->b1_done;
        a.epoch = 0;
        a.err = ws->d.err;
        a.timeline = nullptr;
        skan::launch_head_b1(a, h->b1_grid, h->b1_smem, cs);
        ok = cudaStreamEndCapture(cs, &g) == cudaSuccess && g;
    }
    ok = ok && cudaGraphInstantiate(&ex, g, 0) == cudaSuccess;
    if (g) cudaGraphDestroy(g);
    if (cs) cudaStreamDestroy(cs);
    cudaGetLastError();  // a failed capture leaves no sticky error behind
    if (!ok) {
        if (ex) cudaGraphExecDestroy(ex);
        ws->b1_graph_failed = true;
        return nullptr;
    }
    ws->b1_graph = ex;
    ws->b1_graph_gen = h->gen;
    return ex;
}

skan_status skan_forward(const skan_head* h, skan_workspace* ws, const double* inputs,
                         uint64_t n_inputs, int batch, double* outputs, uint64_t n_outputs,
                         int mode, unsigned ptr_flags, void* stream) {
    return guarded([&] {
        check_head_batch(h, batch);
        const uint64_t in = static_cast<uint64_t>(h->in_dim), out = static_cast<uint64_t>(h->out_dim);
        if (n_inputs != in * static_cast<uint64_t>(batch))
            raise(SKAN_SHAPE_ERROR, "input buffer does not match batch * input_dim");
        if (n_outputs != out * static_cast<uint64_t>(batch))
            raise(SKAN_SHAPE_ERROR, "output buffer does not match batch * output_dim");
        check_workspace_for(h, ws);
        if (mode != SKAN_MODE_FAST && mode != SKAN_MODE_EXACT) raise(SKAN_CONTRACT_ERROR, "unknown mode");
        const bool exact = mode == SKAN_MODE_EXACT;
        const bool host = (ptr_flags & SKAN_PTR_DEVICE) == 0;
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        DeviceGuard g(h->device);
        std::shared_lock<std::shared_mutex> lock(h->swap_mu);
        ws->last_stream = s;
        ws->last_launches = 0;
        if (batch == 0) return;
        // Low-overhead host path: small fast-mode batches the persistent
        // kernel serves, with a page-locked output buffer: x goes over in one
        // H2D copy (every CTA reads all of it, so it must sit in HBM/L2), the
        // kernel writes y straight into host memory and reports a non-finite
        // input in a mapped host flag: copy + launch + sync instead of
        // memset + copy + launch + two D2H copies + sync.
        // One sample: replay the workspace's graph (x staged through pinned
        // memory, y read back from mapped pinned memory: any host buffers).
        if (host && !exact && batch == 1 && h->b1_ok && ws->b1_part && ws->pin_in && !ws->b1_timeline) {
            if (cudaGraphExec_t ge = b1_host_graph(h, ws)) {
                std::memcpy(ws->pin_in, inputs, static_cast<size_t>(in) * 8);
                skan::cuda_check(cudaGraphLaunch(ge, s), "graph launch");
                skan::cuda_check(cudaStreamSynchronize(s), "forward");
                ws->last_launches = 1;
                raise_if_flagged(ws);
                std::memcpy(outputs, ws->pin_out, static_cast<size_t>(out) * 8);
                ws->interp_ops += h->edges;  // after success, as lutham.cpp:849
                return;
            }
        }
        if (host && !exact && batch <= skan::kB1MaxBatch && batch <= ws->max_batch && h->b1_ok && ws->b1_part) {
            double* dy = const_cast<double*>(mapped_alias(outputs));
            if (dy) {
                skan::cuda_check(cudaMemcpyAsync(ws->xin, inputs, static_cast<size_t>(batch) * in * 8,
                                                 cudaMemcpyHostToDevice, s), "H2D inputs");
                ws->last_launches = enqueue_chunk(h, ws, ws->xin, batch, dy, false, s);
                skan::cuda_check(cudaStreamSynchronize(s), "forward");
                raise_if_flagged(ws);
                ws->interp_ops += static_cast<uint64_t>(batch) * h->edges;  // after success, as lutham.cpp:849
                return;
            }
        }
        for (int b0 = 0; b0 < batch; b0 += ws->max_batch) {
            const int B = std::min(ws->max_batch, batch - b0);
            const double* x = inputs + static_cast<size_t>(b0) * in;
            double* y = outputs + static_cast<size_t>(b0) * out;
            if (host) {
                skan::cuda_check(cudaMemcpyAsync(ws->xin, x, static_cast<size_t>(B) * in * 8,
                                                 cudaMemcpyHostToDevice, s), "H2D inputs");
                ws->last_launches += enqueue_chunk(h, ws, ws->xin, B, ws->yout, exact, s);
                skan::cuda_check(cudaMemcpyAsync(y, ws->yout, static_cast<size_t>(B) * out * 8,
                                                 cudaMemcpyDeviceToHost, s), "D2H outputs");
            } else {
                ws->last_launches += enqueue_chunk(h, ws, x, B, y, exact, s);
            }
        }
        if (host) {
            skan::cuda_check(cudaStreamSynchronize(s), "forward");
            raise_if_flagged(ws);
        }
        // host buffers: counted after the call succeeded (lutham.cpp:849);
        // device buffers: at enqueue (a non-finite input surfaces later, in
        // skan_workspace_check)
        ws->interp_ops += static_cast<uint64_t>(batch) * h->edges;
    });
}

skan_status skan_forward_async(const skan_head* h, skan_workspace* ws, const double* x, int batch,
                               double* y, int mode, void* stream) {
    if (!h) return guarded([&] { raise(SKAN_SHAPE_ERROR, "model has no layers"); });
    return skan_forward(h, ws, x, static_cast<uint64_t>(h->in_dim) * (batch > 0 ? batch : 0), batch, y,
                        static_cast<uint64_t>(h->out_dim) * (batch > 0 ? batch : 0), mode, SKAN_PTR_DEVICE,
                        stream);
}

skan_status skan_profile_gather(const skan_head* h, skan_workspace* ws, int layer, int batch, int mode,
                                void* stream) {
    return guarded([&] {
        check_forward_args(h, ws, batch);
        if (layer < 0 || layer >= static_cast<int>(h->dl.size())) raise(SKAN_SHAPE_ERROR, "layer index out of range");
        if (batch < 1 || batch > ws->max_batch) raise(SKAN_CONTRACT_ERROR, "batch outside the workspace capacity");
        DeviceGuard g(h->device);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const DevLayer& L = h->dl[layer];
        const bool exact = mode == SKAN_MODE_EXACT;
        const skan::LaunchCfg c = skan::choose_cfg(L, batch, exact, h->num_sms);
        if (exact) {
            skan::launch_gather_exact(L, c, batch, ws->d.bm, ws->d.btd, ws->d.act[1], s);
        } else {
            if (!ws->last_x) raise(SKAN_CONTRACT_ERROR, "run a forward on this workspace first");
            if (layer > 0 && plan_head(h, batch)[layer - 1].kind == 2)
                raise(SKAN_CONTRACT_ERROR, "layer consumes pair-plane partials; profile it with its predecessor");
            launch_layer_fast(h, ws, plan_head(h, batch).data(), layer, ws->last_x, batch, ws->d.act[layer & 1], false, s);
        }
        skan::cuda_check(cudaGetLastError(), "profile launch");
    });
}

skan_status skan_profile_gemm(const skan_head* h, skan_workspace* ws, int layer, int batch, void* stream,
                              double* issued_flops) {
    return guarded([&] {
        check_forward_args(h, ws, batch);
        if (layer < 0 || layer >= static_cast<int>(h->dl.size())) raise(SKAN_SHAPE_ERROR, "layer index out of range");
        if (batch < 1 || batch > ws->max_batch) raise(SKAN_CONTRACT_ERROR, "batch outside the workspace capacity");
        if (!ws->last_x) raise(SKAN_CONTRACT_ERROR, "run a forward on this workspace first");
        const skan::LaunchCfg* cfg = ws_plan(h, ws, batch);
        if (cfg[layer].kind != 4) raise(SKAN_CONTRACT_ERROR, "layer does not run on the tensor-core GEMM at this batch");
        DeviceGuard g(h->device);
        auto& d = ws->d;
        const size_t plane = static_cast<size_t>(ws->max_batch) * h->max_width;
        skan::FwdArgs a{};
        a.L = h->dl[layer];
        a.B = batch;
        a.rows_per_cta = cfg[layer].ichunk;
        a.bm_in = d.bm + (layer & 1) * plane;
        a.bt_in = d.btf + (layer & 1) * plane;
        a.partial = d.partial + (layer & 1) * ws->partial_floats;
        a.err = d.err;
        skan::launch_layer_gemm(a, cfg[layer], false, static_cast<cudaStream_t>(stream), /*with_reduce=*/false);
        skan::cuda_check(cudaGetLastError(), "profile launch");
        if (issued_flops) *issued_flops = skan::gemm_issued_flops(h->dl[layer], cfg[layer], batch);
    });
}

skan_status skan_debug_b1_timeline(skan_workspace* ws, unsigned long long* d_stamps) {
    return guarded([&] {
        if (!ws) raise(SKAN_CONTRACT_ERROR, "workspace is null");
        ws->b1_timeline = d_stamps;
    });
}

int skan_head_b1_grid(const skan_head* h) { return h && h->b1_ok ? h->b1_grid : 0; }

skan_status skan_workspace_check(skan_workspace* ws) {
    return guarded([&] {
        if (!ws) raise(SKAN_CONTRACT_ERROR, "workspace is null");
        DeviceGuard g(ws->device);
        skan::cuda_check(cudaStreamSynchronize(ws->last_stream), "forward");
        raise_if_flagged(ws);
    });
}

// Side streams for multi-head forwards (per device, created once): heads on
// one feature batch run concurrently, filling each other's wave tails and
// the small trailing kernels, then join the caller's stream.
struct SidePool {
    std::vector<cudaStream_t> streams;
    std::vector<cudaEvent_t> events;  // [0] fork, [1 + q] join of stream q
    std::mutex use;                   // one multi-head enqueue at a time per device
};
SidePool& side_pool(int device) {
    static std::mutex mu;
    static std::map<int, SidePool> pools;
    std::lock_guard<std::mutex> lock(mu);
    SidePool& p = pools[device];
    if (p.streams.empty()) {
        constexpr int kSide = 4;
        for (int q = 0; q < kSide; ++q) {
            cudaStream_t st;
            skan::cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
            p.streams.push_back(st);
        }
        for (int q = 0; q <= kSide; ++q) {
            cudaEvent_t ev;
            skan::cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
            p.events.push_back(ev);
        }
    }
    return p;
}

skan_status skan_forward_multi(const skan_head* const* heads, skan_workspace* const* wss, int n,
                               const double* x, int batch, double* const* ys, int mode, void* stream) {
    return guarded([&] {
        if (n < 0 || (n > 0 && (!heads || !wss || !ys))) raise(SKAN_SHAPE_ERROR, "bad head list");
        for (int q = 0; q < n; ++q) {
            check_forward_args(heads[q], wss[q], batch);
            if (heads[q]->in_dim != heads[0]->in_dim)
                raise(SKAN_SHAPE_ERROR, "heads sharing a feature batch must share input_dim");
            if (heads[q]->device != heads[0]->device)
                raise(SKAN_CONTRACT_ERROR, "heads must live on one device");
        }
        if (n <= 1) {
            for (int q = 0; q < n; ++q) {
                const skan_status st = skan_forward_async(heads[q], wss[q], x, batch, ys[q], mode, stream);
                if (st != SKAN_OK) raise(st, g_err.msg);
            }
            return;
        }
        DeviceGuard g(heads[0]->device);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        SidePool& pool = side_pool(heads[0]->device);
        std::lock_guard<std::mutex> lock(pool.use);
        const int P = static_cast<int>(pool.streams.size());
        const int used = std::min(n, P);
        skan::cuda_check(cudaEventRecord(pool.events[0], s), "fork");
        for (int q = 0; q < used; ++q) skan::cuda_check(cudaStreamWaitEvent(pool.streams[q], pool.events[0], 0), "fork");
        bool persist = false;
        for (int q = 0; q < n; ++q) persist = persist || heads[q]->l2_frac > 0.f;
        for (int q = 0; q < n; ++q) {
            if (persist) {  // this head's persisting window (or none) on the side stream it runs on
                const cudaStreamAttrValue v = l2_window(heads[q]);
                skan::cuda_check(cudaStreamSetAttribute(pool.streams[q % P], cudaStreamAttributeAccessPolicyWindow, &v),
                                 "access policy window");
            }
            const skan_status st =
                skan_forward_async(heads[q], wss[q], x, batch, ys[q], mode, pool.streams[q % P]);
            if (st != SKAN_OK) raise(st, g_err.msg);
        }
        for (int q = 0; q < used; ++q) {
            skan::cuda_check(cudaEventRecord(pool.events[1 + q], pool.streams[q]), "join");
            skan::cuda_check(cudaStreamWaitEvent(s, pool.events[1 + q], 0), "join");
        }
    });
}

skan_status skan_locate(const double* x, int n, double lo, double hi, int G, int* idx, double* t,
                        uint8_t* clamped, void* stream) {
    return guarded([&] {
        if (n < 0) raise(SKAN_SHAPE_ERROR, "negative count");
        if (G < 2) raise(SKAN_SHAPE_ERROR, "grid size must be at least 2");
        int* d_err = nullptr;
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        skan::cuda_check(cudaMallocAsync(&d_err, sizeof(int), s), "cudaMallocAsync");
        skan::cuda_check(cudaMemsetAsync(d_err, 0, sizeof(int), s), "memset");
        skan::launch_locate_raw(x, n, lo, hi, G, idx, t, clamped, d_err, s);
        int herr = 0;
        skan::cuda_check(cudaMemcpyAsync(&herr, d_err, sizeof(int), cudaMemcpyDeviceToHost, s), "copy");
        skan::cuda_check(cudaFreeAsync(d_err, s), "free");
        skan::cuda_check(cudaStreamSynchronize(s), "locate");
        if (herr) raise(SKAN_VALUE_ERROR, "spline evaluated at non-finite x");
    });
}

skan_status skan_pli_lookup(const double* cb, int k, int G, const int* rows, const double* g,
                            const double* b, const double* x, double lo, double hi, int n, double* y,
                            void* stream) {
    return guarded([&] {
        if (n < 0) raise(SKAN_SHAPE_ERROR, "negative count");
        if (G < 2 || k < 1) raise(SKAN_SHAPE_ERROR, "bad codebook shape");
        int* d_err = nullptr;
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        skan::cuda_check(cudaMallocAsync(&d_err, sizeof(int), s), "cudaMallocAsync");
        skan::cuda_check(cudaMemsetAsync(d_err, 0, sizeof(int), s), "memset");
        skan::launch_pli_lookup(cb, k, G, rows, g, b, x, lo, hi, n, y, d_err, s);
        int herr = 0;
        skan::cuda_check(cudaMemcpyAsync(&herr, d_err, sizeof(int), cudaMemcpyDeviceToHost, s), "copy");
        skan::cuda_check(cudaFreeAsync(d_err, s), "free");
        skan::cuda_check(cudaStreamSynchronize(s), "pli_lookup");
        if (herr & 2) raise(SKAN_SHAPE_ERROR, "codebook row out of range");
        if (herr & 1) raise(SKAN_VALUE_ERROR, "spline evaluated at non-finite x");
    });
}

skan_status skan_unpack_indices(const uint8_t* bytes, size_t n_bytes, uint64_t count, int bits,
                                uint32_t* out, void* stream) {
    return guarded([&] {
        if (bits < 0 || bits > 32) raise(SKAN_CONTRACT_ERROR, "index width must be 0..32 bits");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        if (bits == 0) {
            skan::cuda_check(cudaMemsetAsync(out, 0, count * sizeof(uint32_t), s), "memset");
            return;
        }
        if (n_bytes < (count * static_cast<uint64_t>(bits) + 7) / 8)
            raise(SKAN_CONTRACT_ERROR, "packed index buffer is too small");
        skan::launch_unpack_indices(bytes, count, bits, out, s);
        skan::cuda_check(cudaGetLastError(), "unpack launch");
    });
}

}  // extern "C"

namespace skan {

skan_head* create_head_from_sections(const SectionLayer* layers, int n, int device) {
    if (n <= 0 || !layers) raise(SKAN_SHAPE_ERROR, "model has no layers");
    std::vector<Staged> st = stage_sections(layers, n);
    return create_head_staged(st, device);
}

void swap_head_from_sections(skan_head* h, const SectionLayer* layers, int n, cudaStream_t stream) {
    if (!h) raise(SKAN_CONTRACT_ERROR, "null head");
    std::vector<Staged> st = stage_sections(layers, n);
    swap_staged(h, st, stream);
}

}  // namespace skan

extern "C" int skan_debug_set_fuse_reduce(int on) {
    return g_fuse_reduce.exchange(on != 0) ? 1 : 0;
}
