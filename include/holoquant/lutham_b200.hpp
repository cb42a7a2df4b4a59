// holoquant/lutham_b200.hpp — drop-in B200 backend for holoquant's LUTHAM
// forward, header-only C++20 over the C ABI in skan.h (libskan.so).
//
// A holoquant user keeps building and owning the host-side `Model` exactly
// as before (build_model, load_model, deserialize: lutham.hpp:120-132);
// device state is attached explicitly, never hidden behind Model's address:
//
//     holoquant::Model model = holoquant::build_model(cn);        // unchanged
//     holoquant::DeviceHead head = holoquant::upload(model);         // + this line
//     holoquant::DeviceWorkspace ws = holoquant::make_workspace(head);
//     holoquant::compressed_forward(head, inputs, batch, outputs, ws);
//
// The call shapes, argument meanings and the exception taxonomy
// (errors.hpp: ShapeError / ValueError / ContractError / FormatError(fault,
// offset) / PlanError) are those of the reference API in
// proj/include/holoquant/lutham.hpp; every overload below names the
// reference entry point it mirrors.  Include this header next to the
// reference headers and link libskan.so.
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "holoquant/errors.hpp"
#include "holoquant/gsb.hpp"
#include "holoquant/kan.hpp"
#include "holoquant/lutham.hpp"
#include "skan.h"

namespace holoquant {

// Numerics of a device forward (skan.h skan_mode).
enum class DeviceMode : int {
    Fast = SKAN_MODE_FAST,    // f32 edge math, exact knot selection: within 1e-5 (L1-scaled), reproducible
    Exact = SKAN_MODE_EXACT,  // f64 in the reference's operation order: bitwise == compressed_forward
};

namespace b200_detail {

// skan_status -> the reference's exception types (errors.hpp:10-60)
[[noreturn]] inline void throw_last(skan_status st) {
    char msg[1024] = {0};
    std::uint64_t offset = 0;
    int fault = SKAN_FAULT_NONE;
    skan_last_error(msg, sizeof msg, &offset, &fault);
    std::string m(msg);
    switch (st) {
        case SKAN_SHAPE_ERROR: throw ShapeError(m);
        case SKAN_VALUE_ERROR: throw ValueError(m);
        case SKAN_CONTRACT_ERROR: throw ContractError(m);
        case SKAN_PLAN_ERROR: throw PlanError(m);
        case SKAN_FORMAT_ERROR: {
            // FormatError appends " (byte offset N)" itself
            const std::string suffix = " (byte offset " + std::to_string(offset) + ")";
            if (m.size() >= suffix.size() && m.compare(m.size() - suffix.size(), suffix.size(), suffix) == 0)
                m.resize(m.size() - suffix.size());
            throw FormatError(static_cast<FormatFault>(fault), offset, m);
        }
        default: throw std::runtime_error("skan: " + m);
    }
}

inline void check(skan_status st) {
    if (st != SKAN_OK) throw_last(st);
}

inline skan_layer_header to_c(const LayerHeader& h) {
    skan_layer_header c{};
    c.in_dim = h.in_dim;
    c.out_dim = h.out_dim;
    c.grid_size = h.grid_size;
    c.k = h.k;
    c.domain_lo = h.domain_lo;
    c.domain_hi = h.domain_hi;
    c.flags = h.flags;
    c.reserved = h.reserved;
    c.codebook_scale = h.codebook_scale;
    c.gain_log_min = h.gain_log_min;
    c.gain_log_step = h.gain_log_step;
    c.bias_scale = h.bias_scale;
    return c;
}

inline LayerHeader from_c(const skan_layer_header& c) {
    LayerHeader h;
    h.in_dim = c.in_dim;
    h.out_dim = c.out_dim;
    h.grid_size = c.grid_size;
    h.k = c.k;
    h.domain_lo = c.domain_lo;
    h.domain_hi = c.domain_hi;
    h.flags = c.flags;
    h.reserved = c.reserved;
    h.codebook_scale = c.codebook_scale;
    h.gain_log_min = c.gain_log_min;
    h.gain_log_step = c.gain_log_step;
    h.bias_scale = c.bias_scale;
    return h;
}

template <class T>
const T* ptr(const std::vector<T>& v) {
    return v.empty() ? nullptr : v.data();
}

}  // namespace b200_detail

// A resident head on one B200 (the device counterpart of Model).  Immutable
// after creation; shareable by concurrent streams, each with its own
// DeviceWorkspace.
class DeviceHead {
public:
    DeviceHead() = default;
    explicit DeviceHead(skan_head* h) : h_(h) {}
    DeviceHead(const DeviceHead&) = delete;
    DeviceHead& operator=(const DeviceHead&) = delete;
    DeviceHead(DeviceHead&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
    DeviceHead& operator=(DeviceHead&& o) noexcept {
        if (this != &o) {
            reset();
            h_ = std::exchange(o.h_, nullptr);
        }
        return *this;
    }
    ~DeviceHead() { reset(); }

    skan_head* get() const { return h_; }
    int device() const { return skan_head_device(h_); }
    // Model::input_dim / output_dim / max_width (lutham.cpp:160-175)
    int input_dim() const { return skan_head_input_dim(h_); }
    int output_dim() const { return skan_head_output_dim(h_); }
    int max_width() const { return skan_head_max_width(h_); }
    std::uint64_t edge_count() const { return skan_head_edges(h_); }
    // Model::header (lutham.cpp:154)
    ModelHeader header() const {
        ModelHeader mh;
        const int n = skan_head_num_layers(h_);
        for (int l = 0; l < n; ++l) {
            skan_layer_header c{};
            b200_detail::check(skan_head_layer_header(h_, l, &c));
            mh.layers.push_back(b200_detail::from_c(c));
        }
        return mh;
    }
    // Keep the resident tables in L2 across calls on `stream` (cudaStream_t).
    void set_l2_persist(void* stream, float fraction = 1.f) const {
        b200_detail::check(skan_head_set_l2_persist(h_, stream, fraction));
    }

private:
    void reset() {
        if (h_) skan_head_destroy(h_);
        h_ = nullptr;
    }
    skan_head* h_ = nullptr;
};

// Workspace (lutham.hpp:145-151) for one device forward stream.
class DeviceWorkspace {
public:
    DeviceWorkspace() = default;
    explicit DeviceWorkspace(skan_workspace* w) : w_(w) {}
    DeviceWorkspace(const DeviceWorkspace&) = delete;
    DeviceWorkspace& operator=(const DeviceWorkspace&) = delete;
    DeviceWorkspace(DeviceWorkspace&& o) noexcept : w_(std::exchange(o.w_, nullptr)) {}
    DeviceWorkspace& operator=(DeviceWorkspace&& o) noexcept {
        if (this != &o) {
            if (w_) skan_workspace_destroy(w_);
            w_ = std::exchange(o.w_, nullptr);
        }
        return *this;
    }
    ~DeviceWorkspace() {
        if (w_) skan_workspace_destroy(w_);
    }
    skan_workspace* get() const { return w_; }
    // Workspace::interp_ops: += batch * sum_l E_l per forward (test_lutham.cpp:394-409)
    std::uint64_t interp_ops() const { return skan_workspace_interp_ops(w_); }
    int width() const { return skan_workspace_width(w_); }
    int max_batch() const { return skan_workspace_max_batch(w_); }

private:
    skan_workspace* w_ = nullptr;
};

// `DeviceHead upload(const Model&)`: the resident tables of a host Model
// (RuntimeLayer, lutham.hpp:91-109), as built by build_model /
// build_dense_model / deserialize, copied to `device` unchanged.
inline DeviceHead upload(const Model& model, int device = 0) {
    if (model.layers.empty()) throw ShapeError("model has no layers");
    std::vector<skan_layer_desc> d(model.layers.size());
    for (std::size_t l = 0; l < model.layers.size(); ++l) {
        const RuntimeLayer& rl = model.layers[l];
        skan_layer_desc& x = d[l];
        x = skan_layer_desc{};
        x.kind = SKAN_LAYER_RUNTIME;
        x.header = b200_detail::to_c(rl.header);
        x.table_f32 = b200_detail::ptr(rl.table_f32);
        x.table_i8 = b200_detail::ptr(rl.table_i8);
        x.idx16 = b200_detail::ptr(rl.idx16);
        x.idx32 = b200_detail::ptr(rl.idx32);
        x.gains_f32 = b200_detail::ptr(rl.gains_f32);
        x.biases_f32 = b200_detail::ptr(rl.biases_f32);
        x.rt_gain_codes = b200_detail::ptr(rl.gain_codes);
        x.rt_bias_codes = b200_detail::ptr(rl.bias_codes);
    }
    skan_head* h = nullptr;
    b200_detail::check(skan_head_create(d.data(), static_cast<int>(d.size()), device, &h));
    return DeviceHead(h);
}

namespace b200_detail {
// CompressedLayer (+ Int8Tables) views for skan_head_create / skan_head_swap
inline std::vector<skan_layer_desc> compressed_descs(const CompressedNetwork& cn) {
    if (cn.layers.empty()) throw ShapeError("model has no layers");
    std::vector<skan_layer_desc> d(cn.layers.size());
    for (std::size_t l = 0; l < cn.layers.size(); ++l) {
        const CompressedLayer& cl = cn.layers[l];
        skan_layer_desc& x = d[l];
        x = skan_layer_desc{};
        x.kind = SKAN_LAYER_COMPRESSED;
        if (cl.in_dim < 0 || cl.out_dim < 0 || cl.grid_size < 0 || cl.codebook.k < 0)
            throw ShapeError("negative layer dimension");
        LayerHeader h;
        h.in_dim = static_cast<std::uint32_t>(cl.in_dim);
        h.out_dim = static_cast<std::uint32_t>(cl.out_dim);
        h.grid_size = static_cast<std::uint32_t>(cl.grid_size);
        h.k = static_cast<std::uint32_t>(cl.codebook.k);
        h.domain_lo = cl.domain_lo;
        h.domain_hi = cl.domain_hi;
        x.header = to_c(h);
        if (cl.codebook.grid_size != cl.grid_size) throw ContractError("codebook does not match layer grid size");
        x.codebook = ptr(cl.codebook.entries);
        x.n_codebook = cl.codebook.entries.size();
        x.indices = ptr(cl.indices);
        x.gains = ptr(cl.gains);
        x.biases = ptr(cl.biases);
        x.n_indices = cl.indices.size();
        x.n_gains = cl.gains.size();
        x.n_biases = cl.biases.size();
        if (cl.int8) {
            const Int8Tables& t = *cl.int8;
            x.has_int8 = 1;
            x.codebook_codes = ptr(t.codebook_codes);
            x.gain_codes = ptr(t.gain_codes);
            x.bias_codes = ptr(t.bias_codes);
            x.n_codebook_codes = t.codebook_codes.size();
            x.n_gain_codes = t.gain_codes.size();
            x.n_bias_codes = t.bias_codes.size();
            x.codebook_scale = t.codebook_params.scale;
            x.gain_log_min = t.gain_params.log_min;
            x.gain_log_step = t.gain_params.log_step;
            x.bias_scale = t.bias_params.scale;
        }
    }
    return d;
}
}  // namespace b200_detail

// build_model (lutham.cpp:214-271) straight to the device: same validation
// (ContractError on K < 1, size mismatch, index >= K, negative gain) and the
// same f32 / int8 conversion.
inline DeviceHead build_device_model(const CompressedNetwork& cn, int device = 0) {
    const std::vector<skan_layer_desc> d = b200_detail::compressed_descs(cn);
    skan_head* h = nullptr;
    b200_detail::check(skan_head_create(d.data(), static_cast<int>(d.size()), device, &h));
    return DeviceHead(h);
}

// Hot swap: refill `head` in place with a network of the same shapes
// (skan_head_swap); its workspaces stay valid.  Ordered on `stream`.
inline void swap_device_model(DeviceHead& head, const CompressedNetwork& cn, void* stream = nullptr) {
    const std::vector<skan_layer_desc> d = b200_detail::compressed_descs(cn);
    b200_detail::check(skan_head_swap(head.get(), d.data(), static_cast<int>(d.size()), stream));
}

// Hot swap from SKAN v1 bytes (skan_head_swap_bytes): deserialize's faults
// (FormatError with the reference's fault and byte offset) before anything
// is overwritten, then the sections are unpacked on the device into the slot.
inline void swap_device_model(DeviceHead& head, std::span<const std::uint8_t> bytes, void* stream = nullptr) {
    b200_detail::check(skan_head_swap_bytes(head.get(), bytes.data(), bytes.size(), stream));
}

// build_dense_model (lutham.cpp:177-195) straight to the device.
inline DeviceHead build_device_dense_model(const KanNetwork& net, int device = 0) {
    if (net.layers().empty()) throw ShapeError("network needs at least one layer");
    std::vector<skan_layer_desc> d(net.layers().size());
    for (std::size_t l = 0; l < net.layers().size(); ++l) {
        const KanLayer& kl = net.layers()[l];
        skan_layer_desc& x = d[l];
        x = skan_layer_desc{};
        x.kind = SKAN_LAYER_DENSE;
        LayerHeader h;
        h.in_dim = static_cast<std::uint32_t>(kl.in_dim());
        h.out_dim = static_cast<std::uint32_t>(kl.out_dim());
        h.grid_size = static_cast<std::uint32_t>(kl.grid_size());
        h.k = 0;
        h.domain_lo = kl.domain_lo();
        h.domain_hi = kl.domain_hi();
        x.header = b200_detail::to_c(h);
        x.coefficients = b200_detail::ptr(kl.coefficients());
        x.n_coefficients = kl.coefficients().size();
    }
    skan_head* h = nullptr;
    b200_detail::check(skan_head_create(d.data(), static_cast<int>(d.size()), device, &h));
    return DeviceHead(h);
}

// deserialize (lutham.cpp:532-704): SKAN v1 bytes -> device head, with the
// reference's FormatFault kinds and byte offsets.
inline DeviceHead deserialize_device(std::span<const std::uint8_t> bytes, int device = 0) {
    skan_head* h = nullptr;
    b200_detail::check(skan_head_load(bytes.data(), bytes.size(), device, &h));
    return DeviceHead(h);
}

// load_model (lutham.cpp:715-724) -> device head.
inline DeviceHead load_device_model(const std::string& path, int device = 0) {
    skan_head* h = nullptr;
    b200_detail::check(skan_head_load_file(path.c_str(), device, &h));
    return DeviceHead(h);
}

// plan_memory (lutham.cpp:52-86) of a resident head; layer plans carry the
// reference's byte counts (the B200 resident bytes are in skan_head_plan).
inline MemoryPlan plan_memory(const DeviceHead& head) {
    const int n = skan_head_input_dim(head.get()) > 0 ? static_cast<int>(head.header().layers.size()) : 0;
    std::vector<skan_layer_plan> per(static_cast<std::size_t>(n > 0 ? n : 1));
    skan_memory_plan tot{};
    b200_detail::check(skan_head_plan(head.get(), per.data(), &tot));
    MemoryPlan mp;
    for (int l = 0; l < n; ++l) {
        LayerPlan lp;
        lp.codebook_bytes = per[l].codebook_bytes;
        lp.index_bytes = per[l].index_bytes;
        lp.unpacked_index_bytes = per[l].unpacked_index_bytes;
        lp.gain_bytes = per[l].gain_bytes;
        lp.bias_bytes = per[l].bias_bytes;
        mp.layers.push_back(lp);
    }
    mp.scratch_bytes = tot.scratch_bytes;
    mp.payload_total = tot.payload_total;
    mp.working_set_total = tot.working_set_total;
    return mp;
}

// make_workspace (lutham.cpp:757-763): all device scratch for batches up to
// max_batch is allocated here; compressed_forward allocates nothing.
inline DeviceWorkspace make_workspace(const DeviceHead& head, int max_batch = 256) {
    skan_workspace* w = nullptr;
    b200_detail::check(skan_workspace_create(head.get(), max_batch, &w));
    return DeviceWorkspace(w);
}

// compressed_forward (lutham.cpp:819-850): host spans, synchronous; the
// same ShapeError / ContractError / ValueError behaviour; batch == 0 does
// nothing; ws.interp_ops() += batch * sum E.
inline void compressed_forward(const DeviceHead& head, std::span<const double> inputs, int batch,
                               std::span<double> outputs, DeviceWorkspace& ws, DeviceMode mode = DeviceMode::Fast,
                               void* stream = nullptr) {
    b200_detail::check(skan_forward(head.get(), ws.get(), inputs.data(), inputs.size(), batch, outputs.data(),
                                    outputs.size(), static_cast<int>(mode), SKAN_PTR_HOST, stream));
}

// Device-pointer forward, enqueued on `stream` without synchronizing; a
// non-finite input surfaces as ValueError from check_workspace().
inline void compressed_forward_async(const DeviceHead& head, const double* d_inputs, int batch, double* d_outputs,
                                     DeviceWorkspace& ws, DeviceMode mode, void* stream) {
    b200_detail::check(skan_forward_async(head.get(), ws.get(), d_inputs, batch, d_outputs, static_cast<int>(mode),
                                          stream));
}

inline void check_workspace(DeviceWorkspace& ws) { b200_detail::check(skan_workspace_check(ws.get())); }

// assign_indices (gsb.cpp:275-286) on the GPU: same signature and
// ShapeError as the reference, bit-identical indices (skan_assign_indices).
inline std::vector<std::uint32_t> assign_indices_device(std::span<const ShapeRecord> shapes,
                                                        const Codebook& codebook) {
    const int dim = codebook.grid_size;
    std::vector<double> flat;
    flat.reserve(shapes.size() * static_cast<std::size_t>(dim > 0 ? dim : 0));
    for (const ShapeRecord& r : shapes) {
        if (static_cast<int>(r.shape.size()) != dim) throw ShapeError("shape/codebook grid size mismatch");
        flat.insert(flat.end(), r.shape.begin(), r.shape.end());
    }
    std::vector<std::uint32_t> idx(shapes.size());
    if (shapes.empty()) return idx;
    b200_detail::check(skan_assign_indices(flat.data(), shapes.size(), dim, codebook.entries.data(), codebook.k,
                                           idx.data(), SKAN_PTR_HOST, nullptr));
    return idx;
}

}  // namespace holoquant
