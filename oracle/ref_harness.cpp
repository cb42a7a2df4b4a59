// TEST INFRASTRUCTURE ONLY — a C-ABI shim over the UNMODIFIED reference
// (holoquant, /root/reference/proj/src/{kan,quant,gsb,lutham,trainer}.cpp),
// compiled by oracle/Makefile into oracle/_ref/libholoquant_ref.so.
//
// Nothing here re-implements the reference: every entry point calls the
// reference's own function (cited) so that Python tests and bench.py's
// reference arm can drive the real CPU path.  The product never links this.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "holoquant/errors.hpp"
#include "holoquant/gsb.hpp"
#include "holoquant/kan.hpp"
#include "holoquant/lutham.hpp"
#include "holoquant/quant.hpp"
#include "holoquant/trainer.hpp"
#include "skan_oracle.h"

using namespace holoquant;

namespace {

thread_local std::string g_msg;
thread_local std::uint64_t g_offset = 0;
thread_local int g_fault = -1;

// status codes line up with include/skan.h (SKAN_*)
int fail(int code, const char* what) {
    g_msg = what;
    return code;
}

template <class F>
int guarded(F&& f) {
    g_fault = -1;
    g_offset = 0;
    try {
        f();
        return 0;
    } catch (const FormatError& e) {
        g_fault = static_cast<int>(e.fault);
        g_offset = e.offset;
        return fail(4, e.what());
    } catch (const ShapeError& e) {
        return fail(1, e.what());
    } catch (const ValueError& e) {
        return fail(2, e.what());
    } catch (const ContractError& e) {
        return fail(3, e.what());
    } catch (const PlanError& e) {
        return fail(5, e.what());
    } catch (const std::exception& e) {
        return fail(99, e.what());
    }
}

struct Handle {
    Model model;
};

}  // namespace

extern "C" {

// Descriptor of one holoquant::CompressedLayer (gsb.hpp:91-106) + Int8Tables (82-89).
struct hqref_clayer {
    int in_dim, out_dim, grid_size, k;
    double domain_lo, domain_hi;
    const double* codebook;  // k*G
    const std::uint32_t* indices;
    const double* gains;
    const double* biases;
    int has_int8;
    const std::int8_t* codebook_codes;
    const std::int8_t* gain_codes;
    const std::int8_t* bias_codes;
    double codebook_scale, gain_log_min, gain_log_step, bias_scale;
};

int hqref_last_error(char* msg, std::size_t cap, std::uint64_t* offset, int* fault) {
    if (msg && cap) {
        std::strncpy(msg, g_msg.c_str(), cap - 1);
        msg[cap - 1] = 0;
    }
    if (offset) *offset = g_offset;
    if (fault) *fault = g_fault;
    return 0;
}

int hqref_locate(double lo, double hi, int G, double x, int* idx, double* t, int* clamped) {
    return guarded([&] {
        const GridBracket b = locate(lo, hi, G, x);  // kan.cpp:28
        *idx = b.index;
        *t = b.t;
        *clamped = b.clamped ? 1 : 0;
    });
}

// locate over an array; returns the number of ValueErrors (non-finite x)
std::uint64_t hqref_locate_many(double lo, double hi, int G, const double* x, std::uint64_t n, int* idx,
                                double* t, std::uint8_t* clamped) {
    std::uint64_t bad = 0;
    for (std::uint64_t q = 0; q < n; ++q) {
        try {
            const GridBracket b = locate(lo, hi, G, x[q]);
            idx[q] = b.index;
            t[q] = b.t;
            if (clamped) clamped[q] = b.clamped ? 1 : 0;
        } catch (const ValueError&) {
            ++bad;
            idx[q] = 0;
            t[q] = 0.0;
            if (clamped) clamped[q] = 0;
        }
    }
    return bad;
}

double hqref_node_position(double lo, double hi, int G, int i) {
    return node_position(lo, hi, G, i);  // kan.cpp:21
}

double hqref_eval_spline(const double* c, int n, double lo, double hi, double x) {
    return eval_spline(std::span<const double>(c, n), lo, hi, x);  // kan.cpp:60
}

// pli_lookup lutham.cpp:730 on a codebook of k rows x G doubles
int hqref_pli_lookup(const double* entries, int k, int G, int row, double g, double b, double x,
                     double lo, double hi, double* y) {
    return guarded([&] {
        Codebook cb;
        cb.k = k;
        cb.grid_size = G;
        cb.entries.assign(entries, entries + static_cast<std::size_t>(k) * G);
        *y = pli_lookup(cb, row, g, b, x, lo, hi);
    });
}

double hqref_dequantize_gain_code(std::int8_t code, double log_min, double log_step) {
    return dequantize_gain_code(code, {log_min, log_step});  // quant.cpp:88
}

double hqref_round_half_even(double x) { return round_half_even(x); }

int hqref_index_bits(std::uint32_t k) { return index_bits(k); }

// pack_indices lutham.cpp:88; returns byte count or -1 on ContractError
long long hqref_pack_indices(const std::uint32_t* v, std::size_t n, int bits, std::uint8_t* out,
                             std::size_t cap) {
    std::vector<std::uint8_t> bytes;
    int rc = guarded([&] { bytes = pack_indices(std::span<const std::uint32_t>(v, n), bits); });
    if (rc) return -1;
    if (out && bytes.size() <= cap) std::memcpy(out, bytes.data(), bytes.size());
    return static_cast<long long>(bytes.size());
}

int hqref_unpack_indices(const std::uint8_t* bytes, std::size_t nbytes, std::uint64_t count,
                         int bits, std::uint32_t* out) {
    return guarded([&] {
        const auto v = unpack_indices(std::span<const std::uint8_t>(bytes, nbytes), count, bits);
        std::memcpy(out, v.data(), v.size() * sizeof(std::uint32_t));
    });
}

// plan_memory lutham.cpp:52 over raw headers: per layer 5 u64 + 3 totals
int hqref_plan_memory(const std::uint32_t* dims4 /* in,out,G,k per layer */,
                      const std::uint32_t* flags, int n, std::uint64_t* per_layer5,
                      std::uint64_t* totals3) {
    return guarded([&] {
        ModelHeader mh;
        for (int l = 0; l < n; ++l) {
            LayerHeader h;
            h.in_dim = dims4[4 * l + 0];
            h.out_dim = dims4[4 * l + 1];
            h.grid_size = dims4[4 * l + 2];
            h.k = dims4[4 * l + 3];
            h.flags = flags[l];
            mh.layers.push_back(h);
        }
        const MemoryPlan p = plan_memory(mh);
        for (int l = 0; l < n; ++l) {
            const LayerPlan& lp = p.layers[l];
            per_layer5[5 * l + 0] = lp.codebook_bytes;
            per_layer5[5 * l + 1] = lp.index_bytes;
            per_layer5[5 * l + 2] = lp.unpacked_index_bytes;
            per_layer5[5 * l + 3] = lp.gain_bytes;
            per_layer5[5 * l + 4] = lp.bias_bytes;
        }
        totals3[0] = p.scratch_bytes;
        totals3[1] = p.payload_total;
        totals3[2] = p.working_set_total;
    });
}

// build_model(CompressedNetwork) lutham.cpp:214
int hqref_model_build(const hqref_clayer* layers, int n, void** out) {
    return guarded([&] {
        CompressedNetwork cn;
        for (int l = 0; l < n; ++l) {
            const hqref_clayer& d = layers[l];
            CompressedLayer cl;
            cl.in_dim = d.in_dim;
            cl.out_dim = d.out_dim;
            cl.grid_size = d.grid_size;
            cl.domain_lo = d.domain_lo;
            cl.domain_hi = d.domain_hi;
            cl.codebook.k = d.k;
            cl.codebook.grid_size = d.grid_size;
            const std::size_t kg = static_cast<std::size_t>(d.k) * d.grid_size;
            const std::size_t e = static_cast<std::size_t>(d.in_dim) * d.out_dim;
            cl.codebook.entries.assign(d.codebook, d.codebook + kg);
            cl.indices.assign(d.indices, d.indices + e);
            cl.gains.assign(d.gains, d.gains + e);
            cl.biases.assign(d.biases, d.biases + e);
            if (d.has_int8) {
                Int8Tables t;
                t.codebook_codes.assign(d.codebook_codes, d.codebook_codes + kg);
                t.gain_codes.assign(d.gain_codes, d.gain_codes + e);
                t.bias_codes.assign(d.bias_codes, d.bias_codes + e);
                t.codebook_params.scale = d.codebook_scale;
                t.gain_params.log_min = d.gain_log_min;
                t.gain_params.log_step = d.gain_log_step;
                t.bias_params.scale = d.bias_scale;
                cl.int8 = std::move(t);
            }
            cn.layers.push_back(std::move(cl));
        }
        auto* h = new Handle{build_model(cn)};
        *out = h;
    });
}

// build_dense_model(KanNetwork) lutham.cpp:177; coefficients E*G doubles per layer
int hqref_model_build_dense(const int* dims, int ndims, int G, double lo, double hi,
                            const double* const* coeffs, void** out) {
    return guarded([&] {
        std::vector<KanLayer> layers;
        for (int l = 0; l + 1 < ndims; ++l) {
            KanLayer layer(dims[l], dims[l + 1], G, lo, hi);
            auto& c = layer.coefficients();
            std::memcpy(c.data(), coeffs[l], c.size() * sizeof(double));
            layers.push_back(std::move(layer));
        }
        auto* h = new Handle{build_dense_model(KanNetwork(std::move(layers)))};
        *out = h;
    });
}

// The reference tests' own fixture generator: init_network (trainer.cpp:83) +
// compress_network (gsb.cpp:332) (+ quantize_compressed_network, quant.cpp:125).
// k == 0 builds a dense model via build_dense_model.
int hqref_model_random(const int* dims, int ndims, int G, double sigma, std::uint64_t seed,
                       int k, int int8, void** out) {
    return guarded([&] {
        const KanNetwork net =
            init_network(std::span<const int>(dims, static_cast<std::size_t>(ndims)), G, sigma, seed);
        if (k == 0) {
            *out = new Handle{build_dense_model(net)};
            return;
        }
        VqConfig cfg;
        cfg.k = k;
        cfg.seed = seed;
        cfg.int8 = int8 != 0;
        *out = new Handle{build_model(compress_network(net, cfg))};
    });
}

int hqref_model_deserialize(const std::uint8_t* bytes, std::size_t n, void** out) {
    return guarded([&] {
        *out = new Handle{deserialize(std::span<const std::uint8_t>(bytes, n))};  // lutham.cpp:532
    });
}

long long hqref_model_serialize(void* h, std::uint8_t* out, std::size_t cap) {
    std::vector<std::uint8_t> bytes;
    int rc = guarded([&] { bytes = serialize(static_cast<Handle*>(h)->model); });  // lutham.cpp:443
    if (rc) return -1;
    if (out && bytes.size() <= cap) std::memcpy(out, bytes.data(), bytes.size());
    return static_cast<long long>(bytes.size());
}

void hqref_model_free(void* h) { delete static_cast<Handle*>(h); }

int hqref_model_nlayers(void* h) { return static_cast<int>(static_cast<Handle*>(h)->model.layers.size()); }

// Export RuntimeLayer l (lutham.hpp:91-109) as an oracle_layer view; pointers
// stay valid while the handle lives.
int hqref_model_layer(void* h, int l, oracle_layer* o) {
    const RuntimeLayer& rl = static_cast<Handle*>(h)->model.layers.at(static_cast<std::size_t>(l));
    std::memset(o, 0, sizeof *o);
    o->in_dim = rl.header.in_dim;
    o->out_dim = rl.header.out_dim;
    o->grid_size = rl.header.grid_size;
    o->k = rl.header.k;
    o->domain_lo = rl.header.domain_lo;
    o->domain_hi = rl.header.domain_hi;
    o->flags = rl.header.flags;
    o->codebook_scale = rl.header.codebook_scale;
    o->gain_log_min = rl.header.gain_log_min;
    o->gain_log_step = rl.header.gain_log_step;
    o->bias_scale = rl.header.bias_scale;
    o->table_f32 = rl.table_f32.empty() ? nullptr : rl.table_f32.data();
    o->table_i8 = rl.table_i8.empty() ? nullptr : rl.table_i8.data();
    o->idx16 = rl.idx16.empty() ? nullptr : rl.idx16.data();
    o->idx32 = rl.idx32.empty() ? nullptr : rl.idx32.data();
    o->gains_f32 = rl.gains_f32.empty() ? nullptr : rl.gains_f32.data();
    o->biases_f32 = rl.biases_f32.empty() ? nullptr : rl.biases_f32.data();
    o->gain_codes = rl.gain_codes.empty() ? nullptr : rl.gain_codes.data();
    o->bias_codes = rl.bias_codes.empty() ? nullptr : rl.bias_codes.data();
    return 0;
}

// compressed_forward lutham.cpp:819.  threads > 1 splits the batch over
// std::threads, one Workspace each (the reference concurrency model,
// SPEC.md:536); interp_ops accumulates over all streams.
int hqref_forward(void* hp, const double* in, int batch, double* out, int threads,
                  std::uint64_t* interp_ops) {
    const Model& m = static_cast<Handle*>(hp)->model;
    if (threads <= 1 || batch <= 1) {
        return guarded([&] {
            Workspace ws = make_workspace(m);
            const std::size_t ni = static_cast<std::size_t>(batch) * (m.layers.empty() ? 0 : m.input_dim());
            const std::size_t no = static_cast<std::size_t>(batch) * (m.layers.empty() ? 0 : m.output_dim());
            compressed_forward(m, std::span<const double>(in, ni), batch, std::span<double>(out, no), ws);
            if (interp_ops) *interp_ops += ws.interp_ops;
        });
    }
    if (threads > batch) threads = batch;
    std::vector<std::thread> pool;
    std::vector<int> rcs(threads, 0);
    std::vector<std::uint64_t> ops(threads, 0);
    const std::size_t nin = m.input_dim(), nout = m.output_dim();
    for (int t = 0; t < threads; ++t) {
        pool.emplace_back([&, t] {
            const int s0 = static_cast<int>(static_cast<long long>(batch) * t / threads);
            const int s1 = static_cast<int>(static_cast<long long>(batch) * (t + 1) / threads);
            rcs[t] = guarded([&] {
                Workspace ws = make_workspace(m);
                compressed_forward(m, std::span<const double>(in + s0 * nin, (s1 - s0) * nin), s1 - s0,
                                   std::span<double>(out + s0 * nout, (s1 - s0) * nout), ws);
                ops[t] = ws.interp_ops;
            });
        });
    }
    for (auto& th : pool) th.join();
    for (int t = 0; t < threads; ++t) {
        if (interp_ops) *interp_ops += ops[t];
        if (rcs[t]) return rcs[t];
    }
    return 0;
}

// Oracle relation: to_dense_network (lutham.cpp:284) then
// network_forward (kan.cpp:148), one sample at a time.
int hqref_dense_oracle_forward(void* hp, const double* in, int batch, double* out) {
    return guarded([&] {
        const Model& m = static_cast<Handle*>(hp)->model;
        const KanNetwork net = to_dense_network(m);
        const std::size_t ni = net.input_dim(), no = net.output_dim();
        for (int s = 0; s < batch; ++s) {
            const std::vector<double> y = network_forward(net, std::span<const double>(in + s * ni, ni));
            std::memcpy(out + s * no, y.data(), no * sizeof(double));
        }
    });
}

// bench_model lutham.cpp:866 (median/p25/p75 us per sample)
int hqref_bench(void* hp, int batch, int repeats, int warmup, std::uint64_t seed, double* med,
                double* p25, double* p75) {
    return guarded([&] {
        BenchConfig bc;
        bc.batch = batch;
        bc.repeats = repeats;
        bc.warmup = warmup;
        bc.seed = seed;
        const BenchRow r = bench_model(static_cast<Handle*>(hp)->model, bc);
        *med = r.median_us;
        *p25 = r.p25_us;
        *p75 = r.p75_us;
    });
}

// projected_storage lutham.cpp:1007
int hqref_projected_storage(std::uint64_t edges, std::uint64_t k, std::uint64_t G, int codebooks,
                            int int8, std::uint64_t* out4) {
    return guarded([&] {
        const StorageEstimate e = projected_storage(edges, k, G, codebooks, int8 != 0);
        out4[0] = e.index_bytes;
        out4[1] = e.gain_bias_bytes;
        out4[2] = e.codebook_bytes;
        out4[3] = e.total_bytes;
    });
}

// assign_indices gsb.cpp:275 (shapes n x dim, codebook k x dim, row-major)
int hqref_assign_indices(const double* shapes, std::uint64_t n, int dim, const double* entries, int k,
                         std::uint32_t* out) {
    return guarded([&] {
        std::vector<ShapeRecord> recs(n);
        for (std::uint64_t i = 0; i < n; ++i) recs[i].shape.assign(shapes + i * dim, shapes + (i + 1) * dim);
        Codebook cb;
        cb.k = k;
        cb.grid_size = dim;
        cb.entries.assign(entries, entries + static_cast<std::size_t>(k) * dim);
        const std::vector<std::uint32_t> idx = assign_indices(recs, cb);
        std::memcpy(out, idx.data(), idx.size() * sizeof(std::uint32_t));
    });
}

// kmeans_codebook gsb.cpp:236 (entries out: k x dim); returns iterations via *iters
int hqref_kmeans_codebook(const double* shapes, std::uint64_t n, int dim, int k, int max_iters,
                          std::uint64_t seed, double* entries, int* iters) {
    return guarded([&] {
        std::vector<ShapeRecord> recs(n);
        for (std::uint64_t i = 0; i < n; ++i) recs[i].shape.assign(shapes + i * dim, shapes + (i + 1) * dim);
        KMeansConfig cfg;
        cfg.max_iters = max_iters;
        cfg.seed = seed;
        const Codebook cb = kmeans_codebook(recs, k, cfg);
        std::memcpy(entries, cb.entries.data(), cb.entries.size() * sizeof(double));
        if (iters) *iters = cb.training_meta.iterations;
    });
}

}  // extern "C"
