// Parity tests of the C++ drop-in (include/holoquant/lutham_b200.hpp), written
// the way the reference's own doctest suites are (proj/tests/test_lutham.cpp):
// the host Model is built with the reference's build_model, the device head
// with the drop-in, and results are compared against holoquant's own
// compressed_forward / deserialize (linked from oracle/_ref, the unmodified
// reference, as the checker).
//
//   test_lutham_b200 cpu   cases that need no GPU (planner, file faults)
//   test_lutham_b200 gpu   device cases (forward parity, errors, interp_ops)
#include <atomic>
#include <cmath>
#include <algorithm>
#include <cstdlib>
#include <new>
#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "holoquant/lutham_b200.hpp"
#include "holoquant/trainer.hpp"

using namespace holoquant;

// operator new counting, as the reference's acceptance check 7
// (acceptance.cpp:426-447): every heap allocation of the process, including
// those made inside libskan.so, goes through these while tracking is on.
static std::atomic<std::uint64_t> g_alloc_count{0};
static std::atomic<bool> g_alloc_tracking{false};
void* operator new(std::size_t n) {
    if (g_alloc_tracking.load(std::memory_order_relaxed)) g_alloc_count.fetch_add(1, std::memory_order_relaxed);
    if (void* p = std::malloc(n ? n : 1)) return p;
    throw std::bad_alloc();
}
void operator delete(void* p) noexcept { std::free(p); }
void operator delete(void* p, std::size_t) noexcept { std::free(p); }

namespace {

int g_failed = 0, g_checks = 0;
std::vector<std::pair<std::string, std::function<void()>>> g_cpu, g_gpu;

#define CHECK(cond)                                                                  \
    do {                                                                             \
        ++g_checks;                                                                  \
        if (!(cond)) {                                                               \
            ++g_failed;                                                              \
            std::fprintf(stderr, "  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                            \
    } while (0)

template <class E, class F>
bool throws_as(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}
#define CHECK_THROWS_AS(expr, E) CHECK(throws_as<E>([&] { expr; }))

struct Reg {
    Reg(std::vector<std::pair<std::string, std::function<void()>>>& v, const char* n, std::function<void()> f) {
        v.emplace_back(n, std::move(f));
    }
};
#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define TEST_CPU(name) \
    static void CAT(t_, __LINE__)(); static Reg CAT(r_, __LINE__)(g_cpu, name, CAT(t_, __LINE__)); static void CAT(t_, __LINE__)()
#define TEST_GPU(name) \
    static void CAT(t_, __LINE__)(); static Reg CAT(r_, __LINE__)(g_gpu, name, CAT(t_, __LINE__)); static void CAT(t_, __LINE__)()

// test_lutham.cpp:124-145's crafted_layer (K may exceed the edge count)
CompressedLayer crafted_layer(int in, int out, int G, int k, std::uint64_t seed, double gscale = 1.0,
                              double bscale = 1.0) {
    CompressedLayer cl;
    cl.in_dim = in;
    cl.out_dim = out;
    cl.grid_size = G;
    cl.codebook.k = k;
    cl.codebook.grid_size = G;
    cl.codebook.entries.resize(static_cast<std::size_t>(k) * G);
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    for (double& x : cl.codebook.entries) x = u(rng);
    const std::int64_t e = cl.edge_count();
    cl.indices.resize(e);
    cl.gains.resize(e);
    cl.biases.resize(e);
    for (std::int64_t n = 0; n < e; ++n) {
        cl.indices[n] = static_cast<std::uint32_t>(rng() % k);
        cl.gains[n] = ((n % 5 == 0) ? 0.0 : std::fabs(u(rng)) + 0.01) * gscale;
        cl.biases[n] = u(rng) * bscale;
    }
    return cl;
}

CompressedNetwork head(std::vector<int> dims, int G, int k, bool int8, std::uint64_t seed) {
    CompressedNetwork cn;
    for (std::size_t l = 0; l + 1 < dims.size(); ++l)
        cn.layers.push_back(crafted_layer(dims[l], dims[l + 1], G, k, seed + 101 * l, 1.0 / std::sqrt(dims[l]),
                                          1.0 / dims[l]));
    return int8 ? quantize_compressed_network(cn) : cn;
}

std::vector<double> inputs(int batch, int width, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> u(-1.5, 1.5);  // test_lutham.cpp:377, ~33% clamped
    std::vector<double> x(static_cast<std::size_t>(batch) * width);
    for (double& v : x) v = u(rng);
    for (std::size_t n = 0; n < x.size(); n += 97) x[n] = node_position(-1.0, 1.0, 10, static_cast<int>(n % 10));
    return x;
}

bool bitwise_equal(const std::vector<double>& a, const std::vector<double>& b) {
    return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(double)) == 0;
}

// Per-output L1 scale max(|y|, sum_i |term_ij|) of the reconstructed dense
// network (to_dense_network), evaluated with the reference's eval_spline.
std::vector<double> l1_scale(const Model& model, const std::vector<double>& x, int batch) {
    const KanNetwork net = to_dense_network(model);
    std::vector<double> out;
    for (int s = 0; s < batch; ++s) {
        std::vector<double> cur(x.begin() + static_cast<std::ptrdiff_t>(s) * net.input_dim(),
                                x.begin() + static_cast<std::ptrdiff_t>(s + 1) * net.input_dim());
        std::vector<double> scale;
        for (const KanLayer& L : net.layers()) {
            std::vector<double> y(L.out_dim(), 0.0), a(L.out_dim(), 0.0);
            for (int i = 0; i < L.in_dim(); ++i)
                for (int j = 0; j < L.out_dim(); ++j) {
                    const double t = eval_spline(L.grid(i, j), L.domain_lo(), L.domain_hi(), cur[i]);
                    y[j] += t;
                    a[j] += std::fabs(t);
                }
            scale.assign(L.out_dim(), 0.0);
            for (int j = 0; j < L.out_dim(); ++j) scale[j] = std::max(std::fabs(y[j]), a[j]);
            cur = y;
        }
        out.insert(out.end(), scale.begin(), scale.end());
    }
    return out;
}

std::vector<double> ref_forward(const Model& m, const std::vector<double>& x, int batch) {
    Workspace ws = make_workspace(m);
    std::vector<double> y(static_cast<std::size_t>(batch) * m.output_dim());
    compressed_forward(m, x, batch, y, ws);
    return y;
}

std::vector<double> dev_forward(const DeviceHead& h, const std::vector<double>& x, int batch, DeviceMode mode,
                                int max_batch = 64) {
    DeviceWorkspace ws = make_workspace(h, max_batch);
    std::vector<double> y(static_cast<std::size_t>(batch) * h.output_dim());
    compressed_forward(h, x, batch, y, ws, mode);
    return y;
}

// ---------------------------------------------------------------------------
// no GPU needed

TEST_CPU("C ABI planner equals holoquant::plan_memory (test_lutham.cpp:56-95, 495-505)") {
    for (bool q : {false, true}) {
        for (auto [in, out, G, k] : {std::tuple{2, 3, 10, 16}, std::tuple{1000, 3200, 10, 65536},
                                     std::tuple{7, 9, 5, 70000}, std::tuple{3, 4, 6, 1}}) {
            LayerHeader h;
            h.in_dim = in;
            h.out_dim = out;
            h.grid_size = G;
            h.k = k;
            h.flags = q ? kFlagInt8 : 0u;
            ModelHeader mh;
            mh.layers = {h};
            const MemoryPlan want = plan_memory(mh);
            skan_layer_header c = b200_detail::to_c(h);
            skan_layer_plan lp{};
            skan_memory_plan tot{};
            CHECK(skan_plan_memory(&c, 1, &lp, &tot) == SKAN_OK);
            CHECK(lp.codebook_bytes == want.layers[0].codebook_bytes);
            CHECK(lp.index_bytes == want.layers[0].index_bytes);
            CHECK(lp.unpacked_index_bytes == want.layers[0].unpacked_index_bytes);
            CHECK(lp.gain_bytes == want.layers[0].gain_bytes);
            CHECK(lp.bias_bytes == want.layers[0].bias_bytes);
            CHECK(tot.payload_total == want.payload_total);
            CHECK(tot.working_set_total == want.working_set_total);
            CHECK(tot.scratch_bytes == want.scratch_bytes);
        }
    }
}

TEST_CPU("corrupted files throw holoquant::FormatError with the reference's fault and offset") {
    const Model model = build_model(head({3, 5, 2}, 6, 7, true, 11));
    const std::vector<std::uint8_t> good = serialize(model);
    auto mutate = [&](std::size_t at, std::uint8_t v) {
        std::vector<std::uint8_t> b = good;
        b[at] = v;
        return b;
    };
    std::vector<std::vector<std::uint8_t>> cases = {mutate(0, 'X'), mutate(4, 9), mutate(8, 0), mutate(12, 0),
                                                    mutate(16, 0), std::vector<std::uint8_t>(good.begin(), good.begin() + 10),
                                                    std::vector<std::uint8_t>(good.begin(), good.begin() + 200)};
    for (const auto& b : cases) {
        FormatFault ref_fault{};
        std::uint64_t ref_off = 0;
        bool ref_threw = false;
        try {
            (void)deserialize(b);
        } catch (const FormatError& e) {
            ref_threw = true;
            ref_fault = e.fault;
            ref_off = e.offset;
        } catch (...) {
        }
        bool dev_threw = false;
        try {
            (void)deserialize_device(b);
        } catch (const FormatError& e) {
            dev_threw = true;
            CHECK(e.fault == ref_fault);
            CHECK(e.offset == ref_off);
        } catch (...) {
        }
        CHECK(ref_threw == dev_threw);
    }
}

// ---------------------------------------------------------------------------
// device

// faults found on the device (index range checks before a late truncation,
// an index >= K) and the hot swap from SKAN bytes: the reference's fault and
// offset; a failed swap leaves the resident head unchanged
TEST_GPU("SKAN bytes on the device: index faults, late truncation, swap from bytes") {
    const Model model = build_model(head({3, 5, 2}, 6, 7, true, 11));
    const std::vector<std::uint8_t> good = serialize(model);
    auto same_fault = [&](const std::vector<std::uint8_t>& b) {
        FormatFault rf{};
        std::uint64_t ro = 0;
        bool rt = false, dt = false;
        try {
            (void)deserialize(b);
        } catch (const FormatError& e) {
            rt = true;
            rf = e.fault;
            ro = e.offset;
        }
        try {
            (void)deserialize_device(b);
        } catch (const FormatError& e) {
            dt = true;
            CHECK(e.fault == rf);
            CHECK(e.offset == ro);
        } catch (...) {
        }
        CHECK(rt && dt);
    };
    same_fault(std::vector<std::uint8_t>(good.begin(), good.end() - 5));
    // the first index section: set every index bit -> 7 >= K = 7
    std::vector<std::uint8_t> bad = good;
    const std::size_t first_index = 192 + 64;  // 16 + 2*72 -> 192 (codebook 7*6 B), next 64-B boundary
    bad[first_index] = 0xFF;
    same_fault(bad);
    // swap from bytes: a second model of the same shapes, then a corrupt file
    const Model other = build_model(head({3, 5, 2}, 6, 7, true, 12));
    DeviceHead dev = deserialize_device(good);
    swap_device_model(dev, serialize(other));
    const std::vector<double> x = inputs(4, 3, 5);
    CHECK(bitwise_equal(dev_forward(dev, x, 4, DeviceMode::Exact), ref_forward(other, x, 4)));
    CHECK(throws_as<FormatError>([&] { swap_device_model(dev, std::span<const std::uint8_t>(bad)); }));
    CHECK(bitwise_equal(dev_forward(dev, x, 4, DeviceMode::Exact), ref_forward(other, x, 4)));
}

TEST_GPU("upload(build_model(cn)): exact mode is bitwise holoquant::compressed_forward") {
    for (bool q : {false, true}) {
        for (auto [dims, G, k] : {std::tuple{std::vector<int>{40, 33, 6}, 7, 300},
                                  std::tuple{std::vector<int>{256, 256}, 10, 256},
                                  std::tuple{std::vector<int>{7, 9, 5}, 5, 70000}}) {
            const Model model = build_model(head(dims, G, k, q, 5));
            const DeviceHead dev = upload(model);
            for (int batch : {1, 3, 17}) {
                const std::vector<double> x = inputs(batch, dims[0], 100 + batch);
                CHECK(bitwise_equal(dev_forward(dev, x, batch, DeviceMode::Exact), ref_forward(model, x, batch)));
            }
        }
    }
}

TEST_GPU("build_device_model(cn) == upload(build_model(cn)), and fast mode within 1e-5 (L1-scaled)") {
    for (bool q : {false, true}) {
        const CompressedNetwork cn = head({64, 48, 5}, 10, 256, q, 3);
        const Model model = build_model(cn);
        const DeviceHead a = build_device_model(cn), b = upload(model);
        for (int batch : {1, 5, 64}) {
            const std::vector<double> x = inputs(batch, 64, 7 + batch);
            const std::vector<double> want = ref_forward(model, x, batch);
            CHECK(bitwise_equal(dev_forward(a, x, batch, DeviceMode::Exact), want));
            const std::vector<double> fast = dev_forward(b, x, batch, DeviceMode::Fast);
            const std::vector<double> scale = l1_scale(model, x, batch);
            for (std::size_t n = 0; n < want.size(); ++n) CHECK(std::fabs(fast[n] - want[n]) <= 1e-5 * scale[n]);
        }
    }
}

TEST_GPU("deserialize_device(serialize(model)) forwards bitwise like the reference") {
    const Model model = build_model(head({3, 5, 2}, 6, 7, true, 21));
    const DeviceHead dev = deserialize_device(serialize(model));
    CHECK(dev.header().layers.size() == model.layers.size());
    const std::vector<double> x = inputs(4, 3, 1);
    CHECK(bitwise_equal(dev_forward(dev, x, 4, DeviceMode::Exact), ref_forward(model, x, 4)));
    const MemoryPlan p = plan_memory(dev), want = plan_memory(model.header());
    CHECK(p.payload_total == want.payload_total);
}

TEST_GPU("errors, batch 0 and interp_ops follow compressed_forward (lutham.cpp:819-850)") {
    const Model model = build_model(head({2, 4, 1}, 5, 3, false, 18));
    const DeviceHead dev = upload(model);
    DeviceWorkspace ws = make_workspace(dev, 8);
    std::vector<double> x(7 * 2, 0.25), y(7);
    compressed_forward(dev, x, 7, y, ws);
    CHECK(ws.interp_ops() == 7u * (2 * 4 + 4 * 1));
    compressed_forward(dev, std::span<const double>(), 0, std::span<double>(), ws);
    CHECK(ws.interp_ops() == 7u * (2 * 4 + 4 * 1));
    CHECK_THROWS_AS(compressed_forward(dev, std::span<const double>(x.data(), 3), 7, y, ws), ShapeError);
    CHECK_THROWS_AS(compressed_forward(dev, x, 7, std::span<double>(y.data(), 6), ws), ShapeError);
    CHECK_THROWS_AS(compressed_forward(dev, x, -1, y, ws), ShapeError);
    x[3] = std::nan("");
    CHECK_THROWS_AS(compressed_forward(dev, x, 7, y, ws), ValueError);
    const DeviceHead wide = upload(build_model(head({300, 2}, 5, 3, false, 19)));
    std::vector<double> y2(2);
    CHECK_THROWS_AS(compressed_forward(wide, std::vector<double>(300, 0.0), 1, y2, ws), ContractError);
    CHECK_THROWS_AS(compressed_forward(wide, std::vector<double>(299, 0.0), 1, y2, ws), ShapeError);  // spans first
    CompressedNetwork bad = head({2, 2}, 5, 3, false, 20);
    bad.layers[0].indices[0] = 3;  // index >= K
    CHECK_THROWS_AS(build_device_model(bad), ContractError);
}

TEST_GPU("swap_device_model: a resident head refilled in place forwards like the new model") {
    const CompressedNetwork a = head({64, 48, 5}, 10, 256, true, 31), b = head({64, 48, 5}, 10, 256, true, 32);
    DeviceHead dev = build_device_model(a);
    DeviceWorkspace ws = make_workspace(dev, 8);
    swap_device_model(dev, b);
    const std::vector<double> x = inputs(4, 64, 5);
    std::vector<double> y(4 * 5);
    compressed_forward(dev, x, 4, y, ws, DeviceMode::Exact);
    CHECK(bitwise_equal(y, ref_forward(build_model(b), x, 4)));
    CHECK_THROWS_AS(swap_device_model(dev, head({64, 40, 5}, 10, 256, true, 33)), ContractError);
}

TEST_GPU("assign_indices_device == holoquant::assign_indices (test_gsb.cpp:104-132), ties to the lowest row") {
    std::mt19937_64 rng(6);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    std::vector<ShapeRecord> pts(300);
    for (auto& p : pts) {
        p.shape.resize(6);
        for (double& x : p.shape) x = u(rng);
    }
    KMeansConfig cfg;
    cfg.seed = 2;
    Codebook cb = kmeans_codebook(pts, 12, cfg);
    CHECK(assign_indices_device(pts, cb) == assign_indices(pts, cb));
    // duplicated rows: every tie resolves to the first copy
    cb.entries.insert(cb.entries.end(), cb.entries.begin(), cb.entries.end());
    cb.k *= 2;
    const std::vector<std::uint32_t> got = assign_indices_device(pts, cb);
    CHECK(got == assign_indices(pts, cb));
    CHECK(*std::max_element(got.begin(), got.end()) < 12u);
    pts[7].shape.pop_back();
    CHECK_THROWS_AS(assign_indices_device(pts, cb), ShapeError);
}

TEST_GPU("cfg2 head {2048,1408,20} K=65536 int8: batch 1 fast within tolerance, exact bitwise") {
    const CompressedNetwork cn = head({2048, 1408, 20}, 10, 65536, true, 2026);
    const Model model = build_model(cn);
    const DeviceHead dev = upload(model);
    const std::vector<double> x = inputs(2, 2048, 9);
    const std::vector<double> want = ref_forward(model, x, 2);
    CHECK(bitwise_equal(dev_forward(dev, x, 2, DeviceMode::Exact), want));
    const std::vector<double> x1(x.begin(), x.begin() + 2048);
    const std::vector<double> w1(want.begin(), want.begin() + 20);
    const std::vector<double> f1 = dev_forward(dev, x1, 1, DeviceMode::Fast);
    const std::vector<double> scale = l1_scale(model, x1, 1);
    for (int j = 0; j < 20; ++j) CHECK(std::fabs(f1[j] - w1[j]) <= 1e-5 * scale[j]);
}

// acceptance.cpp:426-447 (check 7): 1000 drop-in forwards at batch 8 after
// warm-up make zero heap allocations; here through the device head, in both
// modes, on the reference's check-7 network and on the cfg2 head (whose
// batch 8 runs the tensor-core GEMM route) and its batch-1 persistent path.
TEST_GPU("zero-allocation forward: 1000 calls at B=8 (acceptance.cpp:426-447), both modes") {
    const KanNetwork net = init_network(std::vector<int>{4, 24, 2}, 12, 0.4, 95);
    VqConfig cfg;
    cfg.k = 32;
    cfg.seed = 96;
    cfg.int8 = true;
    const Model small = build_model(compress_network(net, cfg));
    const Model big = build_model(head({2048, 1408, 20}, 10, 65536, true, 2026));
    struct Case {
        const Model* m;
        int batch, calls;
    };
    for (const Case c : {Case{&small, 8, 1000}, Case{&big, 8, 1000}, Case{&big, 1, 1000}}) {
        const DeviceHead dev = upload(*c.m);
        DeviceWorkspace ws = make_workspace(dev, 8);
        const int in = c.m->input_dim();
        const int out = c.m->output_dim();
        std::vector<double> x(static_cast<std::size_t>(c.batch) * in, 0.3), y(static_cast<std::size_t>(c.batch) * out);
        for (DeviceMode mode : {DeviceMode::Fast, DeviceMode::Exact}) {
            for (int warm = 0; warm < 3; ++warm) compressed_forward(dev, x, c.batch, y, ws, mode);
            g_alloc_count.store(0);
            g_alloc_tracking.store(true);
            for (int call = 0; call < c.calls; ++call) compressed_forward(dev, x, c.batch, y, ws, mode);
            g_alloc_tracking.store(false);
            const std::uint64_t n = g_alloc_count.load();
            if (n) std::fprintf(stderr, "  %llu allocations (in %d, batch %d, mode %d)\n",
                                static_cast<unsigned long long>(n), in, c.batch, static_cast<int>(mode));
            CHECK(n == 0);
        }
    }
}

}  // namespace

int main(int argc, char** argv) {
    const std::string which = argc > 1 ? argv[1] : "all";
    auto run = [](auto& v) {
        for (auto& [name, f] : v) {
            const int before = g_failed;
            try {
                f();
            } catch (const std::exception& e) {
                ++g_failed;
                std::fprintf(stderr, "  unexpected exception: %s\n", e.what());
            }
            std::printf("%s %s\n", g_failed == before ? "PASS" : "FAIL", name.c_str());
        }
    };
    if (which == "cpu" || which == "all") run(g_cpu);
    if (which == "gpu" || which == "all") run(g_gpu);
    std::printf("%d checks, %d failed\n", g_checks, g_failed);
    return g_failed ? 1 : 0;
}
