// Internal types shared by the C-ABI host code (skan_api.cpp, skan_format.cpp)
// and the sm_100a kernels (skan_kernels.cu).  Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "skan.h"

namespace skan {

// ---------------------------------------------------------------------------
// Errors: C++ exceptions inside the library, converted to skan_status at the
// ABI boundary (skan_api.cpp: guarded()).  Mirrors errors.hpp.
struct Error : std::runtime_error {
    skan_status status;
    uint64_t offset;
    int fault;
    Error(skan_status s, const std::string& m, uint64_t off = 0, int f = SKAN_FAULT_NONE)
        : std::runtime_error(m), status(s), offset(off), fault(f) {}
};

[[noreturn]] inline void raise(skan_status s, const std::string& m) { throw Error(s, m); }
[[noreturn]] inline void raise_format(int fault, uint64_t off, const std::string& m) {
    throw Error(SKAN_FORMAT_ERROR, m + " (byte offset " + std::to_string(off) + ")", off, fault);
}

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) raise(SKAN_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device,
// size) and thread: a fixed per-thread table, so the per-call launch path
// makes no driver attribute call and allocates nothing.
inline void ensure_smem(const void* f, size_t bytes) {
    if (bytes <= 48 * 1024) return;
    struct Entry {
        const void* f;
        int dev;
        size_t bytes;
    };
    thread_local Entry tab[64];
    thread_local int n = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    for (int i = 0; i < n; ++i)
        if (tab[i].f == f && tab[i].dev == dev) {
            if (tab[i].bytes >= bytes) return;
            cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
            tab[i].bytes = bytes;
            return;
        }
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
    if (n < 64) tab[n++] = Entry{f, dev, bytes};
}
template <class K>
inline void ensure_smem(K* kernel, size_t bytes) {
    ensure_smem(reinterpret_cast<const void*>(kernel), bytes);
}

// ---------------------------------------------------------------------------
// Resident device formats of one layer.
enum Fmt : int {
    // int8 tables, K <= 65536: one 32-bit record per edge
    //   bits 0-15 codebook row, 16-23 log-gain code, 24-31 linear bias code
    // (PAPER.md:193-194's 32 bits/edge), codebook int8 K x G.
    FMT_I8_R32 = 0,
    // int8 tables, K > 65536: u32 row index + u16 (gain code | bias code << 8)
    FMT_I8_WIDE = 1,
    // f32 tables: u32 row index, f32 gain, f32 bias, f32 codebook K x G
    FMT_F32 = 2,
    // dense layer (k == 0): f32 grid E x G (lutham.cpp:778-791)
    FMT_DENSE = 3,
};

// Everything a kernel needs about one layer; passed by value as a kernel
// parameter.  All pointers are device pointers into the head's single
// resident allocation.
struct DevLayer {
    int in, out, G, K, fmt;
    double lo, hi, dx;  // dx = (hi - lo) / (G - 1), computed once on the host (IEEE, as kan.cpp:24)
    double cs, bs;      // int8 codebook scale, bias scale
    const uint32_t* rec;     // FMT_I8_R32
    const uint32_t* idx;     // FMT_I8_WIDE / FMT_F32 (nullptr when K == 1)
    const uint16_t* gb;      // FMT_I8_WIDE
    const float* gain;       // FMT_F32
    const float* bias;       // FMT_F32
    const int8_t* cb8;       // int8 codebook
    const uint8_t* cb8u;     // the same rows, codes biased to c ^ 0x80 (layer GEMM decode)
    const float* cb32;       // f32 codebook, or dense grid
    const float* lutf;       // [128] float(gain(code) * cs) — fast int8 path
    const double* lutd;      // [128] gain(code) as dequantize_gain_code returns it
    const double* bias_sum;  // [out] sum_i b_ij in i order — fast path
    const uint16_t* pair8;   // int8 pair planes [G-1][K]: c[k][m] | c[k][m+1] << 8 — one 2-byte
                             // gather per edge-sample; plane m is contiguous (smem-stageable)
    int rs;                  // int8 codebook row stride in bytes (G rounded up to 16)
    const double* node;      // [G] node positions exactly as kan.cpp:21-26 computes them
    const long long* nkey;   // [G] their order-preserving integer keys (fast locate)
    double inv_dx;           // 1/dx: fast locate's bracket estimate
    double q_eps;            // fast locate trusts floor((x-lo)*inv_dx) when its fraction is
                             // more than q_eps from an integer (< 0: always search)
    float lo_f, inv_dx_f;    // float(lo), float(1/dx): fast locate's t
    float hi_f;              // float(hi)
    float qf_eps;            // bracket_f32 trusts its fp32 bracket when the fraction of
                             // (float(x)-lo_f)*inv_dx_f is more than qf_eps from an integer (< 0: never)
    // fast-path int8 gain, computed instead of looked up:
    //   float(gain(code) * cs) ~= exp2(g_base + code * g_step), code 127 -> 0
    // with g_base = log_min + log2(cs) (dequantize_gain_code, quant.cpp:88-91)
    float g_base, g_step;
    // dense layers: the grid again, pre-tiled in the layer GEMM's shared-memory
    // layout (one TMA bulk copy per chunk, skan_gemm.cu); wt_nch = chunks per
    // output block
    const float* wt;
    int wt_nch;
    // dense tiled layers: power-of-two scale putting max|W| * wsc in [2^14, 2^15)
    // for the fp16 split-precision GEMM (0: no fp16 path, e.g. non-finite grid)
    float wsc;
};

// Per-layer launch plan for one batch size (chosen on the host).
struct LaunchCfg {
    int tj;      // outputs per CTA (32/64/128)
    int spt;     // samples per thread (1/2/4/8)
    int jt, st;  // CTA tiles along j and samples
    int nsplit;  // i-splits (fast path); 1 in exact mode
    int ichunk;  // inputs per split
    int kind;    // fast path kernel: 0 = rows-in-warps (small batch), 1 = samples-in-lanes
                 // (large batch), 2 = pair planes in shared memory (batch 1), 4 = tensor-core
                 // GEMM over the knot basis (large batch, wide layers; skan_gemm.cu),
                 // 5 = narrow dense layer on the CUDA cores (skan_gemm.cu)
    int vj;      // outputs per lane (small kernel); GEMM: W stages
    int rw;      // rows per warp (small kernel); GEMM: dense TMA ring slots
    int ic;      // inputs per staged chunk (large kernel)
    size_t smem; // dynamic shared memory bytes (large kernel)
    int persist; // GEMM: 1 / 2 = dense layer on the persistent schedule (k_dense_persist, tf32 / fp16;
                 // batch <= 64); 3 = int8 layer GEMM in fp16 split precision
    int dn_nch;  // persistent dense: chunks per output tile
};

// Arguments of one fused fast-path layer launch (k_fwd_small / k_fwd_large).
// Each CTA accumulates a row-block (i-split) of edges; the last CTA to finish
// a (j-tile, sample-tile) reduces the split partials in fixed order in
// double, adds the bias sums, writes the layer output and the next layer's
// knot brackets.
struct FwdArgs {
    DevLayer L;
    int B;
    int rows_per_cta;       // inputs per split
    const double* x;        // non-null: locate inline from these f64 inputs [B][in]
    const int* bm_in;       // else: brackets, input-major [in][B], from the previous
    const float* bt_in;     //   layer's finisher or the locate kernel
    float* partial;         // [nsplit][B][out]
    unsigned* counters;     // [jt * st], zero between launches
    double* y;              // [B][out]
    int has_next;
    DevLayer N;             // next layer (its knot grid), valid when has_next
    int* bm_out;            // next layer brackets, input-major [out][B]
    float* bt_out;
    int* err;
    // The previous layer ran the pair-plane kernel and left split partials
    // instead of brackets: this launch reduces them (fixed order, double)
    // for the rows it consumes, adds the previous bias sums, and locates.
    const float* prev_partial;    // [prev_nsplit][B][in]
    int prev_nsplit;
    const double* prev_bias_sum;  // [in]
    unsigned long long* dbg;      // layer GEMM phase stamps (skan_debug_gemm_timeline), or null
    int gemm_wst;                 // layer GEMM: W stages in shared memory (2 or 3)
    int gemm_ring;                // layer GEMM, dense: TMA ring slots
    int gemm_skip;                // experiment (SKAN_GEMM_SKIP): 16 = three N=128 MMAs per K step, 32 = two N=256
};

// Batch-1 persistent head kernel (skan_head_b1.cu).
constexpr int kMaxHeadLayers = 8;
struct HeadB1Args {
    int nl;
    DevLayer L[kMaxHeadLayers];
    int planes0;       // layer 0 served from shared-memory pair planes
    int x_tma;         // x may be bulk-copied (16-byte aligned, in0*8 % 16 == 0)
    const double* x;   // [in]
    double* y;         // [out]
    float* part[2];    // per-CTA partials, [grid][layer width], ping-pong by layer
    unsigned* done;    // [0] arrival counter of the last layer (last CTA reduces), [1] v2's grid
                       // barrier; both 0 at launch, reset to 0 by the last CTA
    unsigned epoch;    // value of *done when this launch starts (always 0 now)
    int* err;
    unsigned long long* timeline;  // optional: [grid][16] %globaltimer stamps per phase
    int rec_cap;           // layer-0 rows whose records are staged in shared memory
    unsigned pref_mask;    // row-split layers whose records are prefetched at kernel start
    unsigned pref_offset;  // byte offset of the prefetch region in dynamic shared memory
    unsigned cbrow_mask;   // v2: row-split layers whose edges' codebook rows are gathered
                           // into shared memory before the layer's inputs are known
    unsigned cbrow_offset; // v2: byte offset of that region in dynamic shared memory
    int version;           // 2 = k_head_b1v2 (static-bucket-free prologue), 1 = k_head_b1
    int exit_at;           // timing experiment (SKAN_B1_EXIT_AT): return after phase stamp n (0 = off)
    int nr1;               // v2: layer-1 rows per consumer block (stride of the consumer-blocked partials)
    unsigned out_offset;   // v2: byte offset of layer 0's per-CTA output staging in dynamic shared memory
    unsigned part_floats;  // floats per partial buffer (part[0], part[1]) the kernel needs
    const uint4* l1rows;   // v2: layer 1's edges' codebook rows, edge-major [in1*out1] x 16 B (built at
                           // upload from layer 1's records: head_b1_build_rows)
    double node0[33];      // layer 0's node positions (kan.cpp:21-26), G <= 33
};
bool head_b1_supported(const DevLayer* L, int nl);
// Shared-memory plan of the batch-1 kernel; fills h->planes0, rec_cap,
// pref_mask, pref_offset.
size_t head_b1_smem(const DevLayer* L, int nl, int num_sms, HeadB1Args* h);
cudaError_t launch_head_b1(const HeadB1Args& h, int grid, size_t smem, cudaStream_t s);
// v2: fill dst[e] = layer 1's codebook row of edge e (16 B) for all in1*out1 edges
size_t head_b1_rows_bytes(const HeadB1Args& h);
cudaError_t head_b1_build_rows(const HeadB1Args& h, uint4* dst, cudaStream_t s);
// Grid for which all CTAs are co-resident (one per SM), or 0 if the kernel
// cannot be resident at this shared-memory size.
int head_b1_max_grid(size_t smem, int num_sms);

// Workspace device buffers (one forward stream).
struct DevScratch {
    double* act[2];     // ping-pong activations [max_batch * max_width]
    int* bm;            // bracket index [max_batch * max_width]
    float* btf;         // bracket t (f32)
    double* btd;        // bracket t (f64)
    float* partial;     // split partial sums
    int* err;           // non-finite flag
    unsigned* counters; // per-layer (j-tile, sample-tile) arrival counters
    size_t counter_stride;  // counters per layer
};

// ---- kernel launchers (skan_kernels.cu) ----
void launch_locate_input(const double* x, int n_rows, int width, const DevLayer& L, int* bm,
                         float* btf, double* btd, int* err, cudaStream_t s, bool input_major = false);
// Fused fast-path layer (gather + split reduction + next-layer locate).
// pdl: launch with programmatic stream serialization (overlaps the
// prologue with the previous kernel's tail).
int launch_fwd_fast(const FwdArgs& a, const LaunchCfg& c, bool pdl, cudaStream_t s);  // returns the launches made
void launch_gather_exact(const DevLayer& L, const LaunchCfg& c, int B, const int* bm,
                         const double* btd, double* y, cudaStream_t s);
// Exact mode at small batch: terms in parallel into `terms` (term_doubles of
// scratch; blocks of inputs when it does not hold a whole layer), then the
// in-order sums per (sample, output), carried in `acc` [B * out].  Returns the
// launches made.
constexpr int kExactSplitMaxBatch = 128;
constexpr size_t kExactTermBytes = 256ull << 20;
// Exact mode, batch 1, int8 layer with pair planes: brackets + their order in
// one launch, the plane-ordered terms, the in-order sums (3 launches); 0 when
// the layer does not qualify (the caller takes the general path).
int launch_exact_b1(const DevLayer& L, const double* xin, int* bm, float* btf, double* btd, int* err, double* y,
                    double* terms, size_t term_doubles, double* acc, cudaStream_t s);
int launch_exact_split(const DevLayer& L, int B, const int* bm, const double* btd, double* y, double* terms,
                       size_t term_doubles, double* acc, cudaStream_t s);
void launch_locate_raw(const double* x, int n, double lo, double hi, int G, int* idx,
                       double* t, uint8_t* clamped, int* err, cudaStream_t s);
void launch_pli_lookup(const double* cb, int k, int G, const int* rows, const double* g,
                       const double* b, const double* x, double lo, double hi, int n, double* y,
                       int* err, cudaStream_t s);
void launch_unpack_indices(const uint8_t* bytes, uint64_t count, int bits, uint32_t* out,
                           cudaStream_t s);

// Tensor-core layer GEMM (skan_gemm.cu), kind 4 of LaunchCfg: two launches
// (the GEMM over input splits, then the fixed-order split reduction).
constexpr int kB1MaxBatch = 2;     // batches served by per-sample persistent batch-1 launches (B = 3 is
                                    // faster on the fp16 layer GEMM: 53 vs 57 us, profiles/r2/latency_by_batch.txt)
constexpr int kGemmMinBatch = 3;  // smallest batch routed to the tensor-core layer GEMM (default; heads the batch-1 kernel takes use it from 4)
extern int g_gemm_min_batch;      // current threshold (skan_debug_set_gemm_min_batch)
bool gemm_supported(const DevLayer& L);
LaunchCfg gemm_cfg(const DevLayer& L, int B, int num_sms);
int gemm_ic(int G);
uint64_t dense_tile_floats(int in, int out, int G);
void build_dense_tiles(const DevLayer& L, float* wt, const float* src, int ch0, int ch1, cudaStream_t s);
float dense_fp16_scale(const float* wt, uint64_t n, cudaStream_t s);
int launch_layer_gemm(const FwdArgs& a, const LaunchCfg& c, bool pdl, cudaStream_t s, bool with_reduce = true);
// Narrow dense layers (out <= 32, natural grid layout) at batch >= 3: CUDA-core
// split kernel + fixed-order reduction (skan_gemm.cu).  LaunchCfg::kind 5.
bool dense_narrow_ok(const DevLayer& L);
LaunchCfg dense_narrow_cfg(const DevLayer& L, int B, int num_sms);
int launch_dense_narrow(const FwdArgs& a, const LaunchCfg& c, bool pdl, cudaStream_t s);
// MMA work one k_layer_gemm launch issues (flops, as 2*M*N*K per tcgen05.mma)
double gemm_issued_flops(const DevLayer& L, const LaunchCfg& c, int B);

// ---- SKAN v1 direct-to-device load (skan_load.cu, skan_format.cpp) ----
// Device pointers to one layer's sections inside a device copy of the file.
struct LayerSrc {
    const uint8_t* codebook;  // K x G int8 / f32 codebook, or the dense E x G f32 grid
    const uint8_t* index;     // packed LSB-first row indices (bits = bit_width(K - 1))
    uint64_t index_bytes;
    const uint8_t* gain;      // E int8 codes or f32
    const uint8_t* bias;
};
// Range check of a packed index section: atomicMin of the first edge >= K into *bad.
void check_index_section(const uint8_t* index, uint64_t index_bytes, int bits, uint32_t K, uint64_t E,
                         unsigned long long* bad, cudaStream_t s);
// Fill layer d's resident regions (records, codebook tables, bias sums) from its sections.
void build_layer_from_sections(const DevLayer& d, const LayerSrc& src, int bits, cudaStream_t s);
struct SectionLayer {
    skan_layer_header h;
    LayerSrc src;
    int bits;
};
// Create a head / hot-swap a resident head from sections already in device
// memory (skan_api.cpp; throws skan::Error).
skan_head* create_head_from_sections(const SectionLayer* layers, int n, int device);
void swap_head_from_sections(skan_head* h, const SectionLayer* layers, int n, cudaStream_t stream);

// Record a thread-local error for skan_last_error and return its status.
skan_status set_error(skan_status s, const std::string& msg, uint64_t offset, int fault);

// allow_planes: the layer has a successor that can reduce its split
// partials (the pair-plane kernel writes partials, not brackets).
LaunchCfg choose_cfg(const DevLayer& L, int B, bool exact, int num_sms, bool allow_planes = false);

}  // namespace skan
