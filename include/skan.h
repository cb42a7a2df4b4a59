/*
 * skan.h — C ABI of the B200-native LUTHAM forward (SHARe-KAN compressed
 * KAN heads).  Drop-in for the reference's C++ operator API in
 * /root/reference/proj/include/holoquant/lutham.hpp (+ gsb.hpp, errors.hpp);
 * every entry point below names the reference interface it replaces.
 *
 * Conventions
 *   - plain pointers + sizes, no C++ or torch types; no exceptions cross the
 *     ABI: every call returns a skan_status and records a thread-local error
 *     (skan_last_error) whose code maps 1:1 onto the reference exception
 *     taxonomy (errors.hpp:10-60).
 *   - all tables are edge-major, edge e = i*out_dim + j (kan.hpp:40-42,
 *     gsb.hpp:98); codebooks are K x G row-major (gsb.hpp:42).
 *   - heads are immutable after creation and may be shared by concurrent
 *     streams; each stream owns a skan_workspace.
 *   - all device memory is allocated at head/workspace creation from a
 *     static plan; skan_forward never allocates (acceptance.cpp:426-447).
 */
#ifndef SKAN_H
#define SKAN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SKAN_ABI_VERSION 1

/* Status codes <-> holoquant exceptions (errors.hpp). */
typedef enum {
    SKAN_OK = 0,
    SKAN_SHAPE_ERROR = 1,    /* holoquant::ShapeError    (errors.hpp:10-13)  */
    SKAN_VALUE_ERROR = 2,    /* holoquant::ValueError    (errors.hpp:15-18)  */
    SKAN_CONTRACT_ERROR = 3, /* holoquant::ContractError (errors.hpp:20-23)  */
    SKAN_FORMAT_ERROR = 4,   /* holoquant::FormatError   (errors.hpp:48-55)  */
    SKAN_PLAN_ERROR = 5,     /* holoquant::PlanError     (errors.hpp:58-60)  */
    SKAN_CUDA_ERROR = 6,     /* device failure (no reference counterpart)    */
} skan_status;

/* holoquant::FormatFault (errors.hpp:37-45), same order. */
typedef enum {
    SKAN_FAULT_NONE = -1,
    SKAN_FAULT_BAD_MAGIC = 0,
    SKAN_FAULT_BAD_VERSION = 1,
    SKAN_FAULT_BAD_ENDIANNESS = 2,
    SKAN_FAULT_BAD_HEADER = 3,
    SKAN_FAULT_TRUNCATED = 4,
    SKAN_FAULT_INDEX_OUT_OF_RANGE = 5,
    SKAN_FAULT_BAD_QUANT_PARAM = 6,
} skan_format_fault;

#define SKAN_FLAG_INT8 1u /* kFlagInt8, lutham.hpp:27 */

/* holoquant::LayerHeader (lutham.hpp:30-49); k == 0 marks a dense layer. */
typedef struct {
    uint32_t in_dim, out_dim, grid_size, k;
    double domain_lo, domain_hi;
    uint32_t flags, reserved;
    double codebook_scale, gain_log_min, gain_log_step, bias_scale;
} skan_layer_header;

/* holoquant::LayerPlan (lutham.hpp:59-71) */
typedef struct {
    uint64_t codebook_bytes, index_bytes, unpacked_index_bytes, gain_bytes, bias_bytes;
    /* B200 resident form actually allocated for this layer (records,
     * codebook, gain LUT, bias sums). */
    uint64_t device_bytes;
} skan_layer_plan;

/* holoquant::MemoryPlan (lutham.hpp:74-80) */
typedef struct {
    uint64_t scratch_bytes, payload_total, working_set_total;
    uint64_t device_total; /* sum of layer device_bytes */
} skan_memory_plan;

/* Layer descriptor kinds accepted by skan_head_create. */
typedef enum {
    /* holoquant::CompressedLayer (+ optional Int8Tables), gsb.hpp:82-106,
     * validated and converted exactly as build_model does (lutham.cpp:214-271):
     * the f32 path casts codebook/gains/biases to float, the int8 path keeps
     * the codes and the four quantization parameters. */
    SKAN_LAYER_COMPRESSED = 0,
    /* holoquant::KanLayer coefficients (E*G doubles), cast to float as
     * build_dense_model does (lutham.cpp:177-195). */
    SKAN_LAYER_DENSE = 1,
    /* holoquant::RuntimeLayer resident tables (lutham.hpp:91-109) as produced
     * by build_model/deserialize; the form a `DeviceHead upload(const Model&)`
     * shim passes through unchanged. */
    SKAN_LAYER_RUNTIME = 2,
} skan_layer_kind;

typedef struct {
    int kind; /* skan_layer_kind */
    skan_layer_header header; /* dims, G, K, domain; int8 flag + params for RUNTIME */

    /* SKAN_LAYER_COMPRESSED (lengths are checked like build_model) */
    const double* codebook;       /* n_codebook = K*G */
    uint64_t n_codebook;
    const uint32_t* indices;      /* n_edges */
    const double* gains;          /* n_edges, must be >= 0 */
    const double* biases;         /* n_edges */
    uint64_t n_indices, n_gains, n_biases;
    int has_int8;                 /* Int8Tables present */
    const int8_t* codebook_codes; /* K*G */
    const int8_t* gain_codes;     /* E, log codes, 127 == exact zero */
    const int8_t* bias_codes;     /* E */
    uint64_t n_codebook_codes, n_gain_codes, n_bias_codes;
    double codebook_scale, gain_log_min, gain_log_step, bias_scale;

    /* SKAN_LAYER_DENSE */
    const double* coefficients;   /* E*G */
    uint64_t n_coefficients;

    /* SKAN_LAYER_RUNTIME (exactly one of table_f32/table_i8; idx16 for
     * 1 < K <= 65536, idx32 for K > 65536, neither for K == 1) */
    const float* table_f32;
    const int8_t* table_i8;
    const uint16_t* idx16;
    const uint32_t* idx32;
    const float* gains_f32;
    const float* biases_f32;
    const int8_t* rt_gain_codes;
    const int8_t* rt_bias_codes;
} skan_layer_desc;

typedef struct skan_head skan_head;
typedef struct skan_workspace skan_workspace;

/* Numerics mode of a forward call. */
typedef enum {
    /* fp32 per-edge math, double knot selection (bit-exact with locate),
     * fixed-order reduction of per-split partials in double: bit-reproducible
     * run to run, within 1e-5 (L1-scaled) of the reference. */
    SKAN_MODE_FAST = 0,
    /* fp64 per-edge math in the reference's operation order
     * ((g*c0+b)*w0 + (g*c1+b)*t, lutham.cpp:810), no FMA contraction, one
     * sequential i-ordered accumulation per output: bitwise identical to
     * holoquant::compressed_forward. */
    SKAN_MODE_EXACT = 1,
} skan_mode;

/* Pointer-location flags for skan_forward. */
#define SKAN_PTR_HOST 0u   /* inputs/outputs are host memory; copies happen inside */
#define SKAN_PTR_DEVICE 1u /* inputs/outputs are device memory on the head's GPU  */

/* ---- errors ---------------------------------------------------------- */

/* Last error of the calling thread.  msg may be NULL.  byte_offset/fault are
 * meaningful for SKAN_FORMAT_ERROR (FormatError::offset / ::fault). */
skan_status skan_last_error(char* msg, size_t msg_cap, uint64_t* byte_offset, int* fault);
const char* skan_status_name(skan_status s);
int skan_abi_version(void);

/* ---- planner ---------------------------------------------------------- */

/* index_bits, lutham.cpp:47-50 */
int skan_index_bits(uint32_t k);

/* plan_memory, lutham.cpp:52-86 — byte-exact sizes from headers alone;
 * per_layer may be NULL.  SKAN_PLAN_ERROR on degenerate dims / overflow. */
skan_status skan_plan_memory(const skan_layer_header* headers, int n_layers,
                             skan_layer_plan* per_layer, skan_memory_plan* totals);

/* ---- heads (holoquant::Model) ----------------------------------------- */

/* build_model (lutham.cpp:214) / build_dense_model (177) / upload of a
 * RuntimeLayer model; uploads the static resident form to `device`. */
skan_status skan_head_create(const skan_layer_desc* layers, int n_layers, int device,
                             skan_head** out);

/* deserialize (lutham.cpp:532-704): SKAN v1 bytes -> device head, with the
 * reference's fault kinds and byte offsets. */
skan_status skan_head_load(const uint8_t* bytes, size_t n_bytes, int device, skan_head** out);

/* load_model (lutham.cpp:715-724) */
skan_status skan_head_load_file(const char* path, int device, skan_head** out);

skan_status skan_head_destroy(skan_head* head);

/* Hot swap (no reference counterpart; the reference reloads a Model,
 * lutham.cpp:715-724): replace every table of `head` in place with the
 * layers described (validated like skan_head_create), keeping its device
 * allocation, plan and workspaces.  The new layers must match the old ones
 * in shape, grid size, K and format.  Forwards are excluded while the
 * tables change and forwards already enqueued on any stream are drained
 * first, so every forward reads either the old tables or the new; the copy
 * is ordered on `stream` (cudaStream_t) and complete on return. */
skan_status skan_head_swap(skan_head* head, const skan_layer_desc* layers, int n_layers, void* stream);
/* Hot swap from SKAN v1 bytes into the pre-planned slot: the same checks,
 * faults and byte offsets as skan_head_load (deserialize, lutham.cpp:532-704),
 * all raised before the resident tables are touched; the sections go to
 * HBM and are unpacked there.  The file must describe the same layer shapes,
 * grids, K and formats (ContractError otherwise). */
skan_status skan_head_swap_bytes(skan_head* head, const uint8_t* bytes, size_t n_bytes, void* stream);

/* Model::input_dim/output_dim/max_width (lutham.cpp:160-175), layer count
 * and per-layer headers (Model::header, lutham.cpp:154). */
int skan_head_num_layers(const skan_head* head);
int skan_head_input_dim(const skan_head* head);
int skan_head_output_dim(const skan_head* head);
int skan_head_max_width(const skan_head* head);
int skan_head_device(const skan_head* head);
skan_status skan_head_layer_header(const skan_head* head, int layer, skan_layer_header* out);
/* plan of the resident head (reference plan + device bytes) */
skan_status skan_head_plan(const skan_head* head, skan_layer_plan* per_layer,
                           skan_memory_plan* totals);
/* Total edges sum_l in_l*out_l (the interp_ops unit per sample). */
uint64_t skan_head_edges(const skan_head* head);

/* Pin the head's resident tables in L2 with a persisting access-policy
 * window on `stream` (cudaStream_t).  fraction in (0,1]; 0 clears it.  The
 * device's persisting carve-out is the sum over the heads that asked for it
 * (capped at cudaDevAttrMaxPersistingL2CacheSize); skan_forward_multi applies
 * each head's window on the side stream that runs it. */
skan_status skan_head_set_l2_persist(const skan_head* head, void* stream, float fraction);

/* ---- workspaces (holoquant::Workspace) --------------------------------- */

/* make_workspace (lutham.cpp:757-763).  All device scratch for batches up
 * to max_batch is allocated here; skan_forward allocates nothing. */
skan_status skan_workspace_create(const skan_head* head, int max_batch, skan_workspace** out);
skan_status skan_workspace_destroy(skan_workspace* ws);
/* Workspace::interp_ops (lutham.hpp:148): += batch * sum E per forward. */
uint64_t skan_workspace_interp_ops(const skan_workspace* ws);
int skan_workspace_max_batch(const skan_workspace* ws);
/* Workspace::width (lutham.hpp:150) */
int skan_workspace_width(const skan_workspace* ws);

/* ---- forward ----------------------------------------------------------- */

/* compressed_forward (lutham.cpp:819-850).  inputs: batch*input_dim f64
 * row-major; outputs: batch*output_dim f64.  n_inputs/n_outputs are the
 * span sizes the reference validates (ShapeError on mismatch); a workspace
 * built for a different head width or a smaller batch is ContractError.
 * ptr_flags: SKAN_PTR_HOST or SKAN_PTR_DEVICE.  stream: cudaStream_t (NULL =
 * the legacy default stream).  With SKAN_PTR_HOST the call is synchronous
 * and non-finite inputs (at any layer) return SKAN_VALUE_ERROR like
 * locate (kan.cpp:29).  batch == 0 does nothing. */
skan_status skan_forward(const skan_head* head, skan_workspace* ws, const double* inputs,
                         uint64_t n_inputs, int batch, double* outputs, uint64_t n_outputs,
                         int mode, unsigned ptr_flags, void* stream);

/* Device-pointer forward that does not synchronize: enqueue only.  The
 * non-finite check is deferred to skan_workspace_check. */
skan_status skan_forward_async(const skan_head* head, skan_workspace* ws, const double* d_inputs,
                               int batch, double* d_outputs, int mode, void* stream);
/* Synchronize ws's last stream and report a deferred SKAN_VALUE_ERROR. */
skan_status skan_workspace_check(skan_workspace* ws);

/* Multi-head forward: H heads with the same input width share one feature
 * batch (cfg5).  outputs[h] receives batch*output_dim(h) doubles.  All heads
 * and workspaces must live on the same device; device pointers only.  The
 * heads run concurrently on up to four library-owned side streams that
 * fork from and join back into `stream` (stream-ordered: the outputs are
 * ready when work enqueued on `stream` after this call runs); a deferred
 * non-finite input is reported by skan_workspace_check(wss[h]). */
skan_status skan_forward_multi(const skan_head* const* heads, skan_workspace* const* wss,
                               int n_heads, const double* d_inputs, int batch,
                               double* const* d_outputs, int mode, void* stream);

/* Number of kernels the last forward on ws enqueued (for launch counting). */
int skan_workspace_last_launches(const skan_workspace* ws);

/* Profiling hook (no reference counterpart): enqueue ONLY layer `layer`'s
 * gather kernel for `batch` samples on `stream`, reading the brackets the
 * previous forward on ws left behind (run one forward of the same batch and
 * mode first).  Lets a caller time the dominant kernel with CUDA events on
 * the stream it is launched on.  Output goes to ws scratch. */
skan_status skan_profile_gather(const skan_head* head, skan_workspace* ws, int layer, int batch,
                                int mode, void* stream);

/* Profiling hook: enqueue ONLY layer `layer`'s tensor-core GEMM kernel
 * (k_layer_gemm, no split reduction) for `batch` samples on `stream`,
 * reading the brackets the previous fast forward of the same batch on ws
 * left behind; ContractError if the layer does not use the GEMM at this
 * batch.  *issued_flops (optional) = the MMA work one launch issues. */
skan_status skan_profile_gemm(const skan_head* head, skan_workspace* ws, int layer, int batch, void* stream,
                              double* issued_flops);

/* Profiling hook: batch-1 forwards on ws record, per CTA of the persistent
 * head kernel, %globaltimer stamps (ns) at 16 fixed phase slots into the
 * device buffer d_stamps[grid][16] (NULL disables). */
skan_status skan_debug_b1_timeline(skan_workspace* ws, unsigned long long* d_stamps);
/* Grid size of the persistent batch-1 kernel for head (0 if not eligible). */
int skan_head_b1_grid(const skan_head* head);

/* Self-test of the tensor-core building blocks (no reference counterpart):
 * D[128][N] = A[128][K] * B[K][N] (row-major f32, device pointers) on
 * tcgen05 kind::tf32 with `passes` = 1 (plain tf32) or 3 (split-precision
 * 3xTF32).  N in [16, 256] step 16, K in [8, 64] step 8. */
/* passes == 1000: one kind::f16 pass with both operands rounded to fp16 in shared memory (M = 128) */
skan_status skan_debug_gemm_tf32(const float* d_a, const float* d_b, float* d_d, int n, int k, int passes,
                                 void* stream);

/* Phase timeline of the tensor-core layer GEMM: while d_stamps is set,
 * every layer-GEMM launch has CTA (0,0,0) write clock64 stamps into
 * d_stamps[2][64][8] (role 0: producer thread 0, role 1: the MMA thread;
 * per chunk < 64, phases as skan_gemm.cu documents).  NULL disables. */
skan_status skan_debug_gemm_timeline(unsigned long long* d_stamps);

/* Smallest batch the fast path routes to the tensor-core layer GEMM
 * (default 3; <= 0 restores it).  Returns the previous value.  A test and
 * tuning knob: the CUDA-core kernels serve the batches below it.  Set it
 * before creating workspaces (their scratch is sized for the launch plans
 * in force then); not thread-safe against concurrent forwards. */
int skan_debug_set_gemm_min_batch(int batch);

/* Whether a layer GEMM at batch <= 32 leaves its split partials to a
 * following one-tile-wide layer GEMM, which reduces them in its prologue
 * (default on; SKAN_GEMM_FUSE_REDUCE=0 turns it off).  Both routes sum the
 * same partials in the same f64 order, so outputs are bitwise equal.
 * Returns the previous setting.  A test knob; not thread-safe against
 * concurrent forwards. */
int skan_debug_set_fuse_reduce(int on);

/* ---- single-edge primitive (lutham.cpp:730-755) ----------------------- */

/* Batched pli_lookup over n independent (row, g, b, x) tuples on the GPU:
 * y[n] = g[n] * LinearInterp(codebook[rows[n]], x[n]) + b[n], with the
 * reference's operation order g*(c0*(1-t)+c1*t)+b (lutham.cpp:738).
 * Device pointers; codebook is K*G doubles. */
skan_status skan_pli_lookup(const double* d_codebook, int k, int grid_size, const int* d_rows,
                            const double* d_g, const double* d_b, const double* d_x,
                            double domain_lo, double domain_hi, int n, double* d_y,
                            void* stream);

/* ---- GSB-VQ nearest-row assignment (gsb.cpp:275-286) ------------------ */

/* indices[i] = the codebook row (of k, each `dim` doubles, row-major) at the
 * least squared distance from shapes[i] (n x dim, row-major), ties to the
 * lowest row: holoquant::assign_indices with nearest_row (gsb.cpp:62-73)
 * and dist2 (23-30), bit-identical (f64, dim order, no contraction).
 * dim in [1, 64]; k == 0 gives row 0 everywhere (as nearest_row does).
 * ptr_flags: SKAN_PTR_HOST (synchronous, copies inside) or SKAN_PTR_DEVICE
 * (device pointers, asynchronous on stream). */
skan_status skan_assign_indices(const double* shapes, uint64_t n, int dim, const double* codebook, int k,
                                uint32_t* indices, unsigned ptr_flags, void* stream);

/* ---- knot selection (kan.cpp:28-58) ------------------------------------ */

/* Bracket n inputs on the GPU: index[n], t[n], clamped[n] (device
 * pointers).  Bit-exact with holoquant::locate; SKAN_VALUE_ERROR if any x
 * is non-finite (outputs for finite x are still written). */
skan_status skan_locate(const double* d_x, int n, double domain_lo, double domain_hi,
                        int grid_size, int* d_index, double* d_t, uint8_t* d_clamped,
                        void* stream);

/* ---- SKAN v1 index bit-packing (lutham.cpp:88-137) ---------------------- */

/* GPU unpack of an LSB-first bit stream at `bits` per index (0..32). */
skan_status skan_unpack_indices(const uint8_t* d_bytes, size_t n_bytes, uint64_t count,
                                int bits, uint32_t* d_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SKAN_H */
