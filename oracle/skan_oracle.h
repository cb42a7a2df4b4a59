/*
 * TEST INFRASTRUCTURE ONLY — not part of the product.
 *
 * Plain-C restatement of the reference LUTHAM CPU forward path
 * (holoquant, /root/reference/proj).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load this; the product library
 * (paper_2512_15742_b200/libskan.so) never links or calls it.
 *
 * Parity pinning: this restatement is checked bit-for-bit against the
 * reference itself (oracle/_ref/libholoquant_ref.so, compiled from the
 * reference sources by oracle/Makefile) and against the golden vectors of
 * the reference's own doctest suites (tests/golden/reference_kats.json).
 * Build flags: -O2 -ffp-contract=off (contraction
 * changes the reference's bits).
 */
#ifndef SKAN_ORACLE_H
#define SKAN_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORACLE_OK = 0, ORACLE_SHAPE = 1, ORACLE_VALUE = 2, ORACLE_CONTRACT = 3, ORACLE_PLAN = 5 };

#define ORACLE_FLAG_INT8 1u

/* Mirrors holoquant::LayerHeader (lutham.hpp:30-49) plus the RuntimeLayer
 * tables (lutham.hpp:91-109).  Exactly one of table_f32/table_i8 is set;
 * idx16 when 1 < K <= 65536, idx32 when K > 65536, neither when K == 1. */
typedef struct {
    uint32_t in_dim, out_dim, grid_size, k; /* k == 0: dense layer */
    double domain_lo, domain_hi;
    uint32_t flags;
    double codebook_scale, gain_log_min, gain_log_step, bias_scale;
    const float* table_f32;  /* K*G codebook, or E*G dense coefficients */
    const int8_t* table_i8;  /* K*G int8 codebook codes */
    const uint16_t* idx16;
    const uint32_t* idx32;
    const float* gains_f32;
    const float* biases_f32;
    const int8_t* gain_codes;
    const int8_t* bias_codes;
} oracle_layer;

typedef struct {
    uint64_t codebook_bytes, index_bytes, unpacked_index_bytes, gain_bytes, bias_bytes;
} oracle_layer_plan;

/* lutham.cpp:47-50 */
int oracle_index_bits(uint32_t k);
/* kan.cpp:21-26 */
double oracle_node_position(double lo, double hi, int grid_size, int i);
/* kan.cpp:28-58; returns ORACLE_VALUE for non-finite x */
int oracle_locate(double lo, double hi, int grid_size, double x, int* index, double* t,
                  int* clamped);
/* locate over an array (convenience for bulk bit-exactness checks); returns
 * the number of non-finite inputs (their idx/t are left at 0). */
uint64_t oracle_locate_many(double lo, double hi, int grid_size, const double* x, uint64_t n,
                            int* index, double* t, uint8_t* clamped);
/* quant.cpp:88-91 */
double oracle_dequantize_gain_code(int8_t code, double log_min, double log_step);
/* quant.cpp:40-42 */
double oracle_dequantize_linear_code(int8_t code, double scale);
/* lutham.cpp:52-86: per-layer plan + totals; ORACLE_PLAN on degenerate dims / overflow */
int oracle_plan_memory(const oracle_layer* layers, int n, oracle_layer_plan* per_layer,
                       uint64_t* scratch, uint64_t* payload_total, uint64_t* working_set_total);
/* lutham.cpp:88-112; returns bytes written, or (size_t)-1 on contract error */
size_t oracle_pack_indices(const uint32_t* v, size_t count, int bits, uint8_t* out, size_t cap);
/* lutham.cpp:114-137 */
int oracle_unpack_indices(const uint8_t* bytes, size_t nbytes, uint64_t count, int bits,
                          uint32_t* out);
/* lutham.cpp:770-815, one layer one sample */
int oracle_forward_layer(const oracle_layer* layer, const double* x, double* y, uint64_t* ops);
/* lutham.cpp:819-850; scratch must hold 2*max_width doubles */
int oracle_compressed_forward(const oracle_layer* layers, int n, const double* inputs, int batch,
                              double* outputs, double* scratch, uint64_t* interp_ops);
/* Same, with the batch split over `threads` std-C threads, one private
 * scratch per stream (SPEC.md:536 concurrency model).  Used for the CPU
 * baseline; results are identical to the single-stream call. */
int oracle_compressed_forward_mt(const oracle_layer* layers, int n, const double* inputs,
                                 int batch, double* outputs, int threads, uint64_t* interp_ops);

/* The forward above plus, per output of the last layer, the fast mode's
 * tolerance scale max(|y|, sum_i |term_ij|) with term_ij the reference's
 * per-edge interpolation (lutham.cpp:791/810).  Tests only. */
int oracle_forward_l1_mt(const oracle_layer* layers, int n, const double* inputs, int batch,
                         double* outputs, double* scale, int threads);

/* assign_indices, gsb.cpp:275-286 with nearest_row 62-73 and dist2 23-30:
 * per shape (n x dim row-major) the codebook row (k x dim) of least
 * squared distance, accumulated in dim order as s += (a-b)*(a-b) (no
 * contraction); strict <, so ties keep the lowest row. */
void oracle_assign_indices(const double* shapes, uint64_t n, int dim, const double* entries, int k,
                           uint32_t* out);

#ifdef __cplusplus
}
#endif
#endif
