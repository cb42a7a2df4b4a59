/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference LUTHAM path.
 * See skan_oracle.h for the pinning story.  Each function cites the
 * reference function it restates (paths relative to /root/reference/proj).
 *
 * Must be compiled with -ffp-contract=off: every double expression below is
 * evaluated in the reference's operation order, one IEEE op at a time.
 */
#include "skan_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

static int is_int8(const oracle_layer* l) { return (l->flags & ORACLE_FLAG_INT8) != 0; }

/* lutham.cpp:47-50: bits = bit_width(k - 1), 0 for k <= 1 */
int oracle_index_bits(uint32_t k) {
    if (k <= 1) return 0;
    uint32_t v = k - 1;
    int bits = 0;
    while (v) {
        ++bits;
        v >>= 1;
    }
    return bits;
}

/* kan.cpp:21-26: endpoints are exact, interior nodes are lo + i*dx */
double oracle_node_position(double lo, double hi, int grid_size, int i) {
    if (i == 0) return lo;
    if (i == grid_size - 1) return hi;
    double dx = (hi - lo) / (double)(grid_size - 1);
    return lo + (double)i * dx;
}

/* kan.cpp:28-58: clamp, floor-divide, correct by one against the exact
 * node positions, then t in [0,1] (t = 1 exactly at or past the upper node). */
int oracle_locate(double lo, double hi, int grid_size, double x, int* index, double* t,
                  int* clamped) {
    if (!isfinite(x)) return ORACLE_VALUE;
    int cl = 0;
    if (x < lo) {
        x = lo;
        cl = 1;
    } else if (x > hi) {
        x = hi;
        cl = 1;
    }
    double dx = (hi - lo) / (double)(grid_size - 1);
    int i = (int)floor((x - lo) / dx);
    if (i < 0) i = 0;
    if (i > grid_size - 2) i = grid_size - 2;
    if (i < grid_size - 2 && x >= oracle_node_position(lo, hi, grid_size, i + 1))
        ++i;
    else if (i > 0 && x < oracle_node_position(lo, hi, grid_size, i))
        --i;
    double tt;
    if (x >= oracle_node_position(lo, hi, grid_size, i + 1)) {
        tt = 1.0;
    } else {
        tt = (x - oracle_node_position(lo, hi, grid_size, i)) / dx;
        if (tt < 0.0) tt = 0.0;
        if (tt > 1.0) tt = 1.0;
    }
    *index = i;
    *t = tt;
    if (clamped) *clamped = cl;
    return ORACLE_OK;
}

uint64_t oracle_locate_many(double lo, double hi, int grid_size, const double* x, uint64_t n,
                            int* index, double* t, uint8_t* clamped) {
    uint64_t bad = 0;
    for (uint64_t q = 0; q < n; ++q) {
        int i = 0, c = 0;
        double tt = 0.0;
        if (oracle_locate(lo, hi, grid_size, x[q], &i, &tt, &c)) ++bad;
        index[q] = i;
        t[q] = tt;
        if (clamped) clamped[q] = (uint8_t)c;
    }
    return bad;
}

/* quant.cpp:88-91 (kGainZeroCode = 127, quant.hpp:26) */
double oracle_dequantize_gain_code(int8_t code, double log_min, double log_step) {
    if (code == 127) return 0.0;
    return exp2(log_min + (double)code * log_step);
}

/* quant.cpp:40-42 */
double oracle_dequantize_linear_code(int8_t code, double scale) { return (double)code * scale; }

/* overflow-checked helpers, lutham.cpp:27-39 */
static int mul_ok(uint64_t a, uint64_t b, uint64_t* r) {
    if (a != 0 && b > UINT64_MAX / a) return 0;
    *r = a * b;
    return 1;
}
static int add_ok(uint64_t a, uint64_t b, uint64_t* r) {
    if (b > UINT64_MAX - a) return 0;
    *r = a + b;
    return 1;
}

/* lutham.cpp:52-86 */
int oracle_plan_memory(const oracle_layer* layers, int n, oracle_layer_plan* per_layer,
                       uint64_t* scratch, uint64_t* payload_total, uint64_t* working_set_total) {
    uint64_t payload = 0, working = 0, max_width = 0;
    for (int l = 0; l < n; ++l) {
        const oracle_layer* h = &layers[l];
        if (h->in_dim == 0 || h->out_dim == 0 || h->grid_size < 2) return ORACLE_PLAN;
        uint64_t e = (uint64_t)h->in_dim * h->out_dim;
        oracle_layer_plan lp;
        memset(&lp, 0, sizeof lp);
        if (h->k == 0) {
            uint64_t a;
            if (!mul_ok(e, h->grid_size, &a) || !mul_ok(a, 4, &lp.codebook_bytes)) return ORACLE_PLAN;
        } else {
            uint64_t w = is_int8(h) ? 1 : 4, a;
            if (!mul_ok(h->k, h->grid_size, &a) || !mul_ok(a, w, &lp.codebook_bytes)) return ORACLE_PLAN;
            int bits = oracle_index_bits(h->k);
            if (!mul_ok(e, (uint64_t)bits, &a) || !add_ok(a, 7, &a)) return ORACLE_PLAN;
            lp.index_bytes = a / 8;
            if (bits > 0 && !mul_ok(e, h->k <= 65536 ? 2 : 4, &lp.unpacked_index_bytes))
                return ORACLE_PLAN;
            if (!mul_ok(e, w, &lp.gain_bytes) || !mul_ok(e, w, &lp.bias_bytes)) return ORACLE_PLAN;
        }
        uint64_t pay = lp.codebook_bytes + lp.index_bytes + lp.gain_bytes + lp.bias_bytes;
        uint64_t ws = lp.codebook_bytes + lp.unpacked_index_bytes + lp.gain_bytes + lp.bias_bytes;
        if (!add_ok(payload, pay, &payload) || !add_ok(working, ws, &working)) return ORACLE_PLAN;
        if (h->in_dim > max_width) max_width = h->in_dim;
        if (h->out_dim > max_width) max_width = h->out_dim;
        if (per_layer) per_layer[l] = lp;
    }
    uint64_t s2, sc;
    if (!mul_ok(max_width, 2, &s2) || !mul_ok(s2, 8, &sc)) return ORACLE_PLAN;
    if (!add_ok(working, sc, &working)) return ORACLE_PLAN;
    if (scratch) *scratch = sc;
    if (payload_total) *payload_total = payload;
    if (working_set_total) *working_set_total = working;
    return ORACLE_OK;
}

/* lutham.cpp:88-112: LSB-first bit stream */
size_t oracle_pack_indices(const uint32_t* v, size_t count, int bits, uint8_t* out, size_t cap) {
    if (bits < 0 || bits > 32) return (size_t)-1;
    for (size_t n = 0; n < count; ++n)
        if (bits < 32 && (uint64_t)v[n] >= ((uint64_t)1 << bits)) return (size_t)-1;
    if (bits == 0) return 0;
    size_t need = (count * (size_t)bits + 7) / 8;
    if (need > cap) return (size_t)-1;
    uint64_t acc = 0;
    int filled = 0;
    size_t pos = 0;
    for (size_t n = 0; n < count; ++n) {
        acc |= (uint64_t)v[n] << filled;
        filled += bits;
        for (; filled >= 8; filled -= 8, acc >>= 8) out[pos++] = (uint8_t)(acc & 0xFF);
    }
    if (filled > 0) out[pos++] = (uint8_t)(acc & 0xFF);
    return pos;
}

/* lutham.cpp:114-137 */
int oracle_unpack_indices(const uint8_t* bytes, size_t nbytes, uint64_t count, int bits,
                          uint32_t* out) {
    if (bits < 0 || bits > 32) return ORACLE_CONTRACT;
    if (bits == 0) {
        memset(out, 0, count * sizeof *out);
        return ORACLE_OK;
    }
    if (nbytes < (count * (uint64_t)bits + 7) / 8) return ORACLE_CONTRACT;
    uint64_t mask = ((uint64_t)1 << bits) - 1, acc = 0;
    int filled = 0;
    size_t pos = 0;
    for (uint64_t n = 0; n < count; ++n) {
        while (filled < bits) {
            acc |= (uint64_t)bytes[pos++] << filled;
            filled += 8;
        }
        out[n] = (uint32_t)(acc & mask);
        acc >>= bits;
        filled -= bits;
    }
    return ORACLE_OK;
}

static uint32_t edge_index(const oracle_layer* l, uint64_t e) {
    if (l->idx16) return l->idx16[e];
    if (l->idx32) return l->idx32[e];
    return 0; /* lutham.hpp:102-106 */
}

/* lutham.cpp:770-815 */
/* forward_layer with an optional per-output L1 accumulator: l1[j] += |term_ij|
 * (test tolerance scale only; y is computed exactly as without it). */
static int forward_layer_l1(const oracle_layer* l, const double* x, double* y, uint64_t* ops, double* l1) {
    const int in = (int)l->in_dim, out = (int)l->out_dim, G = (int)l->grid_size;
    for (int j = 0; j < out; ++j) y[j] = 0.0;
    if (l1)
        for (int j = 0; j < out; ++j) l1[j] = 0.0;
    for (int i = 0; i < in; ++i) {
        int idx, cl;
        double t;
        if (oracle_locate(l->domain_lo, l->domain_hi, G, x[i], &idx, &t, &cl)) return ORACLE_VALUE;
        const double w0 = 1.0 - t;
        const uint64_t e0 = (uint64_t)i * (uint64_t)out;
        if (l->k == 0) { /* dense branch 778-791 */
            const float* base = l->table_f32 + e0 * (uint64_t)G + (uint64_t)idx;
            for (int j = 0; j < out; ++j, base += G) {
                const double term = (double)base[0] * w0 + (double)base[1] * t;
                y[j] += term;
                if (l1) l1[j] += fabs(term);
            }
        } else { /* compressed branch 793-814 */
            for (int j = 0; j < out; ++j) {
                const uint64_t e = e0 + (uint64_t)j;
                double g, b, c0, c1;
                const uint64_t row = (uint64_t)edge_index(l, e) * (uint64_t)G + (uint64_t)idx;
                if (is_int8(l)) {
                    g = oracle_dequantize_gain_code(l->gain_codes[e], l->gain_log_min,
                                                    l->gain_log_step);
                    b = (double)l->bias_codes[e] * l->bias_scale;
                    c0 = (double)l->table_i8[row] * l->codebook_scale;
                    c1 = (double)l->table_i8[row + 1] * l->codebook_scale;
                } else {
                    g = (double)l->gains_f32[e];
                    b = (double)l->biases_f32[e];
                    c0 = (double)l->table_f32[row];
                    c1 = (double)l->table_f32[row + 1];
                }
                const double term = (g * c0 + b) * w0 + (g * c1 + b) * t;
                y[j] += term;
                if (l1) l1[j] += fabs(term);
            }
        }
        *ops += (uint64_t)out;
    }
    return ORACLE_OK;
}

/* lutham.cpp:770-815 */
int oracle_forward_layer(const oracle_layer* l, const double* x, double* y, uint64_t* ops) {
    return forward_layer_l1(l, x, y, ops, NULL);
}

static int max_width(const oracle_layer* layers, int n) {
    uint32_t w = 0;
    for (int l = 0; l < n; ++l) {
        if (layers[l].in_dim > w) w = layers[l].in_dim;
        if (layers[l].out_dim > w) w = layers[l].out_dim;
    }
    return (int)w;
}

/* lutham.cpp:819-850.  scale (optional): per output max(|y|, sum_i |term_ij|)
 * of the last layer (the fast mode's L1 tolerance scale, tests only);
 * scratch then holds 3*max_width doubles. */
static int forward_impl(const oracle_layer* layers, int n, const double* inputs, int batch,
                        double* outputs, double* scratch, uint64_t* interp_ops, double* scale) {
    if (n <= 0) return ORACLE_SHAPE;
    if (batch < 0) return ORACLE_SHAPE;
    const int width = max_width(layers, n);
    const size_t in = layers[0].in_dim, out = layers[n - 1].out_dim;
    uint64_t ops = 0;
    for (int s = 0; s < batch; ++s) {
        double* cur = scratch;
        double* nxt = scratch + width;
        double* l1 = scale ? scratch + 2 * (size_t)width : NULL;
        memcpy(cur, inputs + (size_t)s * in, in * sizeof(double));
        for (int l = 0; l < n; ++l) {
            int rc = forward_layer_l1(&layers[l], cur, nxt, &ops, l == n - 1 ? l1 : NULL);
            if (rc) return rc;
            double* tmp = cur;
            cur = nxt;
            nxt = tmp;
        }
        memcpy(outputs + (size_t)s * out, cur, out * sizeof(double));
        if (scale)
            for (size_t j = 0; j < out; ++j) scale[(size_t)s * out + j] = fabs(cur[j]) > l1[j] ? fabs(cur[j]) : l1[j];
    }
    if (interp_ops) *interp_ops += ops;
    return ORACLE_OK;
}

int oracle_compressed_forward(const oracle_layer* layers, int n, const double* inputs, int batch,
                              double* outputs, double* scratch, uint64_t* interp_ops) {
    return forward_impl(layers, n, inputs, batch, outputs, scratch, interp_ops, NULL);
}

typedef struct {
    const oracle_layer* layers;
    int n, s0, s1, rc;
    const double* inputs;
    double* outputs;
    double* scale;
    uint64_t ops;
} mt_job;

static void* mt_run(void* p) {
    mt_job* j = (mt_job*)p;
    const int width = max_width(j->layers, j->n);
    double* scratch = (double*)malloc(sizeof(double) * 3 * (size_t)(width > 0 ? width : 1));
    const size_t in = j->layers[0].in_dim, out = j->layers[j->n - 1].out_dim;
    j->ops = 0;
    j->rc = forward_impl(j->layers, j->n, j->inputs + (size_t)j->s0 * in, j->s1 - j->s0,
                         j->outputs + (size_t)j->s0 * out, scratch, &j->ops,
                         j->scale ? j->scale + (size_t)j->s0 * out : NULL);
    free(scratch);
    return NULL;
}

static int forward_mt(const oracle_layer* layers, int n, const double* inputs, int batch,
                      double* outputs, int threads, uint64_t* interp_ops, double* scale) {
    if (n <= 0 || batch < 0) return ORACLE_SHAPE;
    if (threads < 1) threads = 1;
    if (threads > batch) threads = batch > 0 ? batch : 1;
    mt_job* jobs = (mt_job*)calloc((size_t)threads, sizeof(mt_job));
    pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    for (int t = 0; t < threads; ++t) {
        jobs[t].layers = layers;
        jobs[t].n = n;
        jobs[t].s0 = (int)((long long)batch * t / threads);
        jobs[t].s1 = (int)((long long)batch * (t + 1) / threads);
        jobs[t].inputs = inputs;
        jobs[t].outputs = outputs;
        jobs[t].scale = scale;
        pthread_create(&tids[t], NULL, mt_run, &jobs[t]);
    }
    int rc = ORACLE_OK;
    for (int t = 0; t < threads; ++t) {
        pthread_join(tids[t], NULL);
        if (jobs[t].rc && !rc) rc = jobs[t].rc;
        if (interp_ops) *interp_ops += jobs[t].ops;
    }
    free(jobs);
    free(tids);
    return rc;
}

int oracle_compressed_forward_mt(const oracle_layer* layers, int n, const double* inputs,
                                 int batch, double* outputs, int threads, uint64_t* interp_ops) {
    return forward_mt(layers, n, inputs, batch, outputs, threads, interp_ops, NULL);
}

int oracle_forward_l1_mt(const oracle_layer* layers, int n, const double* inputs, int batch,
                         double* outputs, double* scale, int threads) {
    return forward_mt(layers, n, inputs, batch, outputs, threads, NULL, scale);
}

/* gsb.cpp:23-30 (dist2), 62-73 (nearest_row), 275-286 (assign_indices). */
void oracle_assign_indices(const double* shapes, uint64_t n, int dim, const double* entries, int k,
                           uint32_t* out) {
    for (uint64_t i = 0; i < n; ++i) {
        const double* a = shapes + i * (uint64_t)dim;
        int best = 0;
        double best_d = INFINITY;
        for (int r = 0; r < k; ++r) {
            const double* b = entries + (uint64_t)r * (uint64_t)dim;
            double s = 0.0;
            for (int c = 0; c < dim; ++c) {
                const double d = a[c] - b[c];
                s += d * d;
            }
            if (s < best_d) {
                best_d = s;
                best = r;
            }
        }
        out[i] = (uint32_t)best;
    }
}
