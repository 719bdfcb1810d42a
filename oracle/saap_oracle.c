/*
 * TEST INFRASTRUCTURE ONLY — the parity checker, never the product.
 *
 * A plain-C restatement of the reference SAAP hot path (arXiv 2502.08246 CPU
 * reproduction, /root/reference/proj/core) used by tests/, smoke() and the
 * bench's cpu_baseline leg to check the CUDA path.  Every function keeps the
 * reference's fp64 operation order and rounding points, so
 * on identical inputs it is bit-identical to the reference; that is pinned by
 * tests/test_oracle.py against tests/golden/ fixtures produced by the
 * reference itself and, when oracle/_ref is built, against the live
 * reference.  Build with -ffp-contract=off and no -march so no FMA is formed
 * (the reference's objects contain only mulsd/addsd).
 *
 * Error convention: functions return 0 on success and a negative code on the
 * conditions where the reference throws std::invalid_argument.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EXPORT __attribute__((visibility("default")))

/* tensor.cpp:46-52 — sequential fp64 mul+add over f32 inputs. */
static double dot_f(const float* a, const float* b, size_t n) {
    double s = 0.0;
    for (size_t k = 0; k < n; ++k) s += (double)a[k] * (double)b[k];
    return s;
}

static double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */

/* partition.cpp:38-48, 181-198: strict '>' keeps ties on the lowest id. */
EXPORT int oracle_assign_keys(const float* keys, uint64_t n, uint64_t d, const float* cent,
                              uint64_t C, uint32_t* out) {
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t best = 0;
        double best_s = -INFINITY;
        for (uint64_t c = 0; c < C; ++c) {
            double s = dot_f(keys + i * d, cent + c * d, d);
            if (s > best_s) {
                best_s = s;
                best = (uint32_t)c;
            }
        }
        out[i] = best;
    }
    return 0;
}

/* partition.cpp:200-223: counting sort; forward scatter keeps ids ascending. */
EXPORT int oracle_build_ivf(const uint32_t* a, uint64_t n, uint64_t C, uint64_t* off,
                            uint64_t* idx) {
    memset(off, 0, (C + 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) {
        if (a[i] >= C) return -1;
        off[a[i] + 1]++;
    }
    for (uint64_t c = 0; c < C; ++c) off[c + 1] += off[c];
    uint64_t* cur = (uint64_t*)malloc((C ? C : 1) * sizeof(uint64_t));
    memcpy(cur, off, C * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) idx[cur[a[i]]++] = i;
    free(cur);
    return 0;
}

/* ---- top-l by (score desc, id asc): attention.cpp:259-271, qmodel.cpp:500-509.
 * The comparator is a total order, so a full sort has the partial_sort prefix. */
static const double* g_sort_score;
static int cmp_score(const void* pa, const void* pb) {
    uint32_t a = *(const uint32_t*)pa, b = *(const uint32_t*)pb;
    double sa = g_sort_score[a], sb = g_sort_score[b];
    if (sa != sb) return sa > sb ? -1 : 1;
    return a < b ? -1 : (a > b ? 1 : 0);
}
static void top_l(const double* score, uint64_t C, uint64_t l, uint32_t* out) {
    uint32_t* ids = (uint32_t*)malloc(C * sizeof(uint32_t));
    for (uint64_t c = 0; c < C; ++c) ids[c] = (uint32_t)c;
    g_sort_score = score;
    qsort(ids, C, sizeof(uint32_t), cmp_score);
    memcpy(out, ids, l * sizeof(uint32_t));
    free(ids);
}

/* attention.cpp:275-306: pooled = sum of the group rows (fp64, rows in order);
 * score_c = sum_j pooled_j * c_cj with the multiply rounded before the add. */
EXPORT int oracle_centroid_scores(const float* cent, uint64_t C, uint64_t d, const float* q,
                                  uint64_t G, double* score) {
    double* pooled = (double*)calloc(d, sizeof(double));
    for (uint64_t i = 0; i < G; ++i)
        for (uint64_t j = 0; j < d; ++j) pooled[j] += (double)q[i * d + j];
    for (uint64_t c = 0; c < C; ++c) {
        double s = 0.0;
        for (uint64_t j = 0; j < d; ++j) s += pooled[j] * (double)cent[c * d + j];
        score[c] = s;
    }
    free(pooled);
    return 0;
}

EXPORT int oracle_centroid_select(const float* cent, uint64_t C, uint64_t d, const float* q,
                                  uint64_t G, uint64_t l, uint32_t* out) {
    if (l == 0) return 0;
    if (l > C) return -1;
    double* score = (double*)malloc(C * sizeof(double));
    oracle_centroid_scores(cent, C, d, q, G, score);
    top_l(score, C, l, out);
    free(score);
    return 0;
}

/* qmodel.cpp:147-225 (eval mode) + 485-511: fp64 MLP, softmax, summed over
 * the group rows.  mm() skips zero inputs (qmodel.cpp:41-43) — harmless, the
 * accumulator starts at +0 — and is kept for fidelity. */
EXPORT int oracle_qmodel_scores(uint64_t d, uint64_t h, uint64_t C, const double* w1,
                                const double* b1, const double* gamma, const double* beta,
                                const double* mean, const double* var, const double* w2,
                                const double* b2, const float* q, uint64_t G, double* score) {
    double* z = (double*)malloc(h * sizeof(double));
    double* inv_std = (double*)malloc(h * sizeof(double));
    double* p = (double*)malloc(C * sizeof(double));
    for (uint64_t j = 0; j < h; ++j) inv_std[j] = 1.0 / sqrt(var[j] + 1e-5);
    for (uint64_t c = 0; c < C; ++c) score[c] = 0.0;
    for (uint64_t i = 0; i < G; ++i) {
        for (uint64_t j = 0; j < h; ++j) z[j] = 0.0;
        for (uint64_t k = 0; k < d; ++k) {
            double av = (double)q[i * d + k];
            if (av == 0.0) continue;
            for (uint64_t j = 0; j < h; ++j) z[j] += av * w1[k * h + j];
        }
        for (uint64_t j = 0; j < h; ++j) {
            z[j] += b1[j];
            double xh = (z[j] - mean[j]) * inv_std[j];
            double y = gamma[j] * xh + beta[j];
            z[j] = y > 0.0 ? y : 0.0; /* r */
        }
        for (uint64_t c = 0; c < C; ++c) p[c] = 0.0;
        for (uint64_t k = 0; k < h; ++k) {
            double av = z[k];
            if (av == 0.0) continue;
            for (uint64_t c = 0; c < C; ++c) p[c] += av * w2[k * C + c];
        }
        double mx = -INFINITY;
        for (uint64_t c = 0; c < C; ++c) {
            p[c] += b2[c];
            mx = dmax(mx, p[c]);
        }
        double total = 0.0;
        for (uint64_t c = 0; c < C; ++c) {
            p[c] = exp(p[c] - mx);
            total += p[c];
        }
        double inv = 1.0 / total;
        for (uint64_t c = 0; c < C; ++c) score[c] += p[c] * inv;
    }
    free(z);
    free(inv_std);
    free(p);
    return 0;
}

EXPORT int oracle_qmodel_select(uint64_t d, uint64_t h, uint64_t C, const double* w1,
                                const double* b1, const double* gamma, const double* beta,
                                const double* mean, const double* var, const double* w2,
                                const double* b2, const float* q, uint64_t G, uint64_t l,
                                uint32_t* out) {
    if (l < 1 || l > C) return -1;
    double* score = (double*)malloc(C * sizeof(double));
    oracle_qmodel_scores(d, h, C, w1, b1, gamma, beta, mean, var, w2, b2, q, G, score);
    top_l(score, C, l, out);
    free(score);
    return 0;
}

/* ---- online-softmax partials (Alg. 1/2): attention.cpp:34-161 ---- */
typedef struct {
    uint64_t G, dv;
    double* out; /* G x dv */
    double* sumexp;
    double* runmax;
} Acc;

static Acc acc_new(uint64_t G, uint64_t dv) {
    Acc a;
    a.G = G;
    a.dv = dv;
    a.out = (double*)calloc(G * dv, sizeof(double));
    a.sumexp = (double*)calloc(G, sizeof(double));
    a.runmax = (double*)malloc(G * sizeof(double));
    for (uint64_t h = 0; h < G; ++h) a.runmax[h] = -INFINITY;
    return a;
}
static void acc_free(Acc* a) {
    free(a->out);
    free(a->sumexp);
    free(a->runmax);
}

/* absorb_impl, attention.cpp:34-78: head-outer; scores dot*scale. */
static void absorb(Acc* acc, const float* q, uint64_t d, const float* K, const float* V,
                   const uint64_t* ids, uint64_t count, double* s) {
    if (count == 0) return;
    const double scale = 1.0 / sqrt((double)d);
    for (uint64_t h = 0; h < acc->G; ++h) {
        double rowmax = -INFINITY;
        for (uint64_t j = 0; j < count; ++j) {
            s[j] = dot_f(q + h * d, K + ids[j] * d, d) * scale;
            rowmax = dmax(rowmax, s[j]);
        }
        const double m_new = dmax(acc->runmax[h], rowmax);
        const double rescale = exp(acc->runmax[h] - m_new);
        double* out = acc->out + h * acc->dv;
        for (uint64_t t = 0; t < acc->dv; ++t) out[t] *= rescale;
        acc->sumexp[h] *= rescale;
        for (uint64_t j = 0; j < count; ++j) {
            const double w = exp(s[j] - m_new);
            const float* v = V + ids[j] * acc->dv;
            for (uint64_t t = 0; t < acc->dv; ++t) out[t] += w * (double)v[t];
            acc->sumexp[h] += w;
        }
        acc->runmax[h] = m_new;
    }
}

/* merge_into, attention.cpp:102-128. */
static void merge_into(Acc* acc, const Acc* part) {
    for (uint64_t h = 0; h < acc->G; ++h) {
        if (part->sumexp[h] == 0.0) continue;
        double* dst = acc->out + h * acc->dv;
        const double* src = part->out + h * acc->dv;
        if (acc->sumexp[h] == 0.0) {
            memcpy(dst, src, acc->dv * sizeof(double));
            acc->sumexp[h] = part->sumexp[h];
            acc->runmax[h] = part->runmax[h];
            continue;
        }
        const double m = dmax(acc->runmax[h], part->runmax[h]);
        const double a_acc = exp(acc->runmax[h] - m);
        const double a_part = exp(part->runmax[h] - m);
        for (uint64_t j = 0; j < acc->dv; ++j) dst[j] = dst[j] * a_acc + src[j] * a_part;
        acc->sumexp[h] = acc->sumexp[h] * a_acc + part->sumexp[h] * a_part;
        acc->runmax[h] = m;
    }
}

/* pattn_finalize, attention.cpp:141-161. */
static int finalize(const Acc* acc, float* out) {
    int empty = 0;
    for (uint64_t h = 0; h < acc->G; ++h) {
        float* dst = out + h * acc->dv;
        if (acc->sumexp[h] == 0.0) {
            empty = 1;
            for (uint64_t j = 0; j < acc->dv; ++j) dst[j] = 0.0f;
            continue;
        }
        const double inv = 1.0 / acc->sumexp[h];
        for (uint64_t j = 0; j < acc->dv; ++j) dst[j] = (float)(acc->out[h * acc->dv + j] * inv);
    }
    return empty;
}

/* full_attention, attention.cpp:163-195 (score = scale*dot, out = acc/denom). */
EXPORT int oracle_full_attention(const float* q, uint64_t G, const float* K, const float* V,
                                 uint64_t n, uint64_t d, float* out) {
    if (n == 0) return -1;
    const double scale = 1.0 / sqrt((double)d);
    double* s = (double*)malloc(n * sizeof(double));
    double* acc = (double*)malloc(d * sizeof(double));
    for (uint64_t h = 0; h < G; ++h) {
        double mx = -INFINITY;
        for (uint64_t k = 0; k < n; ++k) {
            s[k] = scale * dot_f(q + h * d, K + k * d, d);
            mx = dmax(mx, s[k]);
        }
        for (uint64_t j = 0; j < d; ++j) acc[j] = 0.0;
        double denom = 0.0;
        for (uint64_t k = 0; k < n; ++k) {
            const double w = exp(s[k] - mx);
            denom += w;
            for (uint64_t j = 0; j < d; ++j) acc[j] += w * (double)V[k * d + j];
        }
        for (uint64_t j = 0; j < d; ++j) out[h * d + j] = (float)(acc[j] / denom);
    }
    free(s);
    free(acc);
    return 0;
}

/* sparse_attention, attention.cpp:317-376, with the router's output passed in
 * (`selected`, score order) so routing and attention are checked separately.
 * Returns -1 for probes > C, -2 for block_size < 1. */
EXPORT int oracle_sparse_attention(const float* q, uint64_t G, uint64_t d, const float* K,
                                   const float* V, uint64_t n, uint64_t sink, const uint64_t* off,
                                   const uint64_t* idx, uint64_t C, const uint32_t* selected,
                                   uint64_t probes, uint64_t block_size, uint64_t recent,
                                   float* out, uint64_t* keys_scored, uint64_t* max_visited,
                                   int* empty) {
    if (probes > C) return -1;
    if (block_size < 1) return -2;
    *max_visited = 0;
    if (n <= sink + recent) {
        oracle_full_attention(q, G, K, V, n, d, out);
        *keys_scored = n;
        *empty = 0;
        return 0;
    }
    const uint64_t rb = n - recent;
    double* s = (double*)malloc((n > block_size ? n : block_size) * sizeof(double));
    uint64_t* ids = (uint64_t*)malloc((n > block_size ? n : block_size) * sizeof(uint64_t));
    Acc acc = acc_new(G, d);
    for (uint64_t i = 0; i < sink; ++i) ids[i] = i;
    absorb(&acc, q, d, K, V, ids, sink, s);
    for (uint64_t i = rb; i < n; ++i) ids[i - rb] = i;
    absorb(&acc, q, d, K, V, ids, n - rb, s);
    uint64_t scored = sink + (n - rb);
    for (uint64_t b = 0; b < probes; ++b) {
        const uint32_t c = selected[b];
        const uint64_t lo = off[c], len = off[c + 1] - off[c];
        if (len > *max_visited) *max_visited = len;
        Acc part = acc_new(G, d);
        for (uint64_t pos = 0; pos < len; pos += block_size) {
            const uint64_t stop = pos + block_size < len ? pos + block_size : len;
            uint64_t cnt = 0;
            for (uint64_t j = pos; j < stop; ++j) {
                const uint64_t gid = idx[lo + j] + sink;
                if (gid < rb) ids[cnt++] = gid;
            }
            absorb(&part, q, d, K, V, ids, cnt, s);
            scored += cnt;
        }
        merge_into(&acc, &part);
        acc_free(&part);
    }
    *empty = finalize(&acc, out);
    *keys_scored = scored;
    acc_free(&acc);
    free(s);
    free(ids);
    return 0;
}

/* attention_mass_coverage, attention.cpp:427-462. */
EXPORT int oracle_coverage(const float* q, uint64_t G, uint64_t d, const float* K, uint64_t n,
                           uint64_t sink, const uint32_t* assignment, uint64_t C,
                           const uint32_t* selected, uint64_t l, uint64_t recent, double* out) {
    uint64_t lo = sink < n ? sink : n;
    uint64_t hi = n > recent ? n - recent : 0;
    if (hi < lo) hi = lo;
    if (lo == hi) {
        *out = 1.0;
        return 0;
    }
    char* picked = (char*)calloc(C, 1);
    for (uint64_t i = 0; i < l; ++i) {
        if (selected[i] >= C) {
            free(picked);
            return -1;
        }
        picked[selected[i]] = 1;
    }
    const double scale = 1.0 / sqrt((double)d);
    double* s = (double*)malloc((hi - lo) * sizeof(double));
    double total = 0.0;
    for (uint64_t h = 0; h < G; ++h) {
        double mx = -INFINITY;
        for (uint64_t id = lo; id < hi; ++id) {
            s[id - lo] = dot_f(q + h * d, K + id * d, d) * scale;
            mx = dmax(mx, s[id - lo]);
        }
        double denom = 0.0, hit = 0.0;
        for (uint64_t id = lo; id < hi; ++id) {
            const double w = exp(s[id - lo] - mx);
            denom += w;
            if (picked[assignment[id - sink]]) hit += w;
        }
        total += hit / denom;
    }
    *out = total / (double)G;
    free(picked);
    free(s);
    return 0;
}

/* mse, attention.cpp:385-399. */
EXPORT int oracle_mse(const float* a, const float* b, uint64_t count, double* out) {
    if (count == 0) return -1;
    double total = 0.0;
    for (uint64_t i = 0; i < count; ++i) {
        const double dd = (double)a[i] - (double)b[i];
        total += dd * dd;
    }
    *out = total / (double)count;
    return 0;
}

/* rope.cpp:20-41 with sign -1 (rope_remove_block, rope.cpp:87-90). */
EXPORT int oracle_rope_remove(const float* x, uint64_t rows, uint64_t d,
                              const uint64_t* positions, double base, float* out) {
    if (d == 0 || d % 2) return -1;
    const double inv_dim = 1.0 / (double)d;
    double* th = (double*)malloc(d / 2 * sizeof(double));
    for (uint64_t j = 0; j < d / 2; ++j) th[j] = pow(base, -2.0 * (double)j * inv_dim);
    for (uint64_t i = 0; i < rows; ++i) {
        const double p = (double)positions[i];
        for (uint64_t j = 0; j < d / 2; ++j) {
            const double angle = -1.0 * p * th[j];
            const double c = cos(angle), s = sin(angle);
            const double x0 = x[i * d + 2 * j], x1 = x[i * d + 2 * j + 1];
            out[i * d + 2 * j] = (float)(x0 * c - x1 * s);
            out[i * d + 2 * j + 1] = (float)(x0 * s + x1 * c);
        }
    }
    free(th);
    return 0;
}
