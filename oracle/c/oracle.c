/*
 * TEST INFRASTRUCTURE ONLY -- the parity oracle, never the product.
 *
 * Plain-C restatement of the reference (linksim 0.1.0, /root/reference/pkg)
 * hot-path arithmetic that lives in numpy's compiled code or is too slow in
 * pure Python for the parity tests:
 *
 *   * numpy Philox4x64-10 bit generator, as keyed by RngStream
 *     (core.py:37-39; numpy 2.3.5 `Philox`);
 *   * Generator.integers(0, 2, uint8) byte-buffered Lemire draw used by
 *     binary_source (core.py:47-54);
 *   * bp_decode (ldpc.py:86-172) with the reference's exact mixed
 *     f32/f64 arithmetic: f64 check-to-variable messages after the first
 *     iteration, numpy `add.reduceat` summation order (x0 + pairwise-sum of
 *     the rest, pairwise_sum starting from -0.0, 8-way unrolled for 8..128
 *     terms), f32 rounding of the posterior each iteration, clip to +-40,
 *     per-row early stop.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load
 * this library (via oracle/linksim_oracle.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* Philox4x64-10 (numpy/random/src/philox/philox.h restated)           */
/* ------------------------------------------------------------------ */
#define PHILOX_M0 0xD2E7470EE14C6C93ULL
#define PHILOX_M1 0xCA5A826395121157ULL
#define PHILOX_W0 0x9E3779B97F4A7C15ULL
#define PHILOX_W1 0xBB67AE8584CAA73BULL

static inline uint64_t mulhilo64(uint64_t a, uint64_t b, uint64_t *hi) {
    __uint128_t p = (__uint128_t)a * (__uint128_t)b;
    *hi = (uint64_t)(p >> 64);
    return (uint64_t)p;
}

static void philox4x64_10(const uint64_t ctr_in[4], const uint64_t key_in[2], uint64_t out[4]) {
    uint64_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint64_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round) { k0 += PHILOX_W0; k1 += PHILOX_W1; }
        uint64_t hi0, hi1;
        uint64_t lo0 = mulhilo64(PHILOX_M0, c0, &hi0);
        uint64_t lo1 = mulhilo64(PHILOX_M1, c2, &hi1);
        uint64_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Raw uint64 stream of RngStream(seed, stream_id): numpy's Philox keeps the
 * counter at 0 and increments it *before* producing each 4-word block, so
 * word w comes from counter (w/4 + 1), lane w%4. */
void orc_philox_raw(uint64_t seed, uint64_t stream_id, uint64_t first_word,
                    int64_t count, uint64_t *out) {
    uint64_t key[2] = {stream_id, seed};
    uint64_t blk[4];
    int64_t w = 0;
    while (w < count) {
        uint64_t word = first_word + (uint64_t)w;
        uint64_t ctr[4] = {word / 4 + 1, 0, 0, 0};
        philox4x64_10(ctr, key, blk);
        for (uint64_t lane = word % 4; lane < 4 && w < count; ++lane, ++w) out[w] = blk[lane];
    }
}

/* binary_source bits: each uint64 is split low-half then high-half into
 * uint32 words, each word feeds 4 bytes least-significant first, and the
 * Lemire draw for range 2 keeps byte >> 7. */
void orc_binary_source(uint64_t seed, uint64_t stream_id, int64_t count, uint8_t *out) {
    int64_t nwords = (count + 7) / 8;
    uint64_t *raw = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(nwords ? nwords : 1));
    orc_philox_raw(seed, stream_id, 0, nwords, raw);
    for (int64_t i = 0; i < count; ++i) {
        uint64_t w = raw[i / 8];
        int sub = (int)(i % 8);
        uint32_t half = (uint32_t)(sub < 4 ? w : (w >> 32));
        uint32_t byte = (half >> (8 * (sub % 4))) & 0xFFu;
        out[i] = (uint8_t)(byte >> 7);
    }
    free(raw);
}

/* ------------------------------------------------------------------ */
/* Generator.standard_normal: numpy's 256-level ziggurat on next_uint64 */
/* (numpy/random/src/distributions/distributions.c)       */
/* ------------------------------------------------------------------ */
#include "ziggurat_tables.h"

typedef struct {
    uint64_t seed, sid, pos; /* next word index of the stream */
    uint64_t blk[4];
    uint64_t blk_id; /* Philox block held in blk, 0 = none */
} raw_stream;

static uint64_t next_u64(raw_stream *s) {
    uint64_t b = s->pos / 4 + 1;
    if (s->blk_id != b) {
        uint64_t key[2] = {s->sid, s->seed};
        uint64_t ctr[4] = {b, 0, 0, 0};
        philox4x64_10(ctr, key, s->blk);
        s->blk_id = b;
    }
    return s->blk[s->pos++ % 4];
}

static double next_double(raw_stream *s) { return (double)(next_u64(s) >> 11) * (1.0 / 9007199254740992.0); }

static double zig_normal(raw_stream *s) {
    for (;;) {
        uint64_t r = next_u64(s);
        int idx = (int)(r & 0xff);
        r >>= 8;
        int sign = (int)(r & 0x1);
        uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
        double x = (double)rabs * ls_zig_wi[idx];
        if (sign & 0x1) x = -x;
        if (rabs < ls_zig_ki[idx]) return x;
        if (idx == 0) {
            for (;;) {
                double xx = -LS_ZIG_INV_R * log1p(-next_double(s));
                double yy = -log1p(-next_double(s));
                if (yy + yy > xx * xx)
                    return ((rabs >> 8) & 0x1) ? -(LS_ZIG_R + xx) : LS_ZIG_R + xx;
            }
        } else {
            if (((ls_zig_fi[idx - 1] - ls_zig_fi[idx]) * next_double(s) + ls_zig_fi[idx]) < exp(-0.5 * x * x))
                return x;
        }
    }
}

/* count standard normals of RngStream(seed, stream_id), in draw order;
 * returns the number of uint64 words consumed */
int64_t orc_standard_normal(uint64_t seed, uint64_t stream_id, int64_t count, double *out) {
    raw_stream s = {seed, stream_id, 0, {0, 0, 0, 0}, 0};
    for (int64_t i = 0; i < count; ++i) out[i] = zig_normal(&s);
    return (int64_t)s.pos;
}

/* ------------------------------------------------------------------ */
/* numpy pairwise summation and reduceat segment sums                  */
/* ------------------------------------------------------------------ */
static double pairwise_d(const double *x, int64_t n) {
    if (n < 8) {
        double r = -0.0;
        for (int64_t i = 0; i < n; ++i) r += x[i];
        return r;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = x[j];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += x[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += x[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise_d(x, n2) + pairwise_d(x + n2, n - n2);
}

static float pairwise_f(const float *x, int64_t n) {
    if (n < 8) {
        float r = -0.0f;
        for (int64_t i = 0; i < n; ++i) r += x[i];
        return r;
    }
    if (n <= 128) {
        float r[8];
        for (int j = 0; j < 8; ++j) r[j] = x[j];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += x[i + j];
        float res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += x[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise_f(x, n2) + pairwise_f(x + n2, n - n2);
}

/* add.reduceat over one contiguous segment: x0 (+ pairwise of the rest). */
static double segsum_d(const double *x, int64_t n) {
    return n == 1 ? x[0] : x[0] + pairwise_d(x + 1, n - 1);
}
static float segsum_f(const float *x, int64_t n) {
    return n == 1 ? x[0] : x[0] + pairwise_f(x + 1, n - 1);
}

/* phi(x) = -log(tanh(clip(x, 1e-12, 40) / 2))  (ldpc.py:77-83) */
static double phi_d(double x) {
    if (x < 1e-12) x = 1e-12;
    if (x > 40.0) x = 40.0;
    return -log(tanh(x / 2.0));
}
static float phi_f(float x) {
    const float lo = (float)1e-12, hi = 40.0f;
    if (x < lo) x = lo;
    if (x > hi) x = hi;
    return -logf(tanhf(x / 2.0f));
}

/* ------------------------------------------------------------------ */
/* bp_decode (ldpc.py:86-172), one codeword at a time                  */
/* ------------------------------------------------------------------ */
enum { V_SUM_PRODUCT = 0, V_MIN_SUM = 1, V_SCALED_MIN_SUM = 2 };

typedef struct {
    int64_t n, m, E;
    const int64_t *cptr; /* [m+1] check -> edge range (check-major edge order) */
    const int64_t *cvar; /* [E]   variable of each edge, ascending per check */
    int64_t *vptr;       /* [n+1] variable -> range in vedge                  */
    int64_t *vedge;      /* [E]   edges of each variable, ascending check     */
} graph_t;

static void build_var_side(graph_t *g) {
    int64_t *deg = (int64_t *)calloc((size_t)g->n + 1, sizeof(int64_t));
    for (int64_t e = 0; e < g->E; ++e) deg[g->cvar[e] + 1]++;
    for (int64_t v = 0; v < g->n; ++v) deg[v + 1] += deg[v];
    memcpy(g->vptr, deg, sizeof(int64_t) * ((size_t)g->n + 1));
    /* check-major edge order => per-variable lists come out in ascending
     * check order, i.e. numpy's stable argsort of var_idx (ldpc.py:50-54) */
    for (int64_t e = 0; e < g->E; ++e) g->vedge[deg[g->cvar[e]]++] = e;
    free(deg);
}

/* is_f64: the LLR dtype (the reference decodes f32 inputs with an f32
 * posterior and f64 messages, f64 inputs fully in f64). */
static int decode_one(const graph_t *g, const void *llr_row, int is_f64, int num_iter, int variant,
                      double scale, int early_stop, void *out_row, uint8_t *hard_row,
                      double *c2v, double *v2c, double *dbuf, float *fbuf, double *total_d,
                      float *total_f, double *chan) {
    const int64_t n = g->n, m = g->m;
    const double alpha = (variant == V_SCALED_MIN_SUM) ? scale : 1.0;
    for (int64_t v = 0; v < n; ++v) {
        if (is_f64) {
            chan[v] = -((const double *)llr_row)[v];
            total_d[v] = chan[v];
        } else {
            float c = -((const float *)llr_row)[v];
            chan[v] = c;
            total_f[v] = c;
        }
    }
    memset(c2v, 0, sizeof(double) * (size_t)g->E);
    int iters_used = num_iter;

    for (int it = 0; it < num_iter; ++it) {
        /* first f32 iteration: c2v is the f32 zero array, so v2c, |v2c|,
         * phi and the check sums are all f32 (ldpc.py:124-143) */
        const int f32_pass = (!is_f64 && it == 0);
        for (int64_t c = 0; c < m; ++c) {
            int64_t e0 = g->cptr[c], e1 = g->cptr[c + 1], d = e1 - e0;
            int par = 0;
            for (int64_t e = e0; e < e1; ++e) {
                double t = is_f64 ? total_d[g->cvar[e]] : (double)total_f[g->cvar[e]];
                v2c[e] = t - c2v[e];
                par ^= signbit(v2c[e]) ? 1 : 0;
            }
            if (variant == V_SUM_PRODUCT) {
                if (f32_pass) {
                    for (int64_t j = 0; j < d; ++j) fbuf[j] = phi_f((float)fabs(v2c[e0 + j]));
                    float ps = segsum_f(fbuf, d);
                    for (int64_t j = 0; j < d; ++j) {
                        float x = ps - fbuf[j];
                        if (x < (float)1e-12) x = (float)1e-12;
                        float me = phi_f(x);
                        if (me < 0.0f) me = 0.0f;
                        if (me > 30.0f) me = 30.0f;
                        int neg = par ^ (signbit(v2c[e0 + j]) ? 1 : 0);
                        dbuf[j] = (neg ? -1.0 : 1.0) * (double)me;
                    }
                } else {
                    double *pm = dbuf; /* reuse as phi buffer, results go to c2v after */
                    for (int64_t j = 0; j < d; ++j) pm[j] = phi_d(fabs(v2c[e0 + j]));
                    double ps = segsum_d(pm, d);
                    for (int64_t j = 0; j < d; ++j) {
                        double x = ps - pm[j];
                        if (x < 1e-12) x = 1e-12;
                        double me = phi_d(x);
                        if (me < 0.0) me = 0.0;
                        if (me > 30.0) me = 30.0;
                        int neg = par ^ (signbit(v2c[e0 + j]) ? 1 : 0);
                        pm[j] = (neg ? -1.0 : 1.0) * me;
                    }
                }
                for (int64_t j = 0; j < d; ++j) c2v[e0 + j] = dbuf[j];
            } else {
                /* exclusive minimum, tie rule of _segment_min2 (ldpc.py:65-74,
                 * 144-148): unique argmin gets min2, every other edge min1 */
                double min1 = INFINITY, min2 = INFINITY;
                for (int64_t e = e0; e < e1; ++e) {
                    double a = fabs(v2c[e]);
                    if (a < min1) min1 = a;
                }
                int64_t cnt = 0;
                for (int64_t e = e0; e < e1; ++e) {
                    double a = fabs(v2c[e]);
                    if (a == min1) cnt++;
                    else if (a < min2) min2 = a;
                }
                for (int64_t e = e0; e < e1; ++e) {
                    double a = fabs(v2c[e]);
                    double ex = (a == min1 && cnt == 1) ? min2 : min1;
                    int neg = par ^ (signbit(v2c[e]) ? 1 : 0);
                    c2v[e] = (alpha * (neg ? -1.0 : 1.0)) * ex;
                }
            }
        }
        /* variable update: total = clip(f(channel + x0 + pairwise(rest)), +-40) */
        for (int64_t v = 0; v < n; ++v) {
            int64_t p0 = g->vptr[v], p1 = g->vptr[v + 1], d = p1 - p0;
            if (d == 0) {
                if (is_f64) total_d[v] = chan[v];
                else total_f[v] = (float)chan[v];
            } else {
                for (int64_t j = 0; j < d; ++j) dbuf[j] = c2v[g->vedge[p0 + j]];
                double s = segsum_d(dbuf, d);
                if (is_f64) {
                    double t = chan[v] + s;
                    total_d[v] = t < -40.0 ? -40.0 : (t > 40.0 ? 40.0 : t);
                } else {
                    float t = (float)(chan[v] + s);
                    total_f[v] = t < -40.0f ? -40.0f : (t > 40.0f ? 40.0f : t);
                }
            }
        }
        if (early_stop) {
            int ok = 1;
            for (int64_t c = 0; c < m && ok; ++c) {
                int syn = 0;
                for (int64_t e = g->cptr[c]; e < g->cptr[c + 1]; ++e) {
                    int64_t v = g->cvar[e];
                    syn ^= (is_f64 ? signbit(total_d[v]) : signbit(total_f[v])) ? 1 : 0;
                }
                if (syn) ok = 0;
            }
            if (ok) {
                iters_used = it + 1;
                break;
            }
        }
    }
    for (int64_t v = 0; v < n; ++v) {
        if (is_f64) {
            double o = -total_d[v];
            ((double *)out_row)[v] = o;
            hard_row[v] = o > 0.0;
        } else {
            float o = -total_f[v];
            ((float *)out_row)[v] = o;
            hard_row[v] = o > 0.0f;
        }
    }
    return iters_used;
}

/* Decode a [batch, n] LLR array on the check-major CSR graph (cptr, cvar).
 * Returns 0 on success; per-row iteration counts go to iters_used. */
int orc_bp_decode(const void *llr, int is_f64, int64_t batch, int64_t n, int64_t m,
                  const int64_t *cptr, const int64_t *cvar, int num_iter, int variant,
                  double scale, int early_stop, void *llr_out, uint8_t *hard,
                  int32_t *iters_used) {
    graph_t g;
    g.n = n;
    g.m = m;
    g.E = cptr[m];
    g.cptr = cptr;
    g.cvar = cvar;
    g.vptr = (int64_t *)malloc(sizeof(int64_t) * ((size_t)n + 1));
    g.vedge = (int64_t *)malloc(sizeof(int64_t) * ((size_t)g.E + 1));
    build_var_side(&g);
    int64_t maxdeg = 1;
    for (int64_t c = 0; c < m; ++c) if (cptr[c + 1] - cptr[c] > maxdeg) maxdeg = cptr[c + 1] - cptr[c];
    for (int64_t v = 0; v < n; ++v) if (g.vptr[v + 1] - g.vptr[v] > maxdeg) maxdeg = g.vptr[v + 1] - g.vptr[v];
    double *c2v = (double *)malloc(sizeof(double) * ((size_t)g.E + 1));
    double *v2c = (double *)malloc(sizeof(double) * ((size_t)g.E + 1));
    double *dbuf = (double *)malloc(sizeof(double) * (size_t)maxdeg);
    float *fbuf = (float *)malloc(sizeof(float) * (size_t)maxdeg);
    double *total_d = (double *)malloc(sizeof(double) * (size_t)n);
    float *total_f = (float *)malloc(sizeof(float) * (size_t)n);
    double *chan = (double *)malloc(sizeof(double) * (size_t)n);
    size_t esz = is_f64 ? sizeof(double) : sizeof(float);
    for (int64_t b = 0; b < batch; ++b) {
        int it = decode_one(&g, (const char *)llr + (size_t)b * (size_t)n * esz, is_f64, num_iter,
                            variant, scale, early_stop, (char *)llr_out + (size_t)b * (size_t)n * esz,
                            hard + (size_t)b * (size_t)n, c2v, v2c, dbuf, fbuf, total_d, total_f,
                            chan);
        if (iters_used) iters_used[b] = it;
    }
    free(c2v); free(v2c); free(dbuf); free(fbuf); free(total_d); free(total_f); free(chan);
    free(g.vptr); free(g.vedge);
    return 0;
}
