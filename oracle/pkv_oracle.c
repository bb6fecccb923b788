/* pkv_oracle.c — plain-C CPU restatement of the ProxyKV pruning hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see pkv_oracle.h). Pinned against the reference
 * compiled from /root/reference (oracle/_ref/libpkvref.so) and the
 * reference's golden vectors by tests/test_oracle.py.
 */
#include "pkv_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ---------------------------------------------------------------- select -- */

int pkvo_retention_count(double rho, int64_t n, int64_t* k_out) {
    /* pruning.cpp:15-17 */
    if (!(rho > 0.0 && rho <= 1.0)) return 2;
    if (!(n > 0)) return 2;
    *k_out = (int64_t)ceil(rho * (double)n);
    return 0;
}

/* Order-preserving map of an fp32 value to uint32 (ascending value ->
 * ascending key); -0.0 is canonicalised to +0.0 because the reference's
 * `values[a] != values[b]` treats them as equal (pruning.cpp:25). */
static uint32_t order_key(float v) {
    uint32_t u;
    if (v == 0.0f) v = 0.0f;
    memcpy(&u, &v, 4);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

static void swap64(uint64_t* a, uint64_t* b) {
    uint64_t t = *a;
    *a = *b;
    *b = t;
}

/* Deterministic quickselect: afterwards a[0..k) holds the k smallest. */
static void select_smallest(uint64_t* a, int64_t n, int64_t k) {
    int64_t lo = 0, hi = n - 1;
    while (hi > lo) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (a[mid] < a[lo]) swap64(&a[mid], &a[lo]);
        if (a[hi] < a[lo]) swap64(&a[hi], &a[lo]);
        if (a[hi] < a[mid]) swap64(&a[hi], &a[mid]);
        const uint64_t pivot = a[mid];
        int64_t i = lo, j = hi;
        while (i <= j) {
            while (a[i] < pivot) ++i;
            while (a[j] > pivot) --j;
            if (i <= j) {
                swap64(&a[i], &a[j]);
                ++i;
                --j;
            }
        }
        if (k - 1 <= j) {
            hi = j;
        } else if (k - 1 >= i) {
            lo = i;
        } else {
            return;
        }
    }
}

int pkvo_topk_select_f32(const float* scores, int64_t slices, int64_t n, int64_t k,
                         uint8_t* mask_out, int32_t* idx_asc_out) {
    /* pruning.cpp:21 */
    if (!(k >= 1 && k <= n)) return 2;
    for (int64_t i = 0; i < slices * n; ++i) {
        if (scores[i] != scores[i]) return 3;
    }
    uint64_t* keys = (uint64_t*)malloc((size_t)n * sizeof(uint64_t));
    uint8_t* mask = (uint8_t*)malloc((size_t)n);
    for (int64_t s = 0; s < slices; ++s) {
        const float* v = scores + s * n;
        /* composite key: (descending value, ascending index) == the reference's
         * better() order (pruning.cpp:24-31) */
        for (int64_t i = 0; i < n; ++i) {
            keys[i] = ((uint64_t)(~order_key(v[i])) << 32) | (uint64_t)(uint32_t)i;
        }
        if (k < n) select_smallest(keys, n, k);
        memset(mask, 0, (size_t)n);
        for (int64_t j = 0; j < k; ++j) mask[keys[j] & 0xffffffffu] = 1;
        if (mask_out) memcpy(mask_out + s * n, mask, (size_t)n);
        if (idx_asc_out) {
            /* apply_mask: linear scan gives ascending indices (pruning.cpp:202-210) */
            int64_t c = 0;
            for (int64_t i = 0; i < n; ++i) {
                if (mask[i]) idx_asc_out[s * k + c++] = (int32_t)i;
            }
        }
    }
    free(keys);
    free(mask);
    return 0;
}

void pkvo_compact_kv(const uint16_t* k_in, const uint16_t* v_in, const int32_t* idx_asc,
                     int64_t slices, int64_t n, int64_t k, int64_t d, uint16_t* k_out,
                     uint16_t* v_out) {
    for (int64_t s = 0; s < slices; ++s) {
        for (int64_t j = 0; j < k; ++j) {
            const int64_t src = (s * n + idx_asc[s * k + j]) * d;
            const int64_t dst = (s * k + j) * d;
            memcpy(k_out + dst, k_in + src, (size_t)d * 2);
            memcpy(v_out + dst, v_in + src, (size_t)d * 2);
        }
    }
}

/* --------------------------------------------------------------- scoring -- */

static double bf16_to_double(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

static void row_scores(const double* qrow, const double* kd, int64_t nk, int64_t d, int64_t kend,
                       double scale, double* s) {
    for (int64_t j = 0; j < kend; ++j) {
        double acc = 0.0;
        const double* kr = kd + j * d;
        for (int64_t c = 0; c < d; ++c) acc += qrow[c] * kr[c];
        s[j] = acc * scale;
    }
    (void)nk;
}

static double* widen(const uint16_t* x, int64_t n) {
    double* o = (double*)malloc((size_t)n * sizeof(double));
    for (int64_t i = 0; i < n; ++i) o[i] = bf16_to_double(x[i]);
    return o;
}

void pkvo_score_head(const uint16_t* q, const uint16_t* k, int64_t group, int64_t nq, int64_t nk,
                     int64_t d, int reduce, int causal, float* x_out) {
    double* kd = widen(k, nk * d);
    double* qd = widen(q, group * nq * d);
    double* s = (double*)malloc((size_t)nk * sizeof(double));
    double* x = (double*)malloc((size_t)nk * sizeof(double));
    const double scale = 1.0 / sqrt((double)d);
    for (int64_t j = 0; j < nk; ++j) x[j] = 0.0;
    for (int64_t h = 0; h < group; ++h) {
        for (int64_t i = 0; i < nq; ++i) {
            const int64_t kend = causal ? (i + (nk - nq) + 1 < nk ? i + (nk - nq) + 1 : nk) : nk;
            if (kend <= 0) continue;
            row_scores(qd + (h * nq + i) * d, kd, nk, d, kend, scale, s);
            double mx = -INFINITY;
            for (int64_t j = 0; j < kend; ++j) mx = s[j] > mx ? s[j] : mx;
            double z = 0.0;
            for (int64_t j = 0; j < kend; ++j) {
                s[j] = exp(s[j] - mx);
                z += s[j];
            }
            for (int64_t j = 0; j < kend; ++j) {
                const double p = s[j] / z;
                if (reduce == 0) {
                    x[j] += p;
                } else if (p > x[j]) {
                    x[j] = p;
                }
            }
        }
    }
    for (int64_t j = 0; j < nk; ++j) x_out[j] = (float)x[j];
    free(kd);
    free(qd);
    free(s);
    free(x);
}

void pkvo_score_lse(const uint16_t* q, const uint16_t* k, int64_t nq, int64_t nk, int64_t d,
                    int causal, float* lse_out) {
    double* kd = widen(k, nk * d);
    double* qd = widen(q, nq * d);
    double* s = (double*)malloc((size_t)nk * sizeof(double));
    const double scale = 1.0 / sqrt((double)d);
    for (int64_t i = 0; i < nq; ++i) {
        const int64_t kend = causal ? (i + (nk - nq) + 1 < nk ? i + (nk - nq) + 1 : nk) : nk;
        row_scores(qd + i * d, kd, nk, d, kend, scale, s);
        double mx = -INFINITY;
        for (int64_t j = 0; j < kend; ++j) mx = s[j] > mx ? s[j] : mx;
        double z = 0.0;
        for (int64_t j = 0; j < kend; ++j) z += exp(s[j] - mx);
        lse_out[i] = (float)(mx + log(z));
    }
    free(kd);
    free(qd);
    free(s);
}

/* ------------------------------------------------------------ rng + init -- */

/* rng.hpp:11-21 */
static uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

static uint64_t derive_seed(uint64_t base, uint64_t stream) {
    return splitmix64(base ^ splitmix64(stream + 1));
}

/* rng.hpp:25-87 */
typedef struct {
    uint64_t s[4];
    double cached;
    int has_cached;
} rng_t;

static void rng_init(rng_t* r, uint64_t seed) {
    uint64_t x = seed;
    for (int i = 0; i < 4; ++i) {
        x = splitmix64(x);
        r->s[i] = x;
    }
    r->cached = 0.0;
    r->has_cached = 0;
}

static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

static uint64_t rng_next(rng_t* r) {
    uint64_t* s = r->s;
    const uint64_t result = rotl(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
}

static double rng_uniform01(rng_t* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }

static double rng_uniform(rng_t* r, double lo, double hi) {
    const double u = rng_uniform01(r);
    return lo + (hi - lo) * u;
}

static uint64_t rng_below(rng_t* r, uint64_t n) {
    const uint64_t threshold = (0 - n) % n;
    for (;;) {
        const uint64_t x = rng_next(r);
        if (x >= threshold) return x % n;
    }
}

static double rng_normal(rng_t* r) {
    if (r->has_cached) {
        r->has_cached = 0;
        return r->cached;
    }
    double u1 = rng_uniform01(r);
    while (u1 <= 0.0) u1 = rng_uniform01(r);
    const double u2 = rng_uniform01(r);
    const double rad = sqrt(-2.0 * log(u1));
    const double theta = 2.0 * M_PI * u2;
    r->cached = rad * sin(theta);
    r->has_cached = 1;
    return rad * cos(theta);
}

void pkvo_rng_uniform(uint64_t seed, double lo, double hi, int64_t n, double* out) {
    rng_t r;
    rng_init(&r, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = rng_uniform(&r, lo, hi);
}

void pkvo_rng_normal(uint64_t seed, int64_t n, double* out) {
    rng_t r;
    rng_init(&r, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = rng_normal(&r);
}

void pkvo_rng_below(uint64_t seed, uint64_t bound, int64_t n, uint64_t* out) {
    rng_t r;
    rng_init(&r, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = rng_below(&r, bound);
}

typedef struct {
    double* blob;
    int64_t pos;
} writer_t;

static void w_uniform(writer_t* w, rng_t* r, int64_t fan_in, int64_t count) {
    /* uniform_init/linear_init (mapper.cpp:83-93): U(-1/sqrt(fan_in), 1/sqrt(fan_in)) */
    const double b = 1.0 / sqrt((double)fan_in);
    for (int64_t i = 0; i < count; ++i) {
        const double v = rng_uniform(r, -b, b);
        if (w->blob) w->blob[w->pos] = v;
        w->pos++;
    }
}

static void w_fill(writer_t* w, double v, int64_t count) {
    for (int64_t i = 0; i < count; ++i) {
        if (w->blob) w->blob[w->pos] = v;
        w->pos++;
    }
}

int64_t pkvo_mapper_init(const int64_t* geom5, const int64_t* cfg12, uint64_t seed, double* blob) {
    const int64_t hl = geom5[1], hs = geom5[3];
    const int64_t dt = cfg12[0], layers = cfg12[1], ffn = cfg12[3] * cfg12[0], dh = cfg12[4];
    const int64_t syn = cfg12[7] > 0 ? cfg12[7] : hs;
    const int conv_active = cfg12[8] == 0, enc_active = cfg12[9] == 0, cross_active = cfg12[10] == 0;
    const int64_t mid = dt / 2 > 0 ? dt / 2 : 1;
    rng_t r;
    rng_init(&r, derive_seed(seed, 0x6d617070ull)); /* mapper.cpp:102 */
    /* Draw order follows mapper.cpp:107-161; the write order follows
     * named_parameters() (mapper.cpp:171-207) then named_buffers()
     * (mapper.cpp:216-223). Both orders coincide for the parameters; BN
     * running stats (drawn nowhere) go last. */
    writer_t w = {blob, 0};
    if (conv_active) {
        w_uniform(&w, &r, hs * 3, mid * hs * 3); /* stem.conv1.w */
        w_uniform(&w, &r, hs * 3, mid);          /* stem.conv1.b */
        w_fill(&w, 1.0, mid);                    /* stem.bn1.gamma */
        w_fill(&w, 0.0, mid);                    /* stem.bn1.beta */
        w_uniform(&w, &r, mid * 3, dt * mid * 3); /* stem.conv2.w */
        w_uniform(&w, &r, mid * 3, dt);           /* stem.conv2.b */
        w_fill(&w, 1.0, dt);                      /* stem.bn2.gamma */
        w_fill(&w, 0.0, dt);                      /* stem.bn2.beta */
    } else {
        w_uniform(&w, &r, hs, dt * hs); /* stem.bypass.w */
        w_uniform(&w, &r, hs, dt);      /* stem.bypass.b */
    }
    if (enc_active) {
        for (int64_t l = 0; l < layers; ++l) {
            for (int m = 0; m < 4; ++m) { /* wq bq wk bk wv bv wo bo */
                w_uniform(&w, &r, dt, dt * dt);
                w_uniform(&w, &r, dt, dt);
            }
            w_fill(&w, 1.0, dt); /* ln1.gamma */
            w_fill(&w, 0.0, dt); /* ln1.beta */
            w_fill(&w, 1.0, dt); /* ln2.gamma */
            w_fill(&w, 0.0, dt); /* ln2.beta */
            w_uniform(&w, &r, dt, dt * ffn);  /* ffn1.w */
            w_uniform(&w, &r, dt, ffn);       /* ffn1.b */
            w_uniform(&w, &r, ffn, ffn * dt); /* ffn2.w */
            w_uniform(&w, &r, ffn, dt);       /* ffn2.b */
        }
    }
    if (cross_active) {
        w_uniform(&w, &r, dt, dt * syn * dh); /* cross.key.w */
        w_uniform(&w, &r, dt, syn * dh);      /* cross.key.b */
    }
    /* named_parameters order is key, value, queries, out — but the draw order
     * is key, queries, value, out (mapper.cpp:152-163). Draw the queries now
     * and park them until value.w/.b are written. */
    double* queries = NULL;
    if (cross_active) {
        queries = (double*)malloc((size_t)(hl * dh) * sizeof(double));
        for (int64_t i = 0; i < hl * dh; ++i) queries[i] = rng_normal(&r) / sqrt((double)dh);
    }
    w_uniform(&w, &r, dt, dt * syn * dh); /* cross.value.w */
    w_uniform(&w, &r, dt, syn * dh);      /* cross.value.b */
    if (cross_active) {
        for (int64_t i = 0; i < hl * dh; ++i) {
            if (w.blob) w.blob[w.pos] = queries[i];
            w.pos++;
        }
        free(queries);
    }
    w_uniform(&w, &r, dh, dh); /* cross.out.w */
    w_uniform(&w, &r, dh, 1);  /* cross.out.b */
    if (conv_active) {
        w_fill(&w, 0.0, mid); /* stem.bn1.running_mean */
        w_fill(&w, 1.0, mid); /* stem.bn1.running_var */
        w_fill(&w, 0.0, dt);  /* stem.bn2.running_mean */
        w_fill(&w, 1.0, dt);  /* stem.bn2.running_var */
    }
    return w.pos;
}
