/*
 * skl_oracle.c -- CPU restatement of the reference SKLinear hot path (f64).
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * kernels in paper_2601_15473_b200/.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product path never links or calls it (there is no CPU fallback).
 *
 * It restates, operation for operation, the reference "rnla" C++ library
 * (/root/reference/proj, read-only, not vendored):
 *   - Splitmix64 / GaussianStream / derive_seed   rng.hpp:13-69
 *   - realize_sketch (Gaussian, Rademacher)       sketch.cpp:34-49
 *   - gaussian_matrix                             sketch.cpp:120-125
 *   - gemm_rows / matmul (i-k-j, zero skip)       linalg.cpp:13-39
 *   - SkLinear::forward                           nn_layers.cpp:61-76
 *   - SkLinear::backward                          nn_layers.cpp:78-101
 *   - sk_linear_fresh (U init from one stream)    nn_layers.cpp:133-147
 *   - sk_stored_coeffs / exceeds_dense            layers.hpp:21-31
 *
 * Layout is the reference's: column convention (x is d_in x T, y is
 * d_out x T), all matrices row-major f64, per-term matrices stacked:
 *   s1[l][k][d_out], u1[l][k][d_in], s2[l][k][d_in], u2[l][d_out][k].
 *
 * The accumulation order (and the zero-skip of gemm_rows) matches the
 * reference exactly; compiled with -ffp-contract=off and no -march (the
 * reference's CMake flags) the results are bit-identical to the reference,
 * which tests/test_oracle.py checks against oracle/_ref (the reference
 * sources compiled here) and against the known-answer values in
 * tests/golden/.  Single-threaded: the reference's OpenMP split is over
 * output rows with a fixed reduction order, so thread count does not change
 * bits (linalg.cpp:11-12).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_SHAPE 1
#define ORC_ERR_PARAM 2
#define ORC_ERR_ALLOC 3

/* ---- rng.hpp:13-37 Splitmix64 ----------------------------------------- */
typedef struct { uint64_t state; } orc_sm64;

static inline uint64_t sm64_next(orc_sm64* s) {
    uint64_t z = (s->state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
static inline double sm64_open01(orc_sm64* s) {          /* rng.hpp:25-27 */
    return ((double)(sm64_next(s) >> 11) + 0.5) * 0x1.0p-53;
}
static inline int sm64_bool(orc_sm64* s) { return (sm64_next(s) >> 63) != 0; } /* rng.hpp:30 */

/* ---- rng.hpp:41-63 GaussianStream ------------------------------------- */
typedef struct { orc_sm64 rng; double spare; int have_spare; } orc_gauss;

static inline void gauss_init(orc_gauss* g, uint64_t seed) {
    g->rng.state = seed; g->spare = 0.0; g->have_spare = 0;
}
static inline double gauss_next(orc_gauss* g) {
    if (g->have_spare) { g->have_spare = 0; return g->spare; }
    const double u1 = sm64_open01(&g->rng);
    const double u2 = sm64_open01(&g->rng);
    const double r = sqrt(-2.0 * log(u1));
    const double theta = 2.0 * 3.14159265358979323846 * u2;
    g->spare = r * sin(theta);
    g->have_spare = 1;
    return r * cos(theta);
}

/* ---- rng.hpp:66-69 derive_seed ---------------------------------------- */
uint64_t orc_derive_seed(uint64_t master, uint64_t index) {
    orc_sm64 s = { master ^ (0x517cc1b727220a95ULL + index) };
    return sm64_next(&s);
}

/* First n raw u64 draws of Splitmix64(seed) (test_sketch.cpp:25-33 golden). */
void orc_splitmix64_stream(uint64_t seed, uint64_t n, uint64_t* out) {
    orc_sm64 s = { seed };
    for (uint64_t i = 0; i < n; ++i) out[i] = sm64_next(&s);
}

/* First n values of GaussianStream(seed). */
void orc_gaussian_stream(uint64_t seed, uint64_t n, double* out) {
    orc_gauss g; gauss_init(&g, seed);
    for (uint64_t i = 0; i < n; ++i) out[i] = gauss_next(&g);
}

/* ---- sketch.cpp:34-49 realize_sketch; dist 0 = Gaussian, 1 = Rademacher */
int orc_realize_sketch(int dist, uint64_t k, uint64_t d, uint64_t seed, double* out) {
    if (k < 1 || d < 1) return ORC_ERR_SHAPE;              /* sketch.cpp:92 */
    const uint64_t n = k * d;
    if (dist == 0) {
        orc_gauss g; gauss_init(&g, seed);
        const double scale = 1.0 / sqrt((double)k);
        for (uint64_t i = 0; i < n; ++i) out[i] = gauss_next(&g) * scale;
    } else if (dist == 1) {
        orc_sm64 rng = { seed };
        const double v = 1.0 / sqrt((double)k);
        for (uint64_t i = 0; i < n; ++i) out[i] = sm64_bool(&rng) ? v : -v;
    } else {
        return ORC_ERR_PARAM;   /* SparseSign is out of scope (only CQRRPT uses it) */
    }
    return ORC_OK;
}

/* sketch.cpp:120-125 */
void orc_gaussian_matrix(uint64_t rows, uint64_t cols, uint64_t seed, double* out) {
    orc_gauss g; gauss_init(&g, seed);
    for (uint64_t i = 0; i < rows * cols; ++i) out[i] = gauss_next(&g);
}

/* ---- layers.hpp:21-31 ------------------------------------------------- */
uint64_t orc_sk_stored_coeffs(uint64_t l, uint64_t k, uint64_t d_in, uint64_t d_out) {
    return 2 * l * k * (d_in + d_out);
}
int orc_exceeds_dense(uint64_t l, uint64_t k, uint64_t d_in, uint64_t d_out) {
    return orc_sk_stored_coeffs(l, k, d_in, d_out) > d_in * d_out;
}

/* ---- linalg.cpp:13-29 gemm_rows: C[m][n] = A[m][kk] B[kk][n] ----------- */
static void gemm_rows(const double* a, const double* b, double* c,
                      uint64_t m, uint64_t k, uint64_t n) {
    for (uint64_t i = 0; i < m; ++i) {
        double* crow = c + i * n;
        for (uint64_t j = 0; j < n; ++j) crow[j] = 0.0;
        const double* arow = a + i * k;
        for (uint64_t kk = 0; kk < k; ++kk) {
            const double av = arow[kk];
            if (av == 0.0) continue;                         /* linalg.cpp:24 */
            const double* brow = b + kk * n;
            for (uint64_t j = 0; j < n; ++j) crow[j] += av * brow[j];
        }
    }
}

/* linalg.cpp:54-59 */
static void transpose(const double* a, uint64_t r, uint64_t c, double* t) {
    for (uint64_t i = 0; i < r; ++i)
        for (uint64_t j = 0; j < c; ++j) t[j * r + i] = a[i * c + j];
}

/* ---- nn_layers.cpp:133-147 sk_linear_fresh (U part; sketches via seeds) */
int orc_sk_linear_fresh(uint64_t d_in, uint64_t d_out, uint64_t l, uint64_t k,
                        uint64_t seed, int dist,
                        double* s1, double* u1, double* s2, double* u2) {
    if (l < 1 || k < 1) return ORC_ERR_PARAM;              /* nn_layers.cpp:116 */
    for (uint64_t i = 0; i < l; ++i) {                     /* nn_layers.cpp:124-127 */
        int rc = orc_realize_sketch(dist, k, d_out, orc_derive_seed(seed, 2 * i), s1 + i * k * d_out);
        if (rc) return rc;
        rc = orc_realize_sketch(dist, k, d_in, orc_derive_seed(seed, 2 * i + 1), s2 + i * k * d_in);
        if (rc) return rc;
    }
    const double std_dev = sqrt(2.0 / (double)(d_in + d_out));
    for (uint64_t i = 0; i < l; ++i) {
        orc_gauss g; gauss_init(&g, orc_derive_seed(seed, 1000 + i));
        double* pu1 = u1 + i * k * d_in;
        for (uint64_t t = 0; t < k * d_in; ++t) pu1[t] = gauss_next(&g) * std_dev;
        double* pu2 = u2 + i * d_out * k;
        for (uint64_t t = 0; t < d_out * k; ++t) pu2[t] = gauss_next(&g) * std_dev;
    }
    return ORC_OK;
}

/* ---- nn_layers.cpp:61-76 SkLinear::forward ----------------------------- */
int orc_sk_forward(uint64_t d_in, uint64_t d_out, uint64_t l, uint64_t k, uint64_t T,
                   const double* s1, const double* u1, const double* s2, const double* u2,
                   const double* bias, const double* x, double* y) {
    if (l < 1 || k < 1) return ORC_ERR_PARAM;
    double* acc = (double*)calloc(d_out * T, sizeof(double));
    double* a = (double*)malloc(k * T * sizeof(double));
    double* at = (double*)malloc(T * k * sizeof(double));
    double* left = (double*)malloc(T * d_out * sizeof(double));
    double* s2x = (double*)malloc(k * T * sizeof(double));
    double* right = (double*)malloc(d_out * T * sizeof(double));
    if (!acc || !a || !at || !left || !s2x || !right) {
        free(acc); free(a); free(at); free(left); free(s2x); free(right);
        return ORC_ERR_ALLOC;
    }
    for (uint64_t t = 0; t < l; ++t) {
        gemm_rows(u1 + t * k * d_in, x, a, k, d_in, T);         /* U1 x        */
        transpose(a, k, T, at);                                 /* (U1 x)^T    */
        gemm_rows(at, s1 + t * k * d_out, left, T, k, d_out);   /* apply_right_t(s1, .) */
        for (uint64_t i = 0; i < d_out; ++i)                    /* :67-68      */
            for (uint64_t j = 0; j < T; ++j) acc[i * T + j] += left[j * d_out + i];
        gemm_rows(s2 + t * k * d_in, x, s2x, k, d_in, T);       /* apply_left(s2, x) */
        gemm_rows(u2 + t * d_out * k, s2x, right, d_out, k, T); /* U2 (S2 x)   */
        for (uint64_t i = 0; i < d_out * T; ++i) acc[i] += right[i];   /* :70 */
    }
    const double inv = 1.0 / (2.0 * (double)l);
    for (uint64_t i = 0; i < d_out * T; ++i) y[i] = acc[i] * inv;     /* scale :72-73 */
    for (uint64_t i = 0; i < d_out; ++i) {                            /* add_bias_columns :15-21 */
        const double bi = bias[i];
        for (uint64_t j = 0; j < T; ++j) y[i * T + j] += bi;
    }
    free(acc); free(a); free(at); free(left); free(s2x); free(right);
    return ORC_OK;
}

/* ---- nn_layers.cpp:78-101 SkLinear::backward --------------------------- */
int orc_sk_backward(uint64_t d_in, uint64_t d_out, uint64_t l, uint64_t k, uint64_t T,
                    const double* s1, const double* u1, const double* s2, const double* u2,
                    const double* x, const double* g,
                    double* gx, double* gu1, double* gu2, double* gb) {
    if (l < 1 || k < 1) return ORC_ERR_PARAM;
    const double inv = 1.0 / (2.0 * (double)l);
    double* xt = (double*)malloc(T * d_in * sizeof(double));
    double* s1g = (double*)malloc(k * T * sizeof(double));
    double* s2x = (double*)malloc(k * T * sizeof(double));
    double* s2xt = (double*)malloc(T * k * sizeof(double));
    double* tmp = (double*)malloc((d_in > d_out ? d_in : d_out) * k * sizeof(double));
    double* u1t = (double*)malloc(d_in * k * sizeof(double));
    double* gx1 = (double*)malloc(d_in * T * sizeof(double));
    double* u2t = (double*)malloc(k * d_out * sizeof(double));
    double* u2tg = (double*)malloc(k * T * sizeof(double));
    double* u2tgt = (double*)malloc(T * k * sizeof(double));
    double* gx2 = (double*)malloc(T * d_in * sizeof(double));
    int rc = ORC_OK;
    if (!xt || !s1g || !s2x || !s2xt || !tmp || !u1t || !gx1 || !u2t || !u2tg || !u2tgt || !gx2) {
        rc = ORC_ERR_ALLOC; goto done;
    }
    memset(gx, 0, d_in * T * sizeof(double));
    transpose(x, d_in, T, xt);                                        /* :86 */
    for (uint64_t t = 0; t < l; ++t) {
        const double* ps1 = s1 + t * k * d_out;
        const double* ps2 = s2 + t * k * d_in;
        const double* pu1 = u1 + t * k * d_in;
        const double* pu2 = u2 + t * d_out * k;
        gemm_rows(ps1, g, s1g, k, d_out, T);                          /* :88 */
        gemm_rows(ps2, x, s2x, k, d_in, T);                           /* :89 */
        gemm_rows(s1g, xt, tmp, k, T, d_in);                          /* :90 */
        for (uint64_t i = 0; i < k * d_in; ++i) gu1[t * k * d_in + i] = tmp[i] * inv;
        transpose(s2x, k, T, s2xt);                                   /* :91 */
        gemm_rows(g, s2xt, tmp, d_out, T, k);
        for (uint64_t i = 0; i < d_out * k; ++i) gu2[t * d_out * k + i] = tmp[i] * inv;
        transpose(pu1, k, d_in, u1t);                                 /* :92 */
        gemm_rows(u1t, s1g, gx1, d_in, k, T);
        transpose(pu2, d_out, k, u2t);                                /* :93 */
        gemm_rows(u2t, g, u2tg, k, d_out, T);
        transpose(u2tg, k, T, u2tgt);                                 /* :94 */
        gemm_rows(u2tgt, ps2, gx2, T, k, d_in);
        for (uint64_t i = 0; i < d_in; ++i)                           /* :95-97 */
            for (uint64_t j = 0; j < T; ++j)
                gx[i * T + j] += inv * (gx1[i * T + j] + gx2[j * d_in + i]);
    }
    for (uint64_t i = 0; i < d_out; ++i) {                            /* row_sums :23-30 */
        double s = 0.0;
        for (uint64_t j = 0; j < T; ++j) s += g[i * T + j];
        gb[i] = s;
    }
done:
    free(xt); free(s1g); free(s2x); free(s2xt); free(tmp); free(u1t);
    free(gx1); free(u2t); free(u2tg); free(u2tgt); free(gx2);
    return rc;
}

/* ---- nn_layers.cpp:51-59 dense_linear_init: w = gaussian_matrix(d_out, d_in,
 * seed) stream order times sqrt(2/(d_in+d_out)); zero bias ---------------- */
void orc_dense_init(uint64_t d_in, uint64_t d_out, uint64_t seed, double* w, double* b) {
    orc_gauss g; gauss_init(&g, seed);
    const double std_dev = sqrt(2.0 / (double)(d_in + d_out));
    for (uint64_t i = 0; i < d_out * d_in; ++i) w[i] = gauss_next(&g) * std_dev;
    for (uint64_t i = 0; i < d_out; ++i) b[i] = 0.0;
}

/* ---- nn_layers.cpp:32-37 DenseLinear::forward: y = w x + b (column convention) */
int orc_dense_forward(uint64_t d_in, uint64_t d_out, uint64_t T, const double* w, const double* b,
                      const double* x, double* y) {
    gemm_rows(w, x, y, d_out, d_in, T);
    for (uint64_t i = 0; i < d_out; ++i)                              /* add_bias_columns :15-21 */
        for (uint64_t j = 0; j < T; ++j) y[i * T + j] += b[i];
    return ORC_OK;
}

/* ---- nn_layers.cpp:39-49 DenseLinear::backward ------------------------- */
int orc_dense_backward(uint64_t d_in, uint64_t d_out, uint64_t T, const double* w, const double* x,
                       const double* g, double* gx, double* gw, double* gb) {
    double* xt = (double*)malloc(T * d_in * sizeof(double));
    double* wt = (double*)malloc(d_in * d_out * sizeof(double));
    if (!xt || !wt) { free(xt); free(wt); return ORC_ERR_ALLOC; }
    transpose(x, d_in, T, xt);
    gemm_rows(g, xt, gw, d_out, T, d_in);                             /* :44 grad_w = G x^T */
    transpose(w, d_out, d_in, wt);
    gemm_rows(wt, g, gx, d_in, d_out, T);                             /* :45 grad_x = w^T G */
    for (uint64_t i = 0; i < d_out; ++i) {                            /* :46 row_sums */
        double s = 0.0;
        for (uint64_t j = 0; j < T; ++j) s += g[i * T + j];
        gb[i] = s;
    }
    free(xt); free(wt);
    return ORC_OK;
}
