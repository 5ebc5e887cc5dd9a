/*
 * ORACLE -- test infrastructure, NOT product code (see oracle/__init__.py).
 *
 * O1: paged decode attention in double precision with a two-pass full softmax.
 *
 * The paper defines no attention formula of its own; it defers to
 * PagedAttention (§I, §II-A).  What a decode step
 * computes is standard scaled-dot-product attention of one query token per
 * (request, q-head) over that request's KV cache, with the KV cache stored in
 * fixed-size blocks ("implemented using blocks rather than ... tokens",
 * PAPER.md:213, Alg. 1 prose).  Readings: softmax scale 1/sqrt(d);
 * the query attends to every cached token j < ctx_i including the token
 * appended this step; GQA head map g(h) = floor(h / (Hq/Hkv)).
 *
 * Storage layout used HERE (the oracle's own, not the GPU's):
 *   pool_k, pool_v : uint16 bit patterns [page][Hkv][P][d]
 *   block_table    : int32 [n][bt_stride], entry p = physical page of logical page p
 *   q              : uint16 bit patterns [n][Hq][d]
 *   out            : double [n][Hq][d]
 * dtype: 0 = IEEE binary16, 1 = bfloat16.  Both upcast exactly to double.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* IEEE 754 binary16 -> double, written out from the format definition
 * (1 sign bit, 5 exponent bits with bias 15, 10 fraction bits). */
double oracle_half_to_double(uint16_t h) {
    int sign = (h >> 15) & 1;
    int exp = (h >> 10) & 0x1F;
    int frac = h & 0x3FF;
    double v;
    if (exp == 0) {
        v = ldexp((double)frac, -24);            /* subnormal: frac * 2^-14 * 2^-10 */
    } else if (exp == 31) {
        v = frac ? NAN : INFINITY;
    } else {
        v = ldexp((double)(1024 + frac), exp - 25); /* (1 + frac/1024) * 2^(exp-15) */
    }
    return sign ? -v : v;
}

/* bfloat16 -> double: bfloat16 is the top 16 bits of an IEEE binary32
 * (1 sign, 8 exponent bits with bias 127, 7 fraction bits). */
double oracle_bf16_to_double(uint16_t h) {
    int sign = (h >> 15) & 1;
    int exp = (h >> 7) & 0xFF;
    int frac = h & 0x7F;
    double v;
    if (exp == 0) {
        v = ldexp((double)frac, -133);           /* frac * 2^-126 * 2^-7 */
    } else if (exp == 255) {
        v = frac ? NAN : INFINITY;
    } else {
        v = ldexp((double)(128 + frac), exp - 134); /* (1 + frac/128) * 2^(exp-127) */
    }
    return sign ? -v : v;
}

static double up(uint16_t h, int dtype) {
    return dtype == 0 ? oracle_half_to_double(h) : oracle_bf16_to_double(h);
}

/*
 * out[i][h][:] = sum_j softmax_j(s) V_j,   s_j = (q_{i,h} . K_{i,g(h),j}) / sqrt(d),
 * j = 0 .. ctx_i - 1, K_{i,g,j} = pool_k[bt[i][j / P]][g][j % P][:].
 * Returns 0, or -1 on invalid arguments (ctx < 1, bad head ratio, page id < 0).
 */
int oracle_paged_decode_attention(int n, int Hq, int Hkv, int d, int P,
                                  const int32_t *ctx, const int32_t *block_table, int bt_stride,
                                  const uint16_t *pool_k, const uint16_t *pool_v,
                                  const uint16_t *q, int dtype, double *out, int nthreads) {
    if (n < 0 || Hq < 1 || Hkv < 1 || Hq % Hkv != 0 || d < 1 || P < 1) return -1;
    int group = Hq / Hkv;
    int bad = 0;
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads) reduction(| : bad)
    for (long ih = 0; ih < (long)n * Hq; ++ih) {
        int i = (int)(ih / Hq);
        int h = (int)(ih % Hq);
        int g = h / group;
        int c = ctx[i];
        if (c < 1) { bad = 1; continue; }
        double *s = (double *)malloc(sizeof(double) * (size_t)c);
        double *qd = (double *)malloc(sizeof(double) * (size_t)d);
        for (int e = 0; e < d; ++e) qd[e] = up(q[((size_t)i * Hq + h) * d + e], dtype);
        /* pass 1: scores and their maximum */
        double smax = -INFINITY;
        if ((c + P - 1) / P > bt_stride) { bad = 1; free(s); free(qd); continue; }
        for (int j = 0; j < c; ++j) {
            int page = block_table[(size_t)i * bt_stride + j / P];
            if (page < 0) { bad = 1; page = 0; }
            const uint16_t *kj = pool_k + (((size_t)page * Hkv + g) * P + (j % P)) * d;
            double dot = 0.0;
            for (int e = 0; e < d; ++e) dot += qd[e] * up(kj[e], dtype);
            s[j] = dot / sqrt((double)d);
            if (s[j] > smax) smax = s[j];
        }
        /* pass 2: normaliser, then the probability-weighted sum of V */
        double denom = 0.0;
        for (int j = 0; j < c; ++j) {
            s[j] = exp(s[j] - smax);
            denom += s[j];
        }
        double *o = out + ((size_t)i * Hq + h) * d;
        for (int e = 0; e < d; ++e) o[e] = 0.0;
        for (int j = 0; j < c; ++j) {
            int page = block_table[(size_t)i * bt_stride + j / P];
            if (page < 0) page = 0;
            const uint16_t *vj = pool_v + (((size_t)page * Hkv + g) * P + (j % P)) * d;
            double p = s[j] / denom;
            for (int e = 0; e < d; ++e) o[e] += p * up(vj[e], dtype);
        }
        free(s);
        free(qd);
    }
    return bad ? -1 : 0;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
