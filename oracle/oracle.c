/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU softmax for checking the CUDA path of
 * the Two-Pass softmax build (arXiv 2001.04438).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library.  It shares no code, header, constant or table with
 * paper_2001_04438_b200/ (the CUDA path), and includes nothing from it.
 *
 * What it computes is the plain DEFINITION the Two-Pass method reaches
 * (up to rounding): softmax  sigma(x)_i = e^{x_i} / sum_k e^{x_k}
 * (§1 and PAPER.md:76, §3), evaluated through the shift
 * identity sigma(x)_i = e^{x_i - c} / sum_k e^{x_k - c} with c = max_i x_i
 * (§3), in fp64 exp with long-double (x87, 64-bit mantissa)
 * accumulation.  A second, independent formula (no shift, long-double expl)
 * cross-checks it where long double does not overflow (|x| <= 11356).
 *
 * Also here: the plain definition of the paper's ExtExp pair (PAPER.md:143,
 * §4 eq.): n = nearest integer to x*log2(e),  m = e^{x - n ln 2},
 * evaluated in long double.
 *
 * Parity pins for every function live in tests/test_oracle_pins.py.
 */
#include <math.h>
#include <stdint.h>
#include <float.h>
#include <stdlib.h>

#define ORACLE_CHUNK 65536

#ifdef _OPENMP
#include <omp.h>
int oracle_threads(void) { return omp_get_max_threads(); }
#else
int oracle_threads(void) { return 1; }
#endif

static inline double bf16_value(uint16_t b) {
    union { uint32_t u; float f; } v;
    v.u = (uint32_t)b << 16;
    return (double)v.f;
}

/* ---- row statistics: mu = max_i x_i (Alg. 1 pass 1),
 *      S = sum_i exp(x_i - mu)                          */
#define DEFINE_STATS(NAME, T, LOAD)                                                        \
void NAME(const T* x, int64_t n, double* mu_out, long double* S_out) {                     \
    double mu = -INFINITY;                                                                 \
    _Pragma("omp parallel for reduction(max : mu) schedule(static)")                       \
    for (int64_t i = 0; i < n; ++i) { double v = LOAD(x[i]); if (v > mu) mu = v; }        \
    /* fixed chunks, then an ordered sum: the result does not depend on threads */         \
    int64_t nchunk = (n + ORACLE_CHUNK - 1) / ORACLE_CHUNK;                                \
    long double* part = (long double*)malloc(sizeof(long double) * (size_t)(nchunk + 1));  \
    _Pragma("omp parallel for schedule(static)")                                           \
    for (int64_t c = 0; c < nchunk; ++c) {                                                 \
        int64_t lo = c * ORACLE_CHUNK, hi = lo + ORACLE_CHUNK < n ? lo + ORACLE_CHUNK : n; \
        long double s = 0.0L;                                                              \
        for (int64_t i = lo; i < hi; ++i) s += (long double)exp(LOAD(x[i]) - mu);          \
        part[c] = s;                                                                       \
    }                                                                                      \
    long double S = 0.0L;                                                                  \
    for (int64_t c = 0; c < nchunk; ++c) S += part[c];                                     \
    free(part);                                                                            \
    *mu_out = mu; *S_out = S;                                                              \
}

#define LOAD_F32(v) ((double)(v))
#define LOAD_BF16(v) bf16_value(v)
DEFINE_STATS(oracle_row_stats_f32, float, LOAD_F32)
DEFINE_STATS(oracle_row_stats_bf16, uint16_t, LOAD_BF16)

/* ---- full outputs o_i = exp(x_i - mu) / S, long double */
#define DEFINE_SOFTMAX(NAME, STATS, T, LOAD)                                               \
void NAME(const T* x, int64_t n, long double* out) {                                       \
    double mu; long double S;                                                              \
    STATS(x, n, &mu, &S);                                                                  \
    _Pragma("omp parallel for schedule(static)")                                           \
    for (int64_t i = 0; i < n; ++i) out[i] = (long double)exp(LOAD(x[i]) - mu) / S;        \
}
DEFINE_SOFTMAX(oracle_softmax_f32, oracle_row_stats_f32, float, LOAD_F32)
DEFINE_SOFTMAX(oracle_softmax_bf16, oracle_row_stats_bf16, uint16_t, LOAD_BF16)

/* ---- independent cross-check: no shift, o_i = expl(x_i) / sum_k expl(x_k)
 *      (PAPER.md:76 formula taken literally; valid while expl does not
 *      overflow, |x| <= 11356.5).  Sequential long-double sum.            */
void oracle_softmax_unshifted_f32(const float* x, int64_t n, long double* out) {
    long double S = 0.0L;
    for (int64_t i = 0; i < n; ++i) S += expl((long double)x[i]);
    for (int64_t i = 0; i < n; ++i) out[i] = expl((long double)x[i]) / S;
}

/* ---- element-wise tolerance check (BASELINE.json:north_star):
 *   o_i >= FLT_MIN :  |y_i - o_i| <= rtol * o_i
 *   o_i <  FLT_MIN :  |y_i - o_i| <= atol
 * stats[0] = max relative error over the relative branch
 * stats[1] = max absolute error over the absolute branch
 * stats[2] = #elements graded by the relative branch
 * stats[3] = #elements graded by the absolute branch
 * stats[4] = fp64 sum of y
 * returns the number of violations; *first_bad = first violating index or -1.
 * NaN/Inf in y always count as violations.                                  */
#define DEFINE_CHECK(NAME, T, LOAD)                                                         \
int64_t NAME(const T* x, const float* y, int64_t n, double mu, long double S,              \
             double rtol, double atol, double* stats, int64_t* first_bad) {                \
    int64_t bad = 0, nrel = 0, nabs = 0, first = INT64_MAX;                                        \
    double maxrel = 0.0, maxabs = 0.0, ysum = 0.0;                                          \
    _Pragma("omp parallel for schedule(static) reduction(+ : bad, nrel, nabs, ysum) reduction(max : maxrel, maxabs) reduction(min : first)") \
    for (int64_t i = 0; i < n; ++i) {                                                       \
        long double o = (long double)exp(LOAD(x[i]) - mu) / S;                              \
        long double yi = (long double)y[i];                                                 \
        ysum += (double)y[i];                                                               \
        int ok;                                                                             \
        if (!isfinite(y[i])) { ok = 0; if (o >= FLT_MIN) ++nrel; else ++nabs; }             \
        else if (o >= (long double)FLT_MIN) {                                               \
            double rel = (double)(fabsl(yi - o) / o);                                       \
            ++nrel; if (rel > maxrel) maxrel = rel; ok = rel <= rtol;                       \
        } else {                                                                            \
            double ab = (double)fabsl(yi - o);                                              \
            ++nabs; if (ab > maxabs) maxabs = ab; ok = ab <= atol;                          \
        }                                                                                   \
        if (!ok) { ++bad; if (i < first) first = i; }                          \
    }                                                                                       \
    stats[0] = maxrel; stats[1] = maxabs; stats[2] = (double)nrel; stats[3] = (double)nabs; \
    stats[4] = ysum;                                                                        \
    *first_bad = bad ? first : -1;                                                          \
    return bad;                                                                             \
}
DEFINE_CHECK(oracle_check_f32, float, LOAD_F32)
DEFINE_CHECK(oracle_check_bf16, uint16_t, LOAD_BF16)

/* ---- ExtExp, plain definition (§4):
 *   n = round(x * log2 e)  (nearest integer; exact product in long double)
 *   m = e^{x - n ln 2}     so that e^x = m * 2^n,  m in [sqrt(2)/2, sqrt(2)]   */
void oracle_extexp(const float* x, int64_t count, long double* m, double* nexp) {
    const long double LOG2E = 1.4426950408889634073599246810018921L;
    const long double LN2 = 0.6931471805599453094172321214581766L;
    for (int64_t i = 0; i < count; ++i) {
        long double xl = (long double)x[i];
        long double nn = rintl(xl * LOG2E);
        nexp[i] = (double)nn;
        m[i] = expl(xl - nn * LN2);
    }
}

/* ---- e^x * 2^-k in long double: the value a pair (m, n) must represent.
 *      Used to grade GPU pairs whose n differs from the exact nearest
 *      integer (x*log2e within a rounding of a half-integer).              */
void oracle_exp_scaled(const float* x, const double* k, int64_t count, long double* out) {
    const long double LN2 = 0.6931471805599453094172321214581766L;
    for (int64_t i = 0; i < count; ++i) out[i] = expl((long double)x[i] - (long double)k[i] * LN2);
}
