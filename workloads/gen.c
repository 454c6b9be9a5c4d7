/*
 * Seeded synthetic input generators shared by the oracle tests and the CUDA path.
 *
 * This module holds NONE of the softmax method's arithmetic: it only draws
 * numbers.  It is a counter-based generator (SplitMix64 finaliser applied to a
 * keyed counter), so any sub-range of any stream can be produced independently
 * and in parallel: element i of stream (seed, stream) is a pure function of
 * (seed, stream, i).  That is what makes shard-invariant generation of the
 * multi-GPU workloads possible (rank k generates only its chunk).
 *
 * Distributions:
 *   uniform(lo, hi):  lo + (hi - lo) * u,  u = 53-bit uniform in [0, 1), fp64, then RN to fp32
 *   normal(mu, sd):   Box-Muller (cosine branch) from two uniforms of the same counter, fp64 -> fp32
 *   bernoulli(p):     u < p
 * bf16 inputs are fp32 values rounded to nearest-even bf16.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

static inline uint64_t wl_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

static inline uint64_t wl_key(uint64_t seed, uint64_t stream) {
    return wl_mix64(wl_mix64(seed ^ 0x6a09e667f3bcc909ULL) + stream * 0x9e3779b97f4a7c15ULL);
}

/* 53-bit uniform in [0,1) from draw `j` of a keyed stream */
static inline double wl_u01(uint64_t key, uint64_t j) {
    uint64_t r = wl_mix64(key + (j + 1) * 0xd1b54a32d192ed03ULL);
    return (double)(r >> 11) * 0x1.0p-53;
}

void wl_uniform_f32(float* out, int64_t n, uint64_t seed, uint64_t stream, int64_t offset,
                    double lo, double hi) {
    const uint64_t key = wl_key(seed, stream);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double u = wl_u01(key, (uint64_t)(offset + i));
        out[i] = (float)(lo + (hi - lo) * u);
    }
}

/* u in (0,1] for the log argument of Box-Muller */
static inline double wl_u01_open0(uint64_t key, uint64_t j) {
    uint64_t r = wl_mix64(key + (j + 1) * 0xd1b54a32d192ed03ULL);
    return ((double)(r >> 11) + 1.0) * 0x1.0p-53;
}

static inline double wl_normal(uint64_t key, uint64_t i) {
    double u1 = wl_u01_open0(key, 2 * i);
    double u2 = wl_u01(key, 2 * i + 1);
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}

void wl_normal_f32(float* out, int64_t n, uint64_t seed, uint64_t stream, int64_t offset,
                   double mean, double sd) {
    const uint64_t key = wl_key(seed, stream);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = (float)(mean + sd * wl_normal(key, (uint64_t)(offset + i)));
}

/* Row-structured normal: out[r][c] = N(0, sd) [stream s_val, index (row0+r)*ld_cols + col0+c]
 *                                  + U[-off, off] [stream s_off, index row0+r]             */
void wl_rows_normal_offset_f32(float* out, int64_t nrows, int64_t ncols, int64_t row0,
                               int64_t col0, int64_t full_cols, uint64_t seed,
                               uint64_t s_val, uint64_t s_off, double sd, double off) {
    const uint64_t kv = wl_key(seed, s_val), ko = wl_key(seed, s_off);
    #pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < nrows; ++r) {
        double o = -off + 2.0 * off * wl_u01(ko, (uint64_t)(row0 + r));
        float* dst = out + r * ncols;
        uint64_t base = (uint64_t)((row0 + r) * full_cols + col0);
        for (int64_t c = 0; c < ncols; ++c) dst[c] = (float)(o + sd * wl_normal(kv, base + (uint64_t)c));
    }
}

/* Max of the uniform stream over [0, n): the tie value M of config 5. */
float wl_uniform_max_f32(int64_t n, uint64_t seed, uint64_t stream, double lo, double hi) {
    const uint64_t key = wl_key(seed, stream);
    float best = -INFINITY;
    #pragma omp parallel for schedule(static) reduction(max : best)
    for (int64_t i = 0; i < n; ++i) {
        float v = (float)(lo + (hi - lo) * wl_u01(key, (uint64_t)i));
        if (v > best) best = v;
    }
    return best;
}

/* Overwrite positions whose Bernoulli(p) draw fires with `value`.  Returns the count. */
int64_t wl_bernoulli_set_f32(float* out, int64_t n, uint64_t seed, uint64_t stream,
                             int64_t offset, double p, float value) {
    const uint64_t key = wl_key(seed, stream);
    int64_t cnt = 0;
    #pragma omp parallel for schedule(static) reduction(+ : cnt)
    for (int64_t i = 0; i < n; ++i) {
        if (wl_u01(key, (uint64_t)(offset + i)) < p) { out[i] = value; ++cnt; }
    }
    return cnt;
}

/* fp32 -> bf16 round-to-nearest-even (finite inputs) */
void wl_f32_to_bf16(const float* in, uint16_t* out, int64_t n) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        uint32_t b; memcpy(&b, &in[i], 4);
        uint32_t lsb = (b >> 16) & 1u;
        b += 0x7fffu + lsb;
        out[i] = (uint16_t)(b >> 16);
    }
}

void wl_bf16_to_f32(const uint16_t* in, float* out, int64_t n) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        uint32_t b = (uint32_t)in[i] << 16;
        memcpy(&out[i], &b, 4);
    }
}
