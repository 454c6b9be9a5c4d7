// Device building blocks of the Two-Pass softmax (arXiv 2001.04438) for sm_100a.
//
//   L0  ext_exp / exp_flush / pow2_flush   PAPER.md:139-149 (§4), Alg. 4 PAPER.md:234-263 (§6.3)
//   L1  pair_merge, thread accumulate, CTA trees  Alg. 3 PAPER.md:153-170 (§4)
//
// Readings of the paper taken here are listed in DESIGN.md ("Readings"), ids G1..G25 as in
// SURVEY.md §8(c).  Everything is IEEE round-to-nearest fp32 with explicit __f*_rn intrinsics,
// so the arithmetic is fixed by the source and not by compiler contraction choices.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tp {

// ----------------------------------------------------------------------------- constants
// n = round(x * log2 e): fp32 log2(e) = RN32(1/ln 2) (reading G1).
constexpr float kLog2e = 0x1.715476p+0f;          // 0x3FB8AA3B
// Cody-Waite split of ln 2 into two fp32 constants (reading G2).
constexpr float kLn2Hi = 0x1.62e430p-1f;          // RN32(ln 2)            0x3F317218
constexpr float kLn2Lo = -0x1.05c610p-29f;        // RN32(ln 2 - kLn2Hi)   0xB102E308
// 1.5 * 2^23: fma(x, log2e, kMagic) - kMagic is round-to-nearest-even of the exact
// product x*log2e whenever |x*log2e| < 2^22 (guaranteed by the clamp below).
constexpr float kMagic = 0x1.8p23f;
// Guaranteed-accuracy domain |x| <= 2^21 (reading G11); inputs outside are clamped.
constexpr float kXClamp = 0x1.0p21f;
// Degree-5 polynomial p(t) = 1 + t(c1 + t(c2 + t(c3 + t(c4 + t c5)))) for e^t on
// |t| <= 0.3476.  The paper's Sollya coefficients are not printed
// (reading G3); these come from tools/fit_exp_poly.py (relative minimax + fp32
// neighbourhood search, max 1.96 ulp for the fp32 Horner evaluation).
constexpr float kC1 = 0x1.fffff6p-1f;   // 0.999999702
constexpr float kC2 = 0x1.fffddap-2f;   // 0.499991804
constexpr float kC3 = 0x1.555a30p-3f;   // 0.166675925
constexpr float kC4 = 0x1.5738e8p-5f;   // 0.0418972522
constexpr float kC5 = 0x1.1000a8p-7f;   // 0.00830085948

// Canonical decomposition of a row (reading G8): blocks of kBlockElems elements,
// groups of kGroupBlocks blocks.  These, not the grid size, fix every rounding.
constexpr int kBlockElems = 16384;
constexpr int kGroupBlocks = 64;
constexpr int kThreads = 256;                     // one CTA processes one block
constexpr int kPerThread = kBlockElems / kThreads;  // 64 elements per thread per block

struct Pair {
    float m;  // "mantissa" m = e^t, in [sqrt(2)/2, sqrt(2)] for a single element
    float n;  // exponent, an integer held in a float, or -inf for the identity
};

__device__ __forceinline__ Pair pair_identity() { return Pair{0.0f, -__int_as_float(0x7f800000)}; }

// ----------------------------------------------------------------------------- L0
// 2^k for integer-valued k <= 1, flushed to +0 for k < -126 (reading G5),
// and for k = -inf or NaN (identity merges, reading G6): fmaxf drops NaN.
__device__ __forceinline__ float pow2_flush(float k) {
    const float kc = fmaxf(k, -127.0f);
    const float b = __fadd_rn(kc, kMagic + 127.0f);  // low mantissa bits hold kc + 127 in [0, 128]
    return __int_as_float(__float_as_int(b) << 23);   // -> exponent field; kc = -127 -> +0.0
}

// ExtExp: Alg. 4 without the reconstruction step.
__device__ __forceinline__ Pair ext_exp(float x) {
    x = fminf(fmaxf(x, -kXClamp), kXClamp);           // reading G11 (NaN -> -2^21, G14)
    const float v = __fmaf_rn(x, kLog2e, kMagic);
    const float n = __fsub_rn(v, kMagic);             // n = round(x log2 e)
    float t = __fmaf_rn(n, -kLn2Hi, x);               // t = x - n ln2, Cody-Waite
    t = __fmaf_rn(n, -kLn2Lo, t);
    float p = __fmaf_rn(kC5, t, kC4);                 // Horner with FMA
    p = __fmaf_rn(p, t, kC3);
    p = __fmaf_rn(p, t, kC2);
    p = __fmaf_rn(p, t, kC1);
    const float m = __fmaf_rn(p, t, 1.0f);
    return Pair{m, n};
}

// Exp with reconstruction for the Three-Pass comparators (Alg. 4),
// argument d = x - mu <= 0 (PAPER.md:258 footnote); s = 2^n or 0 below -126 (reading G5).
__device__ __forceinline__ float exp_flush(float d) {
    d = fmaxf(d, -kXClamp);
    const float v = __fmaf_rn(d, kLog2e, kMagic);
    const float n = __fsub_rn(v, kMagic);
    float t = __fmaf_rn(n, -kLn2Hi, d);
    t = __fmaf_rn(n, -kLn2Lo, t);
    float p = __fmaf_rn(kC5, t, kC4);
    p = __fmaf_rn(p, t, kC3);
    p = __fmaf_rn(p, t, kC2);
    p = __fmaf_rn(p, t, kC1);
    p = __fmaf_rn(p, t, 1.0f);
    return __fmul_rn(p, pow2_flush(n));              // y = p * s
}

// ----------------------------------------------------------------------------- L1
// (m_a, n_a) + (m_b, n_b) with max-exponent rescaling (Alg. 3 update):
// neither side is ever scaled up.  Both products are exact scalings, so
// the result is one rounding of the exact sum.  Always called as merge(left, right).
__device__ __forceinline__ Pair pair_merge(Pair a, Pair b) {
    const float n = fmaxf(a.n, b.n);
    const float sa = pow2_flush(__fsub_rn(a.n, n));
    const float sb = pow2_flush(__fsub_rn(b.n, n));
    return Pair{__fmaf_rn(a.m, sa, __fmul_rn(b.m, sb)), n};
}

// Accumulate V element pairs into acc, one max and one rescale per vector (Alg. 3 lines
// PAPER.md:160-162 applied to a vector): n_max over the vector and acc, acc scaled by
// 2^(n_acc - n_max), then each m_j 2^(n_j - n_max) added in order with one FMA.
template <int V>
__device__ __forceinline__ void pair_accumulate(Pair& acc, const float (&m)[V], const float (&n)[V]) {
    float nmax = acc.n;
#pragma unroll
    for (int j = 0; j < V; ++j) nmax = fmaxf(nmax, n[j]);
    float s = __fmul_rn(acc.m, pow2_flush(__fsub_rn(acc.n, nmax)));
#pragma unroll
    for (int j = 0; j < V; ++j) s = __fmaf_rn(m[j], pow2_flush(__fsub_rn(n[j], nmax)), s);
    acc.m = s;
    acc.n = nmax;
}

// ----------------------------------------------------------------------------- CTA trees
// Perfect binary tree over the CTA's kThreads values in thread order (left = lower index).
// Padding leaves are identities, and merge(a, identity) == a bit for bit, so a perfect tree
// over a zero-padded power-of-two array equals the canonical "largest power of two < n"
// split tree of n leaves (reading G8).  Result valid in thread 0.
__device__ __forceinline__ Pair cta_tree_pairs(Pair v, Pair* smem /* >= kThreads/32 */) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        Pair r;
        r.m = __shfl_down_sync(0xffffffffu, v.m, o);
        r.n = __shfl_down_sync(0xffffffffu, v.n, o);
        if ((lane & (2 * o - 1)) == 0) v = pair_merge(v, r);
    }
    if (lane == 0) smem[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        constexpr int NW = kThreads / 32;
        Pair w[NW];
#pragma unroll
        for (int i = 0; i < NW; ++i) w[i] = smem[i];
#pragma unroll
        for (int o = 1; o < NW; o <<= 1)
#pragma unroll
            for (int i = 0; i + o < NW; i += 2 * o) w[i] = pair_merge(w[i], w[i + o]);
        v = w[0];
    }
    __syncthreads();
    return v;
}

__device__ __forceinline__ float cta_tree_sum(float v, float* smem) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const float r = __shfl_down_sync(0xffffffffu, v, o);
        if ((lane & (2 * o - 1)) == 0) v = __fadd_rn(v, r);
    }
    if (lane == 0) smem[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        constexpr int NW = kThreads / 32;
        float w[NW];
#pragma unroll
        for (int i = 0; i < NW; ++i) w[i] = smem[i];
#pragma unroll
        for (int o = 1; o < NW; o <<= 1)
#pragma unroll
            for (int i = 0; i + o < NW; i += 2 * o) w[i] = __fadd_rn(w[i], w[i + o]);
        v = w[0];
    }
    __syncthreads();
    return v;
}

__device__ __forceinline__ float cta_max(float v, float* smem) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) smem[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < kThreads / 32; ++i) v = fmaxf(v, smem[i]);
    }
    __syncthreads();
    return v;
}

// Sequential perfect tree over `c` (power of two) consecutive leaves, via a binary-counter
// stack: leaf i is pushed, then while the two top nodes cover equal-size ranges they are
// merged (left = deeper in the stack).  Equals the perfect tree over those leaves.
template <typename LeafFn>
__device__ __forceinline__ Pair seq_tree_pairs(int c, LeafFn leaf) {
    Pair st[24];
    int sz[24];
    int top = 0;
    for (int i = 0; i < c; ++i) {
        Pair v = leaf(i);
        int s = 1;
        while (top > 0 && sz[top - 1] == s) {
            v = pair_merge(st[top - 1], v);
            s *= 2;
            --top;
        }
        st[top] = v;
        sz[top] = s;
        ++top;
    }
    return st[0];
}

template <typename LeafFn>
__device__ __forceinline__ float seq_tree_sum(int c, LeafFn leaf) {
    float st[24];
    int sz[24];
    int top = 0;
    for (int i = 0; i < c; ++i) {
        float v = leaf(i);
        int s = 1;
        while (top > 0 && sz[top - 1] == s) {
            v = __fadd_rn(st[top - 1], v);
            s *= 2;
            --top;
        }
        st[top] = v;
        sz[top] = s;
        ++top;
    }
    return st[0];
}

__host__ __device__ __forceinline__ int64_t next_pow2(int64_t v) {
    int64_t p = 1;
    while (p < v) p <<= 1;
    return p;
}

// Canonical tree over n leaves, computed by the whole CTA: the leaves are padded to a
// power of two P; thread t reduces leaves [t*c, (t+1)*c) with c = max(1, P / kThreads),
// then cta_tree_pairs combines the thread results in order.  Valid in thread 0.
template <typename LeafFn>
__device__ __forceinline__ Pair cta_canonical_tree(int64_t n, LeafFn leaf, Pair* smem) {
    const int64_t P = next_pow2(n);
    const int64_t c = P > kThreads ? P / kThreads : 1;
    const int64_t base = (int64_t)threadIdx.x * c;
    Pair v = pair_identity();
    if (base < n) {
        v = seq_tree_pairs((int)c, [&](int i) {
            const int64_t j = base + i;
            return j < n ? leaf(j) : pair_identity();
        });
    }
    return cta_tree_pairs(v, smem);
}

template <typename LeafFn>
__device__ __forceinline__ float cta_canonical_sum(int64_t n, LeafFn leaf, float* smem) {
    const int64_t P = next_pow2(n);
    const int64_t c = P > kThreads ? P / kThreads : 1;
    const int64_t base = (int64_t)threadIdx.x * c;
    float v = 0.0f;
    if (base < n) {
        v = seq_tree_sum((int)c, [&](int i) {
            const int64_t j = base + i;
            return j < n ? leaf(j) : 0.0f;
        });
    }
    return cta_tree_sum(v, smem);
}

// ----------------------------------------------------------------------------- memory ops
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// streaming (evict-first) 128-bit store of outputs that are not re-read
__device__ __forceinline__ void st_cs_f4(float* p, float4 v) { __stcs(reinterpret_cast<float4*>(p), v); }

// bf16 bits -> fp32: exact 16-bit left shift
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

}  // namespace tp
