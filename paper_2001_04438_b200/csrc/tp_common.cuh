// Device building blocks of the Two-Pass softmax (arXiv 2001.04438) for sm_100a.
//
//   L0  ext_exp2 / exp_flush2 / pow2 (MUFU.EX2)   PAPER.md:139-149 (§4), Alg. 4 PAPER.md:234-263 (§6.3)
//   L1  pair_merge, vector accumulate, CTA trees   Alg. 3 PAPER.md:153-170 (§4)
//
// Readings of the paper taken here are listed in DESIGN.md ("Readings"), ids G1..G25 as in
// SURVEY.md §8(c).  All arithmetic is IEEE round-to-nearest fp32 written with explicit
// intrinsics / PTX (fma.rn.f32x2 packs two independent lanes into one FFMA2 instruction and is
// bit-identical to two scalar fma.rn), so results are fixed by the source, not by the compiler.
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
// product x*log2e whenever |x*log2e| < 2^22.
constexpr float kMagic = 0x1.8p23f;
// Guaranteed-accuracy domain |x| <= 2^21 (reading G11).  Blocks whose extended exponent
// leaves [-kNLimit, kNLimit] (or whose mantissa is not finite) are recomputed with x clamped
// to [-2^21, 2^21]; inside the domain the clamp is the identity, so both paths agree bit for bit.
constexpr float kXClamp = 0x1.0p21f;
constexpr float kNLimit = 3025525.5f;             // > round(2^21 log2 e) = 3025525
// Degree-5 polynomial p(t) = 1 + t(c1 + t(c2 + t(c3 + t(c4 + t c5)))) for e^t on
// |t| <= ln2/2.  The paper's Sollya coefficients are not printed (reading G3);
// these come from tools/fit_exp_gpu.py: minimax in fp32-ulp units (linear program), rounded to
// binary32, then coordinate / pairwise binary32 searches graded on the GPU end to end.  Alg. 4's
// Exp is then within 1.90 ulp of e^x on every fp32 x in [ln FLT_MIN, 0] (exhaustive,
// tools/exp_accuracy.py; the paper's "under 2 ULP").
constexpr float kC1 = 0x1.ffffeep-1f;   // 0.99999946
constexpr float kC2 = 0x1.fffdc6p-2f;   // 0.4999915
constexpr float kC3 = 0x1.555d92p-3f;   // 0.16668238
constexpr float kC4 = 0x1.573998p-5f;   // 0.04189758
constexpr float kC5 = 0x1.0e8b38p-7f;   // 0.008256342

// Canonical decomposition of a row (reading G8): blocks of kBlockElems elements,
// groups of kGroupBlocks blocks.  These, not the grid size, fix every rounding.
constexpr int kBlockElems = 16384;
constexpr int kGroupBlocks = 64;
constexpr int kThreads = 512;                       // one CTA processes one block
constexpr int kPerThread = kBlockElems / kThreads;  // 32 elements per thread per block
constexpr float kFltMax = 3.40282347e38f;

struct Pair {
    float m;  // "mantissa" m = e^t, in [sqrt(2)/2, sqrt(2)] for a single element
    float n;  // exponent, an integer held in a float, or -inf for the identity
};

__device__ __forceinline__ Pair pair_identity() { return Pair{0.0f, -__int_as_float(0x7f800000)}; }

// ----------------------------------------------------------------------------- f32x2 (FFMA2 / FADD2 / FMUL2)
__device__ __forceinline__ unsigned long long pk2(float2 a) { return *reinterpret_cast<unsigned long long*>(&a); }
__device__ __forceinline__ float2 upk2(unsigned long long a) { return *reinterpret_cast<float2*>(&a); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)), "l"(pk2(c)));
    return upk2(d);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)));
    return upk2(d);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)));
    return upk2(d);
}
__device__ __forceinline__ float2 bc2(float v) { return make_float2(v, v); }

// ----------------------------------------------------------------------------- L0
// 2^k for integer-valued k <= 1 by MUFU.EX2 (exact on integers; pinned by the exhaustive GPU
// unit test), flushed to +0 below 2^-126 by .ftz (reading G5); 2^-inf = 0.
__device__ __forceinline__ float ex2_ftz(float k) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(k));
    return r;
}

// The same function for the tree merges, NaN-safe: k = NaN (identity + identity) gives 0
// (reading G6).  Exponent-field construction: fmaxf drops NaN, kc + 127 lands in the low
// mantissa bits of kc + 1.5*2^23 + 127 and is shifted into the exponent field.
__device__ __forceinline__ float pow2_flush(float k) {
    const float kc = fmaxf(k, -127.0f);
    const float b = __fadd_rn(kc, kMagic + 127.0f);
    return __int_as_float(__float_as_int(b) << 23);
}

// ExtExp of two elements: Alg. 4 without the reconstruction step.
template <bool CLAMP>
__device__ __forceinline__ void ext_exp2(float2 x, float2& m, float2& n) {
    if (CLAMP) {  // reading G11 (NaN -> -2^21, reading G14)
        x.x = fminf(fmaxf(x.x, -kXClamp), kXClamp);
        x.y = fminf(fmaxf(x.y, -kXClamp), kXClamp);
    }
    const float2 v = ffma2(x, bc2(kLog2e), bc2(kMagic));
    n = fadd2(v, bc2(-kMagic));                        // n = round(x log2 e)
    float2 t = ffma2(n, bc2(-kLn2Hi), x);              // t = x - n ln2, Cody-Waite
    t = ffma2(n, bc2(-kLn2Lo), t);
    float2 p = ffma2(bc2(kC5), t, bc2(kC4));           // Horner with FMA
    p = ffma2(p, t, bc2(kC3));
    p = ffma2(p, t, bc2(kC2));
    p = ffma2(p, t, bc2(kC1));
    m = ffma2(p, t, bc2(1.0f));
}

// The same, also returning v = x log2e + 1.5*2^23 (the rounding sum): for |n| < 2^22 its bits
// are bits(1.5*2^23) + n, so 2^(n - c) can be built with integer operations (pow2_bits).
template <bool CLAMP>
__device__ __forceinline__ void ext_exp2v(float2 x, float2& m, float2& v) {
    if (CLAMP) {
        x.x = fminf(fmaxf(x.x, -kXClamp), kXClamp);
        x.y = fminf(fmaxf(x.y, -kXClamp), kXClamp);
    }
    v = ffma2(x, bc2(kLog2e), bc2(kMagic));
    const float2 n = fadd2(v, bc2(-kMagic));
    float2 t = ffma2(n, bc2(-kLn2Hi), x);
    t = ffma2(n, bc2(-kLn2Lo), t);
    float2 p = ffma2(bc2(kC5), t, bc2(kC4));
    p = ffma2(p, t, bc2(kC3));
    p = ffma2(p, t, bc2(kC2));
    p = ffma2(p, t, bc2(kC1));
    m = ffma2(p, t, bc2(1.0f));
}

// 2^(d - 127) for an integer d <= 255, flushed to +0 for d <= 0: the value ex2_ftz gives for the
// integer exponent d - 127 (reading G5), built in the exponent field on the integer pipe
// (no MUFU): max, shift.  With d = bits(v) - c this is 2^(n - (c - bits(1.5*2^23) + 127)).
__device__ __forceinline__ float pow2_bits(int d) {
    // funnel shift: SHF on the integer pipe (a plain << compiles to IMAD.SHL on the FMA pipe)
    return __int_as_float((int)__funnelshift_l(0u, (unsigned)max(d, 0), 23));
}
__device__ __forceinline__ int magic_bits() { return __float_as_int(kMagic); }

// Exp with reconstruction for the Three-Pass comparators (Alg. 4), argument
// d = x - mu <= 0 (PAPER.md:258 footnote): y = p * s, s = 2^n or 0 below 2^-126 (reading G5).
__device__ __forceinline__ float2 exp_flush2(float2 d) {
    d.x = fmaxf(d.x, -kXClamp);
    d.y = fmaxf(d.y, -kXClamp);
    float2 m, n;
    ext_exp2<false>(d, m, n);
    return fmul2(m, make_float2(ex2_ftz(n.x), ex2_ftz(n.y)));
}

// Scalar ExtExp (unit-test hook and the rare scalar paths): the same arithmetic as ext_exp2.
__device__ __forceinline__ Pair ext_exp(float x) {
    float2 m, n;
    ext_exp2<true>(make_float2(x, x), m, n);
    return Pair{m.x, n.x};
}

// ----------------------------------------------------------------------------- L1
// (m_a, n_a) + (m_b, n_b) with max-exponent rescaling (Alg. 3 update):
// neither side is ever scaled up.  Both products are exact scalings, so the
// result is one rounding of the exact sum.  Always called as merge(left, right).
__device__ __forceinline__ Pair pair_merge(Pair a, Pair b) {
    const float n = fmaxf(a.n, b.n);
    const float sa = pow2_flush(__fsub_rn(a.n, n));
    const float sb = pow2_flush(__fsub_rn(b.n, n));
    return Pair{__fmaf_rn(a.m, sa, __fmul_rn(b.m, sb)), n};
}

// Thread accumulator: two mantissa lanes sharing one exponent (Alg. 3's (m_sum, n_sum),
// PAPER.md:155-162, kept as two partial sums for FFMA2).  n starts at -FLT_MAX (not -inf) so
// that n - n_max is never -inf - (-inf); a thread with no element keeps m = 0, which merges
// like the identity.
struct Acc {
    float2 m;
    float n;
};
__device__ __forceinline__ Acc acc_init() { return Acc{make_float2(0.0f, 0.0f), -kFltMax}; }

// Accumulate 8 element pairs (4 float2): one max and one rescale per group of 8, then
// m_j 2^(n_j - n_max) added with one FFMA2 per two elements (Alg. 3 lines PAPER.md:160-162).
__device__ __forceinline__ void acc_add8(Acc& acc, const float2 (&m)[4], const float2 (&n)[4]) {
    float nmax = acc.n;
#pragma unroll
    for (int j = 0; j < 4; ++j) nmax = fmaxf(nmax, fmaxf(n[j].x, n[j].y));
    const float sa = ex2_ftz(__fsub_rn(acc.n, nmax));
    float2 s = fmul2(acc.m, bc2(sa));
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const float2 k = fadd2(n[j], bc2(-nmax));
        s = ffma2(m[j], make_float2(ex2_ftz(k.x), ex2_ftz(k.y)), s);
    }
    acc.m = s;
    acc.n = nmax;
}

__device__ __forceinline__ Pair acc_pair(const Acc& a) { return Pair{__fadd_rn(a.m.x, a.m.y), a.n}; }

// The same accumulator keyed by vb = bits of the rounding sum v of its exponent (ext_exp2v;
// 0 = no element yet).  acc_add8v computes exactly what acc_add8 computes (the scales are the
// same powers of two, flushed below 2^-126 alike) with the scales built on the integer pipe.
struct AccV {
    float2 m;
    int vb;
};
__device__ __forceinline__ AccV accv_init() { return AccV{make_float2(0.0f, 0.0f), 0}; }

__device__ __forceinline__ void acc_add8v(AccV& acc, const float2 (&m)[4], const float2 (&v)[4]) {
    float vmax = __int_as_float(acc.vb);  // v >= 2^22 > 0 for every element: float order = bits order
#pragma unroll
    for (int j = 0; j < 4; ++j) vmax = fmaxf(vmax, fmaxf(v[j].x, v[j].y));
    const int c = __float_as_int(vmax) - 127;  // pow2_bits(bits(v_i) - c) = 2^(n_i - n_max)
    float2 s = fmul2(acc.m, bc2(pow2_bits(acc.vb - c)));
#pragma unroll
    for (int j = 0; j < 4; ++j)
        s = ffma2(m[j], make_float2(pow2_bits(__float_as_int(v[j].x) - c), pow2_bits(__float_as_int(v[j].y) - c)), s);
    acc.m = s;
    acc.vb = __float_as_int(vmax);
}

// (m, n) of the accumulator; no element -> (0, -FLT_MAX) as acc_init.
__device__ __forceinline__ Pair accv_pair(const AccV& a) {
    const float n = a.vb ? __fsub_rn(__int_as_float(a.vb), kMagic) : -kFltMax;
    return Pair{__fadd_rn(a.m.x, a.m.y), n};
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

// The same perfect tree over N (power of two, compile time) leaves, fully unrolled: registers
// only, log2(N) levels of independent merges.
template <int N, typename LeafFn>
__device__ __forceinline__ Pair tree_pairs_n(LeafFn leaf) {
    Pair t[N];
#pragma unroll
    for (int i = 0; i < N; ++i) t[i] = leaf(i);
#pragma unroll
    for (int o = 1; o < N; o <<= 1)
#pragma unroll
        for (int i = 0; i + o < N; i += 2 * o) t[i] = pair_merge(t[i], t[i + o]);
    return t[0];
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

// True when the block result needs the clamped recomputation (see kNLimit).
__device__ __forceinline__ bool pair_out_of_domain(Pair p) {
    return !(fabsf(p.m) <= kFltMax) || !(fabsf(p.n) <= kNLimit);
}

// ----------------------------------------------------------------------------- memory ops
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
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
#ifndef TP_STORE_MODE
#define TP_STORE_MODE 0
#endif
__device__ __forceinline__ void st_cs_f4(float* p, float4 v) {
#if TP_STORE_MODE == 0
    __stcs(reinterpret_cast<float4*>(p), v);
#elif TP_STORE_MODE == 1
    *reinterpret_cast<float4*>(p) = v;
#else
    asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
#endif
}

// 256-bit store of 8 consecutive floats (STG.E.ENL2.256 on sm_100a), evict-first
__device__ __forceinline__ void st_cs_f8(float* p, const float* v) {
    asm volatile("st.global.cs.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "f"(v[0]), "f"(v[1]), "f"(v[2]),
                 "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
}

// bf16 bits -> fp32: exact 16-bit left shift
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// ----------------------------------------------------------------------------- TMA bulk copies + mbarriers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ bool mbar_try_parity(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ bool mbar_test_parity(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// L2 policies for the bulk loads: keep pass-1 data for the re-read, drop last reads first.
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// global -> shared bulk copy (TMA, non-tensor), completion counted on the mbarrier
__device__ __forceinline__ void tma_load_1d(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar,
                                            uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(smem_dst)),
        "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// shared -> global bulk copy (TMA store), tracked by this thread's bulk async-groups
__device__ __forceinline__ void tma_store_1d(void* gmem_dst, const void* smem_src, uint32_t bytes, uint64_t policy) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gmem_dst),
                 "r"(smem_u32(smem_src)), "r"(bytes), "l"(policy)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// at most N of this thread's committed bulk groups still reading shared memory
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// global -> L2 bulk prefetch (no shared memory, no completion): starts the DRAM traffic of a
// block the CTA will stage later
__device__ __forceinline__ void bulk_prefetch_l2(const void* gmem_src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(gmem_src), "r"(bytes) : "memory");
}

__device__ __forceinline__ void tma_load_1d_nohint(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                                   uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(smem_dst)),
                 "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// ----------------------------------------------------------------------------- clusters / DSMEM
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t nclusters_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
    return r;
}
// shared::cta address -> the same variable's shared::cluster address in CTA `rank`
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster_f2(uint32_t addr, float2 v) {
    asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ bool mbar_try_parity_cluster(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Programmatic dependent launch: wait until the stream's previous grid has completed and its
// memory is visible (a no-op when the launch was not programmatic), then let the next grid on
// the stream be scheduled early (it waits the same way before touching memory).
__device__ __forceinline__ void pdl_wait_and_release() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// System-scope release store / acquire load (flags read by peer GPUs over NVLink).
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

}  // namespace tp
