// Block-level pieces of the Two-Pass and Three-Pass kernels: per-thread loads (shared-memory
// stage or global), per-thread pass computations, stores.
//
// A block is kBlockElems consecutive elements of one row (reading G8), in two contiguous halves
// of 8192 elements: threads 0-255 own the first half, 256-511 the second; within its half,
// thread t owns the vectors (t mod 256) + 256 k (k = 0..NV-1) of V consecutive elements (V = 4
// fp32, 8 bf16): every warp-wide access is a contiguous 512-byte segment, and a half block is
// one contiguous copy (the cluster kernel stages halves separately).  The per-thread element
// assignment, and therefore every rounding, is the same whatever the data source (TMA stage,
// 128-bit global loads, scalar loads of misaligned rows).  A partial last block is masked
// element by element.
#pragma once
#include "tp_common.cuh"

namespace tp {

// Offset of vector k of thread tid in the canonical block layout (above).
template <int V>
__device__ __forceinline__ int vec_off(int tid, int k) {
    return V * ((tid & 255) + 256 * k) + (tid >> 8) * (kBlockElems / 2);
}

template <typename In> struct InTraits;
template <> struct InTraits<float> { static constexpr int V = 4; };
template <> struct InTraits<uint16_t> { static constexpr int V = 8; };

// This thread's 32 values of a block; v[k*V + q] = element V*(t + kThreads*k) + q.
struct BlockVals {
    float v[kPerThread];
};

// Element offset of this thread's value i (= k*V + q).  `tid` is the thread's index in the
// block's canonical layout: threadIdx.x, unless a kernel runs one thread's share on another
// physical thread (tp_rowcl.cu's compute teams); the arithmetic depends only on tid.
template <int V>
__device__ __forceinline__ int elem_off(int i, int tid) {
    return vec_off<V>(tid, i / V) + (i % V);
}
template <int V>
__device__ __forceinline__ int elem_off(int i) {
    return elem_off<V>(i, (int)threadIdx.x);
}

__device__ __forceinline__ void unpack_bf16x8(uint4 a, float* d) {
    d[0] = bf16_lo(a.x); d[1] = bf16_hi(a.x); d[2] = bf16_lo(a.y); d[3] = bf16_hi(a.y);
    d[4] = bf16_lo(a.z); d[5] = bf16_hi(a.z); d[6] = bf16_lo(a.w); d[7] = bf16_hi(a.w);
}

// From a shared-memory stage holding the block (elements past `valid` are stale: callers mask).
template <typename In>
__device__ __forceinline__ void load_stage(const In* stage, BlockVals& r, int tid = (int)threadIdx.x) {
    constexpr int V = InTraits<In>::V, NV = kPerThread / V;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const int e = vec_off<V>(tid, k);
        if constexpr (V == 4) {
            const float4 a = *reinterpret_cast<const float4*>(stage + e);
            r.v[4 * k] = a.x; r.v[4 * k + 1] = a.y; r.v[4 * k + 2] = a.z; r.v[4 * k + 3] = a.w;
        } else {
            unpack_bf16x8(*reinterpret_cast<const uint4*>(stage + e), &r.v[8 * k]);
        }
    }
}

// This thread's values of logical warp (8 h + wl) from half-stage `half` (a half-stage holds one contiguous half of a block: the values of logical warps 8 h .. 8 h + 7).
template <typename In>
__device__ __forceinline__ void load_half(const In* half, int wl, int lane, BlockVals& r) {
    constexpr int V = InTraits<In>::V, NV = kPerThread / V;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const int e = vec_off<V>(32 * wl + lane, k);  // wl < 8: offset within the half
        if constexpr (V == 4) {
            const float4 a = *reinterpret_cast<const float4*>(half + e);
            r.v[4 * k] = a.x; r.v[4 * k + 1] = a.y; r.v[4 * k + 2] = a.z; r.v[4 * k + 3] = a.w;
        } else {
            unpack_bf16x8(*reinterpret_cast<const uint4*>(half + e), &r.v[8 * k]);
        }
    }
}

// From global memory.  `vec`: 16-byte aligned rows (128-bit loads); otherwise scalar loads.
// Elements past `valid` read as 0 (callers mask).  `last` = evict-first L2 policy.
template <typename In>
__device__ __forceinline__ void load_global(const In* xb, int valid, bool vec, bool last, BlockVals& r,
                                            int tid = (int)threadIdx.x) {
    constexpr int V = InTraits<In>::V, NV = kPerThread / V;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const int e = vec_off<V>(tid, k);
        if (vec && e + V <= valid) {
            if constexpr (V == 4) {
                const float4* p = reinterpret_cast<const float4*>(xb + e);
                const float4 a = last ? __ldcs(p) : __ldg(p);
                r.v[4 * k] = a.x; r.v[4 * k + 1] = a.y; r.v[4 * k + 2] = a.z; r.v[4 * k + 3] = a.w;
            } else {
                const uint4* p = reinterpret_cast<const uint4*>(xb + e);
                unpack_bf16x8(last ? __ldcs(p) : __ldg(p), &r.v[8 * k]);
            }
        } else {
#pragma unroll
            for (int q = 0; q < V; ++q) {
                float val = 0.0f;
                if (e + q < valid) {
                    if constexpr (V == 4) val = __ldg(xb + e + q);
                    else val = __uint_as_float((uint32_t)__ldg(xb + e + q) << 16);
                }
                r.v[k * V + q] = val;
            }
        }
    }
}

// Coherent loads of fp32 data written earlier in the same kernel (Reload's Y), fp32 layout.
__device__ __forceinline__ void load_global_y(const float* yb, int valid, bool vec, BlockVals& r) {
    constexpr int NV = kPerThread / 4;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const int e = vec_off<4>((int)threadIdx.x, k);
        if (vec && e + 4 <= valid) {
            const float4 a = __ldcg(reinterpret_cast<const float4*>(yb + e));
            r.v[4 * k] = a.x; r.v[4 * k + 1] = a.y; r.v[4 * k + 2] = a.z; r.v[4 * k + 3] = a.w;
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) r.v[4 * k + q] = (e + q < valid) ? __ldcg(yb + e + q) : 0.0f;
        }
    }
}

// Store this thread's outputs (fp32 for every input dtype), V-element layout of In.
template <int V>
__device__ __forceinline__ void store_block(float* yb, int valid, bool vec, const BlockVals& r,
                                            int tid = (int)threadIdx.x) {
    constexpr int NV = kPerThread / V;
    if (vec && valid == kBlockElems) {  // whole block: unconditional 128-bit stores
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int e = vec_off<V>(tid, k);
#pragma unroll
            for (int h = 0; h < V; h += 4)
                st_cs_f4(yb + e + h, make_float4(r.v[k * V + h], r.v[k * V + h + 1], r.v[k * V + h + 2],
                                                 r.v[k * V + h + 3]));
        }
        return;
    }
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const int e = vec_off<V>(tid, k);
        if (vec && e + V <= valid) {
#pragma unroll
            for (int h = 0; h < V; h += 4)
                st_cs_f4(yb + e + h, make_float4(r.v[k * V + h], r.v[k * V + h + 1], r.v[k * V + h + 2],
                                                 r.v[k * V + h + 3]));
        } else {
#pragma unroll
            for (int q = 0; q < V; ++q)
                if (e + q < valid) yb[e + q] = r.v[k * V + q];
        }
    }
}

// Pass 1 on this thread's values: ExtExp and the pair accumulation
// in 4 groups of 8 elements.  Masked elements are (m, n) = (0, -inf).
template <int V, bool FULL, bool CLAMP>
__device__ __forceinline__ Pair pass1_thread(const BlockVals& r, int valid, int tid = (int)threadIdx.x) {
    AccV acc = accv_init();
#pragma unroll
    for (int g = 0; g < kPerThread / 8; ++g) {
        // a partial block: this thread's later elements are all masked (element offsets grow
        // with the index), and a masked group adds exactly nothing: stop (short rows, tails)
        if (!FULL && !(elem_off<V>(8 * g, tid) < valid)) break;
        float2 m[4], v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            ext_exp2v<CLAMP>(make_float2(r.v[8 * g + 2 * j], r.v[8 * g + 2 * j + 1]), m[j], v[j]);
            if (!FULL) {  // masked: m = 0 with v = 0 (scale 0, never the max)
                if (!(elem_off<V>(8 * g + 2 * j, tid) < valid)) { m[j].x = 0.0f; v[j].x = 0.0f; }
                if (!(elem_off<V>(8 * g + 2 * j + 1, tid) < valid)) { m[j].y = 0.0f; v[j].y = 0.0f; }
            }
        }
        acc_add8v(acc, m, v);
    }
    return accv_pair(acc);
}

// Pass 2: y = (m * lambda') * 2^(n - (n_sum - 1)), lambda' = 0.5 / m_sum (PAPER.md:166-168 with
// reading G9: never form lambda * 2^k first).  m lambda' = lambda' p(t) is evaluated with the
// coefficients lambda' c_i (one rounding each, once per block): a multiply less per element, and
// p(0) lambda' = lambda' exactly.  2^(n - nsum1) = pow2_bits(bits(v) - c), flushed to 0 below
// 2^-126; |nsum1| <= 3025526 (reading G11) is exactly an int.
struct Pass2Consts {
    int c;
    float l1, l2, l3, l4, l5, l0;
};
__device__ __forceinline__ Pass2Consts pass2_consts(float nsum1, float lam_half) {
    return Pass2Consts{magic_bits() + __float2int_rn(nsum1) - 127, __fmul_rn(lam_half, kC1),
                       __fmul_rn(lam_half, kC2), __fmul_rn(lam_half, kC3), __fmul_rn(lam_half, kC4),
                       __fmul_rn(lam_half, kC5), lam_half};
}

template <bool CLAMP>
__device__ __forceinline__ float2 pass2_pair(float2 x, const Pass2Consts& k) {
    if (CLAMP) {
        x.x = fminf(fmaxf(x.x, -kXClamp), kXClamp);
        x.y = fminf(fmaxf(x.y, -kXClamp), kXClamp);
    }
    const float2 v = ffma2(x, bc2(kLog2e), bc2(kMagic));  // ExtExp
    const float2 n = fadd2(v, bc2(-kMagic));
    float2 t = ffma2(n, bc2(-kLn2Hi), x);
    t = ffma2(n, bc2(-kLn2Lo), t);
    float2 p = ffma2(bc2(k.l5), t, bc2(k.l4));
    p = ffma2(p, t, bc2(k.l3));
    p = ffma2(p, t, bc2(k.l2));
    p = ffma2(p, t, bc2(k.l1));
    p = ffma2(p, t, bc2(k.l0));
    const float2 s = make_float2(pow2_bits(__float_as_int(v.x) - k.c), pow2_bits(__float_as_int(v.y) - k.c));
    return fmul2(p, s);
}

// In place on this thread's values (those at element offsets >= valid are left as they are:
// the caller stores only valid elements).
template <bool CLAMP, int V = 4>
__device__ __forceinline__ void pass2_thread(BlockVals& r, float nsum1, float lam_half, int valid = kBlockElems,
                                             int tid = (int)threadIdx.x) {
    const Pass2Consts k = pass2_consts(nsum1, lam_half);
#pragma unroll
    for (int i = 0; i < kPerThread; i += 2) {
        if (valid < kBlockElems && !(elem_off<V>(i, tid) < valid)) break;
        const float2 y = pass2_pair<CLAMP>(make_float2(r.v[i], r.v[i + 1]), k);
        r.v[i] = y.x;
        r.v[i + 1] = y.y;
    }
}

// Whole 16-byte aligned block: each vector's outputs stored as soon as they are computed, so
// the stores overlap the arithmetic of the next vectors.
template <int V, bool CLAMP>
__device__ __forceinline__ void pass2_store_full(const BlockVals& r, float nsum1, float lam_half, float* yb,
                                                 int tid = (int)threadIdx.x) {
    const Pass2Consts k = pass2_consts(nsum1, lam_half);
#pragma unroll
    for (int j = 0; j < kPerThread / V; ++j) {
        float o[V];
#pragma unroll
        for (int q = 0; q < V; q += 2) {
            const float2 y = pass2_pair<CLAMP>(make_float2(r.v[j * V + q], r.v[j * V + q + 1]), k);
            o[q] = y.x;
            o[q + 1] = y.y;
        }
        const int e = vec_off<V>(tid, j);
#pragma unroll
        for (int h = 0; h < V; h += 4) st_cs_f4(yb + e + h, make_float4(o[h], o[h + 1], o[h + 2], o[h + 3]));
    }
}

// ---- warp-level pass 1 with the out-of-domain fallback (reading G11)
// A lane is out of domain when its accumulator is not finite or its exponent leaves
// [-kNLimit, kNLimit]; then the whole warp recomputes its 32 x 32 values with x clamped to
// [-2^21, 2^21].  The clamp is the identity inside the domain, so the choice never changes an
// in-domain result; pass 2 of the same block applies the same per-warp choice (block mask).
__device__ __forceinline__ bool acc_out_of_domain(Pair p) {
    return !(fabsf(p.m) <= kFltMax) || !(fabsf(p.n) <= kNLimit);
}

// Tree over the 32 lanes of a warp in lane order (left = lower lane); result in lane 0.
__device__ __forceinline__ Pair warp_tree_pairs(Pair v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        Pair r;
        r.m = __shfl_down_sync(0xffffffffu, v.m, o);
        r.n = __shfl_down_sync(0xffffffffu, v.n, o);
        if ((lane & (2 * o - 1)) == 0) v = pair_merge(v, r);
    }
    return v;
}

__device__ __forceinline__ float warp_tree_sum(float v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const float r = __shfl_down_sync(0xffffffffu, v, o);
        if ((lane & (2 * o - 1)) == 0) v = __fadd_rn(v, r);
    }
    return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Perfect tree over the kThreads/32 warp pairs of a block, in warp order.
constexpr int kWarps = kThreads / 32;
__device__ __forceinline__ Pair block_tree_warps(const Pair* w) {
    Pair t[kWarps];
#pragma unroll
    for (int i = 0; i < kWarps; ++i) t[i] = w[i];
#pragma unroll
    for (int o = 1; o < kWarps; o <<= 1)
#pragma unroll
        for (int i = 0; i + o < kWarps; i += 2 * o) t[i] = pair_merge(t[i], t[i + o]);
    return t[0];
}
__device__ __forceinline__ float block_tree_warps_sum(const float* w) {
    float t[kWarps];
#pragma unroll
    for (int i = 0; i < kWarps; ++i) t[i] = w[i];
#pragma unroll
    for (int o = 1; o < kWarps; o <<= 1)
#pragma unroll
        for (int i = 0; i + o < kWarps; i += 2 * o) t[i] = __fadd_rn(t[i], t[i + o]);
    return t[0];
}

// ---- warp value of a block's thread pairs (reading G8): maximum first, then a sum tree.
// The 32 thread pairs (m_t, n_t) of a warp combine to (M, N): N = max_t n_t, M = the perfect
// binary tree of correctly rounded additions, in lane order, of m_t 2^(n_t - N) (exact power-of-two
// scalings, flushed to 0 below 2^-126 as every 2^k of the path, reading G5).  This is Alg. 3's
// max-exponent rescaling applied to the whole warp at once: where no scaled
// value is subnormal it is bit for bit the perfect tree of pair merges over the same leaves
// (scaling by 2^(n_node - N) commutes with each rounding), and it costs one integer max
// (REDUX) and a tree of additions instead of a tree of merges (shuffles of m and n, two 2^k per
// level).  Every kernel forms warp values with these functions, so all stay bit-identical.
//
// Key of a thread pair: the bits of n + 1.5*2^23, i.e. bits(1.5*2^23) + n for the integer n
// (|n| <= 3025526 after the clamp decision, reading G11), so keys order like exponents; 0 for a
// thread without elements (n = -FLT_MAX).
__device__ __forceinline__ int pair_key(Pair p) {
    return p.n > -4194304.0f ? __float_as_int(__fadd_rn(p.n, kMagic)) : 0;
}
// m 2^(n - N) for the warp's key kw (2^(key - kw), flushed to 0 for key - kw <= -127)
__device__ __forceinline__ float pair_scaled(Pair p, int key, int kw) {
    return __fmul_rn(p.m, pow2_bits(key - kw + 127));
}
// (M, N) from the sum and the warp's key; no element in the warp: (0, -FLT_MAX) like accv_pair
__device__ __forceinline__ Pair warp_value_pair(float msum, int kw) {
    return Pair{msum, kw ? __fsub_rn(__int_as_float(kw), kMagic) : -kFltMax};
}
// The warp value of this lane's thread pair and the 31 others; result in lane 0.
__device__ __forceinline__ Pair warp_value(Pair p) {
    const int key = pair_key(p);
    const int kw = (int)__reduce_max_sync(0xffffffffu, (unsigned)key);
    return warp_value_pair(warp_tree_sum(pair_scaled(p, key, kw)), kw);
}

// Pass 1 of this warp's share of a block: warp value in lane 0, returns the clamp decision.
template <int V>
__device__ __forceinline__ bool warp_pass1(const BlockVals& r, int valid, Pair* wp) {
    Pair acc = valid == kBlockElems ? pass1_thread<V, true, false>(r, valid) : pass1_thread<V, false, false>(r, valid);
    const bool clamped = __any_sync(0xffffffffu, acc_out_of_domain(acc));
    if (clamped) acc = pass1_thread<V, false, true>(r, valid);
    *wp = warp_value(acc);
    return clamped;
}

// The same without the warp tree: this thread's pair (after the warp's clamp decision, which
// *clamped receives); the tree is left to the caller (tp_rowcl.cu's tree warp).
template <int V>
__device__ __forceinline__ Pair thread_pass1(const BlockVals& r, int valid, bool* clamped, int tid = (int)threadIdx.x) {
    Pair acc = valid == kBlockElems ? pass1_thread<V, true, false>(r, valid, tid)
                                    : pass1_thread<V, false, false>(r, valid, tid);
    *clamped = __any_sync(0xffffffffu, acc_out_of_domain(acc));
    if (*clamped) acc = pass1_thread<V, false, true>(r, valid, tid);
    return acc;
}

// ---- Three-Pass helpers (Alg. 1/2)
template <int V, bool FULL>
__device__ __forceinline__ float max_thread(const BlockVals& r, int valid) {
    float mx = -__int_as_float(0x7f800000);
#pragma unroll
    for (int i = 0; i < kPerThread; ++i) {
        if (!FULL && !(elem_off<V>(i) < valid)) break;  // later elements are all masked
        mx = fmaxf(mx, r.v[i]);
    }
    return mx;
}

// e_i = Exp(x_i - mu) in place (Alg. 1 line PAPER.md:93 / Alg. 2), returns the
// thread's sum in element order (two lanes, then lane x + lane y).
template <int V, bool FULL>
__device__ __forceinline__ float exp_sum_thread(BlockVals& r, int valid, float mu) {
    float2 s = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int i = 0; i < kPerThread; i += 2) {
        if (!FULL && !(elem_off<V>(i) < valid)) break;  // later elements masked: + 0 exactly
        float2 e = exp_flush2(fadd2(make_float2(r.v[i], r.v[i + 1]), bc2(-mu)));
        if (!FULL) {
            if (!(elem_off<V>(i) < valid)) e.x = 0.0f;
            if (!(elem_off<V>(i + 1) < valid)) e.y = 0.0f;
        }
        r.v[i] = e.x;
        r.v[i + 1] = e.y;
        s = fadd2(s, e);
    }
    return __fadd_rn(s.x, s.y);
}

__device__ __forceinline__ void scale_thread(BlockVals& r, float lam) {
#pragma unroll
    for (int i = 0; i < kPerThread; i += 2) {
        const float2 y = fmul2(bc2(lam), make_float2(r.v[i], r.v[i + 1]));
        r.v[i] = y.x;
        r.v[i + 1] = y.y;
    }
}

}  // namespace tp
