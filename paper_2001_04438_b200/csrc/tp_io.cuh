// Block-level load / compute / store of the Two-Pass and Three-Pass kernels.
//
// A block is kBlockElems consecutive elements of one row (reading G8).  Thread t of the
// CTA owns the vectors j = t + kThreads*k (k = 0..NV-1) of V consecutive elements, so
// every warp-wide load is a coalesced 512-byte (fp32) or 512-byte (bf16, 8 per thread)
// transaction.  The per-thread element assignment is the same whether the row is 16-byte
// aligned (128-bit vector loads) or not (scalar loads), so results never depend on
// alignment.  A partial last block is masked element by element.
#pragma once
#include "tp_common.cuh"

namespace tp {

template <typename In> struct InTraits;
template <> struct InTraits<float> { static constexpr int V = 4; };
template <> struct InTraits<uint16_t> { static constexpr int V = 8; };

template <typename In>
struct BlockRegs {
    static constexpr int V = InTraits<In>::V;
    static constexpr int NV = kPerThread / V;
    float v[NV][V];
};

// Element offset (within the block) of element q of this thread's k-th vector.
template <int V>
__device__ __forceinline__ int elem_off(int k, int q) {
    return V * ((int)threadIdx.x + kThreads * k) + q;
}

// Load this thread's part of a block.  x_blk points at the block's first element;
// `valid` = number of real elements in the block (<= kBlockElems); `vec` = 16-byte aligned.
// Masked elements are left as 0 (callers mask by index).  `stream_hint` selects the
// evict-first L2 policy for a last read of the data.
template <typename In, bool FULL>
__device__ __forceinline__ void load_block(const In* x_blk, int valid, bool vec, bool last_read,
                                           BlockRegs<In>& r) {
    constexpr int V = InTraits<In>::V, NV = BlockRegs<In>::NV;
    if (vec && (FULL || valid == kBlockElems)) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int e = elem_off<V>(k, 0);
            if constexpr (V == 4) {
                const float4* p = reinterpret_cast<const float4*>(x_blk + e);
                const float4 a = last_read ? __ldcs(p) : __ldg(p);
                r.v[k][0] = a.x; r.v[k][1] = a.y; r.v[k][2] = a.z; r.v[k][3] = a.w;
            } else {
                const uint4* p = reinterpret_cast<const uint4*>(x_blk + e);
                const uint4 a = last_read ? __ldcs(p) : __ldg(p);
                r.v[k][0] = bf16_lo(a.x); r.v[k][1] = bf16_hi(a.x);
                r.v[k][2] = bf16_lo(a.y); r.v[k][3] = bf16_hi(a.y);
                r.v[k][4] = bf16_lo(a.z); r.v[k][5] = bf16_hi(a.z);
                r.v[k][6] = bf16_lo(a.w); r.v[k][7] = bf16_hi(a.w);
            }
        }
    } else if (vec) {
        // aligned partial block: whole vectors in range use vector loads, the straddling one scalars
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int e = elem_off<V>(k, 0);
            if (e + V <= valid) {
                if constexpr (V == 4) {
                    const float4 a = __ldg(reinterpret_cast<const float4*>(x_blk + e));
                    r.v[k][0] = a.x; r.v[k][1] = a.y; r.v[k][2] = a.z; r.v[k][3] = a.w;
                } else {
                    const uint4 a = __ldg(reinterpret_cast<const uint4*>(x_blk + e));
                    r.v[k][0] = bf16_lo(a.x); r.v[k][1] = bf16_hi(a.x);
                    r.v[k][2] = bf16_lo(a.y); r.v[k][3] = bf16_hi(a.y);
                    r.v[k][4] = bf16_lo(a.z); r.v[k][5] = bf16_hi(a.z);
                    r.v[k][6] = bf16_lo(a.w); r.v[k][7] = bf16_hi(a.w);
                }
            } else {
#pragma unroll
                for (int q = 0; q < V; ++q) {
                    float val = 0.0f;
                    if (e + q < valid) {
                        if constexpr (V == 4) val = __ldg(x_blk + e + q);
                        else val = __uint_as_float((uint32_t)__ldg(x_blk + e + q) << 16);
                    }
                    r.v[k][q] = val;
                }
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
#pragma unroll
            for (int q = 0; q < V; ++q) {
                const int e = elem_off<V>(k, q);
                float val = 0.0f;
                if (FULL || e < valid) {
                    if constexpr (V == 4) val = __ldg(x_blk + e);
                    else val = __uint_as_float((uint32_t)__ldg(x_blk + e) << 16);
                }
                r.v[k][q] = val;
            }
        }
    }
}

// Store this thread's outputs of a block (fp32 output for every input dtype).
template <typename In, bool FULL>
__device__ __forceinline__ void store_block(float* y_blk, int valid, bool vec, const BlockRegs<In>& r) {
    constexpr int V = InTraits<In>::V, NV = BlockRegs<In>::NV;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const int e = elem_off<V>(k, 0);
        if (vec && (FULL || e + V <= valid)) {
#pragma unroll
            for (int h = 0; h < V; h += 4)
                st_cs_f4(y_blk + e + h, make_float4(r.v[k][h], r.v[k][h + 1], r.v[k][h + 2], r.v[k][h + 3]));
        } else {
#pragma unroll
            for (int q = 0; q < V; ++q)
                if (FULL || e + q < valid) y_blk[e + q] = r.v[k][q];
        }
    }
}

// Pass 1 on registers: ExtExp of every element and the thread's pair accumulation
// (Alg. 3 lines PAPER.md:158-162), 8 elements per rescale; masked elements are identities.
template <typename In, bool FULL>
__device__ __forceinline__ Pair pass1_thread(const BlockRegs<In>& r, int valid) {
    constexpr int V = InTraits<In>::V, NV = BlockRegs<In>::NV;
    constexpr int G = 8 / V;  // vectors per accumulation group
    Pair acc = pair_identity();
#pragma unroll
    for (int k = 0; k < NV; k += G) {
        float m[8], n[8];
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
            for (int q = 0; q < V; ++q) {
                Pair e = ext_exp(r.v[k + g][q]);
                if (!FULL && !(elem_off<V>(k + g, q) < valid)) e = pair_identity();
                m[g * V + q] = e.m;
                n[g * V + q] = e.n;
            }
        pair_accumulate<8>(acc, m, n);
    }
    return acc;
}

// Pass 2 on registers, in place: y = (m * lambda') * 2^(n - (n_sum - 1)) with
// lambda' = 0.5 / m_sum (PAPER.md:166-168 with reading G9: never form lambda * 2^k first).
template <typename In>
__device__ __forceinline__ void pass2_thread(BlockRegs<In>& r, float nsum1, float lam_half) {
    constexpr int V = InTraits<In>::V, NV = BlockRegs<In>::NV;
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
        for (int q = 0; q < V; ++q) {
            const Pair e = ext_exp(r.v[k][q]);
            r.v[k][q] = __fmul_rn(__fmul_rn(e.m, lam_half), pow2_flush(__fsub_rn(e.n, nsum1)));
        }
}

// ---- Three-Pass helpers (Alg. 1/2)
template <typename In, bool FULL>
__device__ __forceinline__ float max_thread(const BlockRegs<In>& r, int valid) {
    constexpr int V = InTraits<In>::V, NV = BlockRegs<In>::NV;
    float mx = -__int_as_float(0x7f800000);
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
        for (int q = 0; q < V; ++q)
            if (FULL || elem_off<V>(k, q) < valid) mx = fmaxf(mx, r.v[k][q]);
    return mx;
}

// e_i = Exp(x_i - mu) in place, returns the thread's sum of the e_i in element order.
template <typename In, bool FULL>
__device__ __forceinline__ float exp_sum_thread(BlockRegs<In>& r, int valid, float mu) {
    constexpr int V = InTraits<In>::V, NV = BlockRegs<In>::NV;
    float s = 0.0f;
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
        for (int q = 0; q < V; ++q) {
            float e = exp_flush(__fsub_rn(r.v[k][q], mu));
            if (!FULL && !(elem_off<V>(k, q) < valid)) e = 0.0f;
            r.v[k][q] = e;
            s = __fadd_rn(s, e);
        }
    return s;
}

template <typename In>
__device__ __forceinline__ void scale_thread(BlockRegs<In>& r, float lam) {
    constexpr int V = InTraits<In>::V, NV = BlockRegs<In>::NV;
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
        for (int q = 0; q < V; ++q) r.v[k][q] = __fmul_rn(lam, r.v[k][q]);
}

// Coherent (L2) load of fp32 data written earlier in the same kernel (Reload's Y).
__device__ __forceinline__ void load_block_y(const float* y_blk, int valid, bool vec, BlockRegs<float>& r) {
    constexpr int NV = BlockRegs<float>::NV;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const int e = elem_off<4>(k, 0);
        if (vec && e + 4 <= valid) {
            const float4 a = __ldcg(reinterpret_cast<const float4*>(y_blk + e));
            r.v[k][0] = a.x; r.v[k][1] = a.y; r.v[k][2] = a.z; r.v[k][3] = a.w;
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) r.v[k][q] = (e + q < valid) ? __ldcg(y_blk + e + q) : 0.0f;
        }
    }
}

}  // namespace tp
