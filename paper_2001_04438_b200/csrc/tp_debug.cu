// Unit-test kernels: expose the device building blocks (tp_common.cuh) element by element so
// tests can check them against the oracle's plain definitions and exact pair arithmetic.
#include "tp_block.cuh"
#include "tp_internal.h"

namespace tp {

__global__ void debug_kernel(int what, const float* a, const float* b, float* o0, float* o1, int64_t count) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (what == 8) {  // whole warps (count % 32 == 0, checked by the caller)
        if (i - (threadIdx.x & 31) >= count) return;
        const Pair p{a[2 * i], a[2 * i + 1]};
        const Pair wv = warp_value(p), pt = warp_tree_pairs(p);  // both valid in lane 0
        const int lane = threadIdx.x & 31;
        const float r[4] = {wv.m, wv.n, pt.m, pt.n};
        float mine = 0.0f;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float v = __shfl_sync(0xffffffffu, r[j], 0);
            if (lane == j) mine = v;
        }
        if (lane < 4) o0[i] = mine;
        return;
    }
    if (i >= count) return;
    switch (what) {
        case 0: {
            const Pair p = ext_exp(a[i]);
            o0[i] = p.m;
            o1[i] = p.n;
            break;
        }
        case 1: o0[i] = pow2_flush(a[i]); break;
        case 2: {
            const Pair p = pair_merge(Pair{a[2 * i], a[2 * i + 1]}, Pair{b[2 * i], b[2 * i + 1]});
            o0[i] = p.m;
            o1[i] = p.n;
            break;
        }
        case 3: o0[i] = exp_flush2(make_float2(a[i], a[i])).x; break;
        case 4: o0[i] = ex2_ftz(a[i]); break;
        case 5: reinterpret_cast<unsigned long long*>(o0)[i] = globaltimer_ns(); break;  // timeline marker
        case 6: {  // the hot path's ExtExp: ext_exp2v<false> (no clamp), n recovered from v
            float2 m, v;
            ext_exp2v<false>(make_float2(a[i], a[i]), m, v);
            o0[i] = m.x;
            o1[i] = __fsub_rn(v.x, kMagic);
            break;
        }
        case 7: o0[i] = pow2_bits(__float2int_rn(a[i])); break;  // the hot path's 2^(d - 127)
        default: break;
    }
}

// Compute-only throughput of the per-block operations (development / roofline evidence): each
// CTA of 512 threads runs `reps` times over one shared-memory block of synthetic logits:
// what = 0 pass 1 (ExtExp + pair accumulation + warp tree), 1 pass 2 (ExtExp + output
// scaling, no store), 2 both.  One value per CTA goes to `sink` so nothing is optimised away.
template <typename In>
__global__ void __launch_bounds__(kThreads, 1) bench_compute_kernel(int what, int reps, float* sink) {
    constexpr int V = InTraits<In>::V;
    extern __shared__ __align__(16) unsigned char dsm_probe[];
    In* blk = reinterpret_cast<In*>(dsm_probe);
    for (int i = threadIdx.x; i < kBlockElems; i += kThreads) {
        const float v = (float)((i * 7919 + blockIdx.x * 104729) % 20011) * 0.05f - 500.0f;
        if constexpr (sizeof(In) == 4) blk[i] = v;
        else blk[i] = (uint16_t)(__float_as_uint(v) >> 16);
    }
    __syncthreads();
    float acc = 0.0f;
    if (what >= 3 && what <= 6) {  // instruction throughput: 8 independent chains per thread, 64 ops per rep
        float2 c[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) c[j] = make_float2(blk[threadIdx.x + j], blk[threadIdx.x + 8 + j]);
        const float2 mul = make_float2(blk[5], blk[6]), add = make_float2(blk[7], blk[8]);
        for (int r = 0; r < reps; ++r) {
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (what == 3) c[j] = ffma2(c[j], mul, add);               // FFMA2 3-register
                    else if (what == 4) c[j] = ffma2(c[j], mul, bc2(0.5f));    // FFMA2 immediate addend
                    else if (what == 5) c[j].x = __fmaf_rn(c[j].x, mul.x, add.x);  // scalar FFMA
                    else c[j] = make_float2(__int_as_float(max(__float_as_int(c[j].x) - 3, 0) << 1), c[j].y);  // ALU
                }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) acc += c[j].x + c[j].y;
        if ((threadIdx.x & 31) == 0) sink[blockIdx.x * kWarps + (threadIdx.x >> 5)] = acc;
        return;
    }
    for (int r = 0; r < reps; ++r) {
        BlockVals v;
        load_stage<In>(blk, v);
        const float off = acc * 0.0f + (float)(r & 1);  // defeats hoisting the loop-invariant work
#pragma unroll
        for (int i = 0; i < kPerThread; i += 2) {
            const float2 t = fadd2(make_float2(v.v[i], v.v[i + 1]), bc2(off));
            v.v[i] = t.x;
            v.v[i + 1] = t.y;
        }
        if (what == 7) {  // pass 1 without the warp tree
            acc += pass1_thread<V, true, false>(v, kBlockElems).m;
            continue;
        }
        if (what == 10) {  // stores through shared memory: STS, then one 64 KB bulk (TMA) store
            float* yb = sink + (size_t)gridDim.x * kWarps + (size_t)blockIdx.x * kBlockElems;
            float* st = reinterpret_cast<float*>(blk);
            if (threadIdx.x == 0) bulk_wait_read<0>();
            __syncthreads();
#pragma unroll
            for (int j = 0; j < kPerThread / 4; ++j)
                *reinterpret_cast<float4*>(st + vec_off<4>((int)threadIdx.x, j)) =
                    make_float4(v.v[4 * j], v.v[4 * j + 1], v.v[4 * j + 2], v.v[4 * j + 3]);
            fence_proxy_async_smem();
            __syncthreads();
            if (threadIdx.x == 0) {
                tma_store_1d(yb, st, kBlockElems * 4, policy_evict_first());
                bulk_commit();
            }
            continue;
        }
        if (what == 11) {  // 256-bit stores (8 consecutive floats per thread per instruction)
            float* yb = sink + (size_t)gridDim.x * kWarps + (size_t)blockIdx.x * kBlockElems;
#pragma unroll
            for (int j = 0; j < kPerThread / 8; ++j) st_cs_f8(yb + vec_off<8>((int)threadIdx.x, j), &v.v[8 * j]);
            continue;
        }
        if (what == 8 || what == 9) {  // pass 2 with 128-bit evict-first stores to a per-CTA 64 KB buffer
            float* yb = sink + (size_t)gridDim.x * kWarps + (size_t)blockIdx.x * kBlockElems;
            if (what == 8) pass2_store_full<V, false>(v, acc * 1e-30f + 300.0f, 0.25f, yb);
            else {  // stores only
#pragma unroll
                for (int j = 0; j < kPerThread / 4; ++j)
                    st_cs_f4(yb + vec_off<4>((int)threadIdx.x, j),
                             make_float4(v.v[4 * j], v.v[4 * j + 1], v.v[4 * j + 2], v.v[4 * j + 3]));
            }
            continue;
        }
        if (what != 1) {
            Pair wp;
            warp_pass1<V>(v, kBlockElems, &wp);
            acc += wp.m;
        }
        if (what != 0) {
            pass2_thread<false>(v, acc * 1e-30f + 300.0f, 0.25f);
#pragma unroll
            for (int i = 0; i < kPerThread; ++i) acc += v.v[i];
        }
    }
    if (threadIdx.x == 0) bulk_wait<0>();
    if ((threadIdx.x & 31) == 0) sink[blockIdx.x * kWarps + (threadIdx.x >> 5)] = acc;
}

cudaError_t launch_bench_compute(int what, int in_bf16, int64_t ctas, int reps, float* sink, cudaStream_t s) {
    const int dyn = kBlockElems * (in_bf16 ? 2 : 4);
    if (in_bf16) {
        cudaFuncSetAttribute(bench_compute_kernel<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
        bench_compute_kernel<uint16_t><<<(unsigned)ctas, kThreads, dyn, s>>>(what, reps, sink);
    } else {
        cudaFuncSetAttribute(bench_compute_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
        bench_compute_kernel<float><<<(unsigned)ctas, kThreads, dyn, s>>>(what, reps, sink);
    }
    return cudaGetLastError();
}

// STREAM-style bandwidth baselines (measurement only, not part of the method):
// 0 copy y = x, 1 scale y = a x, 2 in-place scale x = a x, 3 read-only sum (one partial per
// CTA into y).  128-bit accesses, grid-stride, n a multiple of 4 and 16-byte aligned pointers.
__global__ void __launch_bounds__(512) stream_baseline_kernel(int what, float* x, float* y, int64_t n4, float a) {
    float4* x4 = reinterpret_cast<float4*>(x);
    float4* y4 = reinterpret_cast<float4*>(y);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    float s = 0.0f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += 4 * stride) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (i + u * stride < n4) v[u] = __ldcs(x4 + i + u * stride);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (i + u * stride >= n4) continue;
            if (what == 3) {
                s += (v[u].x + v[u].y) + (v[u].z + v[u].w);
                continue;
            }
            if (what != 0) v[u] = make_float4(a * v[u].x, a * v[u].y, a * v[u].z, a * v[u].w);
            __stcs((what == 2 ? x4 : y4) + i + u * stride, v[u]);
        }
    }
    if (what == 3) {
        __shared__ float red[16];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            float t = 0.0f;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
            y[blockIdx.x] = t;
        }
    }
}

// Read-only sum with U independent 128-bit loads in flight per thread (what 4: U = 8, 5: 16).
template <int U>
__global__ void __launch_bounds__(512) read_deep_kernel(const float* x, float* y, int64_t n4) {
    const float4* x4 = reinterpret_cast<const float4*>(x);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    float s = 0.0f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += U * stride) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = i + u * stride < n4 ? __ldcs(x4 + i + u * stride) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < U; ++u) s += (v[u].x + v[u].y) + (v[u].z + v[u].w);
    }
    if (s == 1.2345f) y[blockIdx.x] = s;  // keeps the loads alive
}

// Bulk-copy (TMA) read throughput: each CTA walks chunks blockIdx.x + k * gridDim.x of
// chunk_bytes through a ring of `stages` shared-memory buffers, one elected thread issuing; a
// chunk is re-issued as soon as the previous copy into its buffer has landed.
__global__ void read_tma_kernel(const char* x, int64_t nchunks, uint32_t chunk_bytes, int stages, float* y) {
    extern __shared__ __align__(128) unsigned char buf[];
    __shared__ __align__(8) uint64_t bar[32];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < stages; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
    int64_t c = blockIdx.x;
    int k = 0;
    for (; k < stages && c < nchunks; ++k, c += gridDim.x) {
        mbar_arrive_expect_tx(&bar[k], chunk_bytes);
        tma_load_1d_nohint(buf + (size_t)k * chunk_bytes, x + c * chunk_bytes, chunk_bytes, &bar[k]);
    }
    unsigned par = 0;
    for (int64_t j = 0;; ++j) {
        const int s = (int)(j % stages);
        if (blockIdx.x + j * gridDim.x >= nchunks) break;
        mbar_wait_parity(&bar[s], (par >> s) & 1u);
        par ^= 1u << s;
        if (c < nchunks) {
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&bar[s], chunk_bytes);
            tma_load_1d_nohint(buf + (size_t)s * chunk_bytes, x + c * chunk_bytes, chunk_bytes, &bar[s]);
            c += gridDim.x;
        }
    }
    if (buf[0] == 0xAB && buf[1] == 0xCD) y[blockIdx.x] = 1.0f;
}

cudaError_t launch_read_probe(const void* x, int64_t bytes, int64_t chunk_bytes, int stages, int64_t ctas, float* y,
                              cudaStream_t s) {
    const size_t dyn = (size_t)chunk_bytes * stages;
    cudaFuncSetAttribute(read_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    read_tma_kernel<<<(unsigned)ctas, 32, dyn, s>>>(static_cast<const char*>(x), bytes / chunk_bytes,
                                                   (uint32_t)chunk_bytes, stages, y);
    return cudaGetLastError();
}

// Copy probe (measurement only): y = x by bulk (TMA) copies both ways, one thread per CTA: chunk
// j lands in stage j mod stages, is stored from there with a bulk store, and the stage is reloaded
// once that store has read it.  backward != 0: a CTA walks its chunks in descending order.
__global__ void copy_tma_kernel(const char* x, char* y, int64_t nchunks, uint32_t chunk_bytes, int stages,
                                int backward) {
    extern __shared__ __align__(128) unsigned char buf[];
    __shared__ __align__(8) uint64_t bar[32];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < stages; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
    const int64_t mine = nchunks > blockIdx.x ? (nchunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    auto chunk = [&](int64_t j) -> int64_t {  // this CTA's j-th chunk
        const int64_t q = backward ? mine - 1 - j : j;
        return blockIdx.x + q * gridDim.x;
    };
    const uint64_t keep = policy_evict_first();
    for (int64_t j = 0; j < stages && j < mine; ++j) {
        mbar_arrive_expect_tx(&bar[j], chunk_bytes);
        tma_load_1d(buf + (size_t)j * chunk_bytes, x + chunk(j) * chunk_bytes, chunk_bytes, &bar[j], keep);
    }
    unsigned par = 0;
    for (int64_t j = 0; j < mine; ++j) {
        const int s = (int)(j % stages);
        mbar_wait_parity(&bar[s], (par >> s) & 1u);
        par ^= 1u << s;
        tma_store_1d(y + chunk(j) * chunk_bytes, buf + (size_t)s * chunk_bytes, chunk_bytes, keep);
        bulk_commit();
        if (j + stages < mine) {
            bulk_wait_read<0>();  // this stage's store has read shared memory
            mbar_arrive_expect_tx(&bar[s], chunk_bytes);
            tma_load_1d(buf + (size_t)s * chunk_bytes, x + chunk(j + stages) * chunk_bytes, chunk_bytes, &bar[s], keep);
        }
    }
    bulk_wait<0>();
}

cudaError_t launch_copy_probe(const void* x, void* y, int64_t bytes, int64_t chunk_bytes, int stages, int64_t ctas,
                              int backward, cudaStream_t s) {
    const size_t dyn = (size_t)chunk_bytes * stages;
    cudaFuncSetAttribute(copy_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    copy_tma_kernel<<<(unsigned)ctas, 32, dyn, s>>>(static_cast<const char*>(x), static_cast<char*>(y),
                                                   bytes / chunk_bytes, (uint32_t)chunk_bytes, stages, backward);
    return cudaGetLastError();
}

cudaError_t launch_stream_baseline(int what, float* x, float* y, int64_t n, float a, int64_t ctas, cudaStream_t s) {
    if (what == 4) read_deep_kernel<8><<<(unsigned)ctas, 512, 0, s>>>(x, y, n / 4);
    else if (what == 5) read_deep_kernel<16><<<(unsigned)ctas, 512, 0, s>>>(x, y, n / 4);
    else stream_baseline_kernel<<<(unsigned)ctas, 512, 0, s>>>(what, x, y, n / 4, a);
    return cudaGetLastError();
}

// Exhaustive accuracy sweeps: x = the fp32 with bit pattern bits0 + i.
// what 0: ExtExp -> (m, n); 1: Exp with reconstruction (Alg. 4) -> y.
__global__ void exp_sweep_kernel(int what, uint32_t bits0, int64_t count, float* o0, float* o1) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const float x = __uint_as_float(bits0 + (uint32_t)i);
    if (what == 0) {
        const Pair p = ext_exp(x);
        o0[i] = p.m;
        o1[i] = p.n;
    } else {
        o0[i] = exp_flush2(make_float2(x, x)).x;
    }
}

cudaError_t launch_exp_sweep(int what, uint32_t bits0, int64_t count, float* o0, float* o1, cudaStream_t s) {
    if (count <= 0) return cudaSuccess;
    exp_sweep_kernel<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(what, bits0, count, o0, o1);
    return cudaGetLastError();
}

// Coefficient search support (tools/fit_exp_gpu.py): the Exp of Alg. 4 with runtime
// coefficients c[0..4] = c1..c5 (same fp32 operations as exp_flush2), graded against the double
// exponential: max ulp (as float bits, atomicMax) and the count above 2 ulp over the inputs
// x = as_float(bits0 + i * stride), i < count.  Normal outputs only (x >= ln FLT_MIN).
__global__ void exp_fit_kernel(float c1, float c2, float c3, float c4, float c5, uint32_t bits0, int64_t count,
                               int stride, unsigned* max_bits, unsigned long long* n_over2) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    float err = 0.0f;
    if (i < count) {
        const float x = __uint_as_float(bits0 + (uint32_t)(i * stride));
        const float v = __fmaf_rn(x, kLog2e, kMagic);
        const float n = __fsub_rn(v, kMagic);
        float t = __fmaf_rn(n, -kLn2Hi, x);
        t = __fmaf_rn(n, -kLn2Lo, t);
        float p = __fmaf_rn(c5, t, c4);
        p = __fmaf_rn(p, t, c3);
        p = __fmaf_rn(p, t, c2);
        p = __fmaf_rn(p, t, c1);
        p = __fmaf_rn(p, t, 1.0f);
        const float y = __fmul_rn(p, pow2_bits(__float_as_int(v) - (magic_bits() - 127)));
        const double ref = exp((double)x);
        int e;
        frexp(ref, &e);  // ref = f 2^e, f in [0.5, 1): fp32 ulp = 2^(e - 24)
        err = (float)(fabs((double)y - ref) / ldexp(1.0, e - 24));
    }
    unsigned long long over = __ballot_sync(0xffffffffu, err > 2.0f);
    float m = err;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) {
        atomicMax(max_bits, __float_as_uint(m));
        if (over) atomicAdd(n_over2, (unsigned long long)__popc((unsigned)over));
    }
}

cudaError_t launch_exp_fit(const float* c, uint32_t bits0, int64_t count, int stride, unsigned* max_bits,
                           unsigned long long* n_over2, cudaStream_t s) {
    if (count <= 0) return cudaSuccess;
    exp_fit_kernel<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(c[0], c[1], c[2], c[3], c[4], bits0, count, stride,
                                                                   max_bits, n_over2);
    return cudaGetLastError();
}

cudaError_t launch_debug(int what, const float* a, const float* b, float* o0, float* o1, int64_t count,
                         cudaStream_t s) {
    if (count <= 0) return cudaSuccess;
    const int64_t grid = (count + 255) / 256;
    debug_kernel<<<(unsigned)grid, 256, 0, s>>>(what, a, b, o0, o1, count);
    return cudaGetLastError();
}

}  // namespace tp
