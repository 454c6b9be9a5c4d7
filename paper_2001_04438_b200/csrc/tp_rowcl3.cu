// Row-cluster schedule for the Three-Pass comparators (Alg. 1 Recompute; Alg. 2
// Reload) on rows of 2..256 blocks: the schedule the Two-Pass uses for such
// rows (tp_rowcl.cu), so that the comparison is algorithm against algorithm on one footing.
//
// One thread-block cluster of CL CTAs per row; CTA q owns blocks [lo, lo + n) of each of its rows
// (shares rotate over the cluster's CTAs as in tp_rowcl.cu).  A producer thread streams the
// CTA's blocks through a ring of bulk copies, pass by pass: the max pass forwards (from HBM,
// kept in L2), the exp-sum pass backwards and the output pass forwards (the most recently read
// blocks first: L2), the passes of consecutive rows interleaved (below) so that the exchanges
// complete behind other work.  The 16 compute warps run the stream kernel's per-block
// operations; after the max and the exp-sum pass, warp 0 stores the CTA's block values into
// every cluster CTA's shared memory and arrives on their exchange barrier; before the pass that
// needs them, every warp forms the row value with the canonical tree (blocks -> groups of 64 ->
// row: the stream kernel's reductions) and the statistics.  Reload's pass 3 re-reads y (written
// by the same threads in pass 2) from memory.
// Bit-identical to the stream-kernel comparators (tested).
#include "tp_ops.cuh"

namespace tp {

constexpr int kCl3Threads = kThreads + 32;  // 16 compute warps + the producer warp
constexpr int kCl3MaxLocal = 32;            // blocks per CTA per row
constexpr int kCl3MaxNb = 256;              // blocks per row

template <typename In> struct Cl3Ring { static constexpr int S = 3; };     // 3 x 64 KB fp32
template <> struct Cl3Ring<uint16_t> { static constexpr int S = 6; };       // 6 x 32 KB bf16

__device__ __forceinline__ void cl3_share(int nb, int CL, int r, int* lo, int* n) {
    *lo = (r * nb) / CL;
    *n = ((r + 1) * nb) / CL - *lo;
}

__device__ __forceinline__ bool cl3_wait(uint64_t* bar, uint32_t parity, unsigned* err, unsigned bit) {
    if (mbar_try_parity_cluster(bar, parity)) return true;
    const unsigned long long t0 = globaltimer_ns();
    for (unsigned i = 1;; ++i) {
        if (mbar_try_parity_cluster(bar, parity)) return true;
        if ((i & 63u) == 0) {
            if (aborted(err)) return false;
            if (globaltimer_ns() - t0 > kWaitTimeoutNs) {
                raise_abort(err, bit);
                return false;
            }
        }
    }
}

template <typename In, int A>
__global__ void __launch_bounds__(kCl3Threads, 1) rowcl3_kernel(const KArgs a, int CL) {
    constexpr int V = InTraits<In>::V;
    constexpr int S = Cl3Ring<In>::S;
    extern __shared__ __align__(128) unsigned char dsm[];
    In* stages = reinterpret_cast<In*>(dsm);
    __shared__ __align__(8) uint64_t full_bar[S];
    __shared__ __align__(8) uint64_t empty_bar[S];
    __shared__ __align__(8) uint64_t xbar[2];                // exchange barriers, by exchange parity
    __shared__ float partv[kCl3MaxLocal][kWarps];            // per local block, per warp
    __shared__ __align__(8) float2 rowvals[2][kCl3MaxNb];    // the row's block values, by parity
    __shared__ float2 gvals[kCl3MaxNb / kGroupBlocks];
    __shared__ float4 s_st;

    publish_abort_word(a);
    WsHeader* hdr = reinterpret_cast<WsHeader*>(a.ws);
    unsigned* err = &hdr->error;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = (int)cluster_ctarank();
    const int64_t cid = cluster_id_x(), ncl = nclusters_x();
    const int nb = (int)a.nb;
    const int64_t K = a.rows > cid ? (a.rows - 1 - cid) / ncl + 1 : 0;  // rows of this cluster
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], kWarps);
        }
        mbar_init(&xbar[0], CL);
        mbar_init(&xbar[1], CL);
        fence_mbar_init();
    }
    cluster_sync_all();  // every CTA's barriers exist before any remote arrival

    if (warp == kWarps) {
        // =============================================================== producer
        if (lane != 0) return;
        const In* x = static_cast<const In*>(a.x);
        long long seq = 0;
        for (int64_t k = 0; k < K; ++k) {
            const int64_t row = cid + k * ncl;
            int lo, n;
            cl3_share(nb, CL, (int)((q + k) % CL), &lo, &n);
            for (int phase = 0; phase < 3; ++phase) {
                for (int t = 0; t < n; ++t, ++seq) {
                    const int li = phase == 1 ? n - 1 - t : t;
                    const int st = (int)(seq % S);
                    if (seq >= S && !wait_or_abort(&empty_bar[st], (uint32_t)(((seq / S) - 1) & 1), err, 64u)) return;
                    if (A == kReload && phase == 2) {  // pass 3 reads Y, not X: no copy
                        mbar_arrive(&full_bar[st]);
                        continue;
                    }
                    const int64_t e0 = (int64_t)(lo + li) * kBlockElems;
                    const uint32_t bytes = (uint32_t)min((int64_t)kBlockElems, a.cols - e0) * (uint32_t)sizeof(In);
                    fence_proxy_async_smem();
                    mbar_arrive_expect_tx(&full_bar[st], bytes);
                    tma_load_1d(stages + (size_t)st * kBlockElems, x + row * a.cols + e0, bytes, &full_bar[st],
                                phase < 2 ? policy_evict_last() : policy_evict_first());
                }
            }
        }
        return;
    }

    // =================================================================== compute warps
    long long seq = 0;
    unsigned xc = 0;
    bool ok = true;
    for (int64_t k = 0; k < K && ok; ++k) {
        const int64_t row = cid + k * ncl;
        int lo, n;
        cl3_share(nb, CL, (int)((q + k) % CL), &lo, &n);
        float mu = 0.0f;
        float4 st = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int phase = 0; phase < 3 && ok; ++phase) {
            for (int t = 0; t < n; ++t, ++seq) {
                const int li = phase == 1 ? n - 1 - t : t;
                const int64_t e0 = (int64_t)(lo + li) * kBlockElems;
                const int valid = (int)min((int64_t)kBlockElems, a.cols - e0);
                const int sg = (int)(seq % S);
                if (!wait_or_abort(&full_bar[sg], (uint32_t)((seq / S) & 1), err, 4u)) {
                    ok = false;
                    break;
                }
                BlockVals v;
                if (!(A == kReload && phase == 2)) load_stage<In>(stages + (size_t)sg * kBlockElems, v);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty_bar[sg]);
                float* yb = a.y + row * a.cols + e0;
                if (phase == 0) {  // max, as op_max
                    const float m = warp_max(valid == kBlockElems ? max_thread<V, true>(v, valid)
                                                                  : max_thread<V, false>(v, valid));
                    if (lane == 0) partv[li][warp] = m;
                } else if (phase == 1) {  // sum of exp(x - mu) (and Reload's y = exp(x - mu)), as op_expsum
                    float s = valid == kBlockElems ? exp_sum_thread<V, true>(v, valid, mu)
                                                   : exp_sum_thread<V, false>(v, valid, mu);
                    if (A == kReload) store_block<V>(yb, valid, true, v);
                    s = warp_tree_sum(s);
                    if (lane == 0) partv[li][warp] = s;
                } else if (A == kRecompute) {
                    op_out_recompute<V>(v, st, yb, valid, true);
                } else {
                    op_out_reload(st, yb, valid, true);
                }
            }
            if (!ok || phase == 2) break;
            // ---- exchange: block values to every CTA, then the row value (canonical trees)
            asm volatile("bar.sync 1, %0;" ::"r"(kThreads) : "memory");  // partv complete (compute warps)
            const int par = (int)(xc & 1u);
            if (warp == 0) {
                if (lane < n) {
                    float bv;
                    if (phase == 0) {
                        bv = partv[lane][0];
                        for (int w = 1; w < kWarps; ++w) bv = fmaxf(bv, partv[lane][w]);
                    } else {
                        float tt[kWarps];
                        for (int w = 0; w < kWarps; ++w) tt[w] = partv[lane][w];
                        bv = block_tree_warps_sum(tt);
                    }
                    const uint32_t dst = smem_u32(&rowvals[par][lo + lane]);
                    for (int r = 0; r < CL; ++r) st_cluster_f2(mapa(dst, (uint32_t)r), make_float2(bv, 0.0f));
                }
                __syncwarp();
                if (lane < CL) mbar_arrive_remote(mapa(smem_u32(&xbar[par]), (uint32_t)lane));
            }
            if (!cl3_wait(&xbar[par], (xc >> 1) & 1u, err, 4096u)) {
                ok = false;
                break;
            }
            ++xc;
            if (warp == 0) {
                const int kind = phase == 0 ? kRedMax : kRedSum;
                const int ng = (nb + kGroupBlocks - 1) / kGroupBlocks;
                for (int g = 0; g < ng; ++g) {  // blocks -> groups of 64 (stream kernel retire path)
                    const int gs = min(kGroupBlocks, nb - g * kGroupBlocks);
                    const float2* gv = &rowvals[par][g * kGroupBlocks];
                    const float2 r = warp_reduce_leaves(kind, gs, [&](int64_t j) { return gv[j]; });
                    const float rx = __shfl_sync(0xffffffffu, r.x, 0);
                    if (lane == 0) gvals[g] = make_float2(rx, 0.0f);
                }
                __syncwarp();
                const float2 root = warp_reduce_leaves(kind, ng, [&](int64_t j) { return gvals[j]; });
                if (lane == 0) s_st = row_stats_of<A>(phase, make_float2(root.x, 0.0f), mu);
            }
            asm volatile("bar.sync 1, %0;" ::"r"(kThreads) : "memory");  // s_st ready; y stores ordered
            st = s_st;
            if (phase == 0) mu = st.x;
        }
    }
}

// ---- bf16 rows: rowcl3p_kernel, the same per-block operations, trees and exchanges in a software
// pipeline over a CTA's rows: for k = 0..K the max pass of row k (forwards), the output pass of row
// k - 1 (forwards: the blocks its exp-sum pass read last come first, from L2), the exp-sum pass of
// row k (backwards).  Each exchange then completes behind a whole pass of another row instead of
// stalling the CTA, and every warp forms the row value itself (no CTA barrier): C4 bf16 Recompute
// 483 -> 452 us, Reload 654 -> 601.  fp32 rows keep rowcl3_kernel: two rows in flight per cluster
// cost fp32 C4 L2 misses (Recompute 467 -> 506 us pipelined, 484 with this kernel's barrier-free
// exchanges in the sequential order).
// Pass `step` of iteration k of a CTA: returns the row iteration and sets the phase (0 max,
// 1 exp-sum, 2 output).
__device__ __forceinline__ int64_t cl3_step(int64_t k, int step, int* phase) {
    *phase = step == 0 ? 0 : step == 1 ? 2 : 1;
    return *phase == 2 ? k - 1 : k;
}

template <typename In, int A>
__global__ void __launch_bounds__(kCl3Threads, 1) rowcl3p_kernel(const KArgs a, int CL) {
    constexpr int V = InTraits<In>::V;
    constexpr int S = Cl3Ring<In>::S;
    extern __shared__ __align__(128) unsigned char dsm[];
    In* stages = reinterpret_cast<In*>(dsm);
    __shared__ __align__(8) uint64_t full_bar[S];
    __shared__ __align__(8) uint64_t empty_bar[S];
    __shared__ __align__(8) uint64_t xbar[4];                // exchange e: xbar[e & 3], count CL
    __shared__ __align__(8) uint64_t pdone[2];               // a pass's warp values written (count 16)
    __shared__ float partv[2][kCl3MaxLocal][kWarps];         // [max pass, exp-sum pass][local block][warp]
    __shared__ __align__(8) float2 rowvals[4][kCl3MaxNb];    // the row's block values of exchange e & 3
    __shared__ float2 gvals[kWarps][kCl3MaxNb / kGroupBlocks];  // per warp: its group values

    publish_abort_word(a);
    WsHeader* hdr = reinterpret_cast<WsHeader*>(a.ws);
    unsigned* err = &hdr->error;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = (int)cluster_ctarank();
    const int64_t cid = cluster_id_x(), ncl = nclusters_x();
    const int nb = (int)a.nb;
    const int64_t K = a.rows > cid ? (a.rows - 1 - cid) / ncl + 1 : 0;  // rows of this cluster
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], kWarps);
        }
        for (int i = 0; i < 4; ++i) mbar_init(&xbar[i], CL);
        for (int i = 0; i < 2; ++i) mbar_init(&pdone[i], kWarps);
        fence_mbar_init();
    }
    cluster_sync_all();  // every CTA's barriers exist before any remote arrival

    // Order of a CTA's passes (cl3_step): exchange 2k (the max of row k) is awaited at the start
    // of row k's exp-sum pass, exchange 2k + 1 (its sum) at the start of its output pass.
    // Buffers by e & 3: a CTA pushes exchange e + 4 only after every CTA pushed e + 3, which each
    // does after awaiting e (in both orders a CTA awaits e before it pushes e + 1).
    if (warp == kWarps) {
        // =============================================================== producer
        if (lane != 0) return;
        const In* x = static_cast<const In*>(a.x);
        long long seq = 0;
        for (int64_t k = 0; k <= K; ++k) {
            for (int step = 0; step < 3; ++step) {
                int phase;
                const int64_t kr = cl3_step(k, step, &phase);
                if (kr < 0 || kr >= K) continue;
                const int64_t row = cid + kr * ncl;
                int lo, n;
                cl3_share(nb, CL, (int)((q + kr) % CL), &lo, &n);
                for (int t = 0; t < n; ++t, ++seq) {
                    const int li = phase == 1 ? n - 1 - t : t;
                    const int st = (int)(seq % S);
                    if (seq >= S && !wait_or_abort(&empty_bar[st], (uint32_t)(((seq / S) - 1) & 1), err, 64u)) return;
                    if (A == kReload && phase == 2) {  // pass 3 reads Y, not X: no copy
                        mbar_arrive(&full_bar[st]);
                        continue;
                    }
                    const int64_t e0 = (int64_t)(lo + li) * kBlockElems;
                    const uint32_t bytes = (uint32_t)min((int64_t)kBlockElems, a.cols - e0) * (uint32_t)sizeof(In);
                    mbar_arrive_expect_tx(&full_bar[st], bytes);
                    tma_load_1d(stages + (size_t)st * kBlockElems, x + row * a.cols + e0, bytes, &full_bar[st],
                                phase < 2 ? policy_evict_last() : policy_evict_first());
                }
            }
        }
        return;
    }

    // =================================================================== compute warps
    long long seq = 0;
    bool ok = true;
    float mu = 0.0f;                                  // row k's max (exchange 2k)
    float4 st_out = make_float4(0.f, 0.f, 0.f, 0.f);  // row k - 1's (mu, 1 / sigma) (exchange 2k - 1)
    // await exchange e and form the row value with the canonical trees (blocks -> groups of 64 ->
    // row, the stream kernel's reductions), every warp on its own: no CTA barrier
    auto consume = [&](long long e, int phase, float mu_row) -> float4 {
        if (!cl3_wait(&xbar[e & 3], (uint32_t)((e >> 2) & 1), err, 4096u)) return make_float4(0.f, 0.f, -1.f, 0.f);
        const float2* rv = rowvals[e & 3];
        const int kind = phase == 0 ? kRedMax : kRedSum;
        const int ng = (nb + kGroupBlocks - 1) / kGroupBlocks;
        for (int g = 0; g < ng; ++g) {
            const int gs = min(kGroupBlocks, nb - g * kGroupBlocks);
            const float2* gv = rv + g * kGroupBlocks;
            const float2 r = warp_reduce_leaves(kind, gs, [&](int64_t j) { return gv[j]; });
            const float rx = __shfl_sync(0xffffffffu, r.x, 0);
            if (lane == 0) gvals[warp][g] = make_float2(rx, 0.0f);
        }
        __syncwarp();
        const float2 root = warp_reduce_leaves(kind, ng, [&](int64_t j) { return gvals[warp][j]; });
        const float rx = __shfl_sync(0xffffffffu, root.x, 0);
        __syncwarp();
        float4 r = row_stats_of<A>(phase, make_float2(rx, 0.0f), mu_row);
        r.w = 0.0f;
        return r;
    };
    // after a pass of row k: warp 0 sends the CTA's block values (exchange e) once every warp has
    // written its values (pdone), the other warps go on
    auto push = [&](long long e, int phase, int lo, int n) -> bool {
        __syncwarp();
        if (lane == 0) mbar_arrive(&pdone[phase]);
        if (warp != 0) return true;
        if (!wait_or_abort(&pdone[phase], (uint32_t)((e >> 1) & 1), err, 4096u)) return false;
        if (lane < n) {
            float bv;
            if (phase == 0) {
                bv = partv[0][lane][0];
                for (int w = 1; w < kWarps; ++w) bv = fmaxf(bv, partv[0][lane][w]);
            } else {
                float tt[kWarps];
                for (int w = 0; w < kWarps; ++w) tt[w] = partv[1][lane][w];
                bv = block_tree_warps_sum(tt);
            }
            const uint32_t dst = smem_u32(&rowvals[e & 3][lo + lane]);
            for (int r = 0; r < CL; ++r) st_cluster_f2(mapa(dst, (uint32_t)r), make_float2(bv, 0.0f));
        }
        asm volatile("fence.acq_rel.cluster;" ::: "memory");
        __syncwarp();
        if (lane < CL) mbar_arrive_remote(mapa(smem_u32(&xbar[e & 3]), (uint32_t)lane));
        return true;
    };
    for (int64_t k = 0; k <= K && ok; ++k) {
        for (int step = 0; step < 3 && ok; ++step) {
            int phase;
            const int64_t kr = cl3_step(k, step, &phase);
            if (kr < 0 || kr >= K) continue;
            const int64_t row = cid + kr * ncl;
            int lo, n;
            cl3_share(nb, CL, (int)((q + kr) % CL), &lo, &n);
            if (phase == 1) {  // row k's max
                const float4 r = consume(2 * kr, 0, 0.0f);
                if (r.z < 0.0f) { ok = false; break; }
                mu = r.x;
            } else if (phase == 2) {  // row k - 1's (mu, 1 / sigma)
                st_out = consume(2 * kr + 1, 1, mu);  // mu: still row k - 1's (updated by sum(k) below)
                if (st_out.z < 0.0f) { ok = false; break; }
            }
            for (int t = 0; t < n; ++t, ++seq) {
                const int li = phase == 1 ? n - 1 - t : t;
                const int64_t e0 = (int64_t)(lo + li) * kBlockElems;
                const int valid = (int)min((int64_t)kBlockElems, a.cols - e0);
                const int sg = (int)(seq % S);
                if (!wait_or_abort(&full_bar[sg], (uint32_t)((seq / S) & 1), err, 4u)) {
                    ok = false;
                    break;
                }
                BlockVals v;
                if (!(A == kReload && phase == 2)) load_stage<In>(stages + (size_t)sg * kBlockElems, v);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty_bar[sg]);
                float* yb = a.y + row * a.cols + e0;
                if (phase == 0) {  // max, as op_max
                    const float m = warp_max(valid == kBlockElems ? max_thread<V, true>(v, valid)
                                                                  : max_thread<V, false>(v, valid));
                    if (lane == 0) partv[0][li][warp] = m;
                } else if (phase == 1) {  // sum of exp(x - mu) (and Reload's y = exp(x - mu)), as op_expsum
                    float s = valid == kBlockElems ? exp_sum_thread<V, true>(v, valid, mu)
                                                   : exp_sum_thread<V, false>(v, valid, mu);
                    if (A == kReload) store_block<V>(yb, valid, true, v);
                    s = warp_tree_sum(s);
                    if (lane == 0) partv[1][li][warp] = s;
                } else if (A == kRecompute) {
                    op_out_recompute<V>(v, st_out, yb, valid, true);
                } else {
                    op_out_reload(st_out, yb, valid, true);
                }
            }
            if (!ok) break;
            if (phase == 0 && !push(2 * kr, 0, lo, n)) ok = false;
            if (phase == 1 && !push(2 * kr + 1, 1, lo, n)) ok = false;
        }
    }
}

// the kernel of an input type: the pipelined one for bf16 rows
template <typename In, int A>
static auto rowcl3_kern() {
    if constexpr (sizeof(In) == 2) return rowcl3p_kernel<In, A>;
    else return rowcl3_kernel<In, A>;
}

static size_t rowcl3_dyn(int in_bytes) { return (size_t)(in_bytes == 4 ? 3 : 6) * kBlockElems * in_bytes; }

template <typename In, int A>
static int rowcl3_clusters(int dev, int CL) {
    static DevCache cache[kMaxDevices][5];
    const int ci = CL == 1 ? 0 : CL == 2 ? 1 : CL == 4 ? 2 : CL == 8 ? 3 : 4;
    if (const int c = cache[dev][ci].load(std::memory_order_relaxed)) return c > 0 ? c : 0;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(CL * 8));
    cfg.blockDim = dim3(kCl3Threads);
    cfg.dynamicSmemBytes = rowcl3_dyn(sizeof(In));
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, rowcl3_kern<In, A>(), &cfg) != cudaSuccess || n < 1) {
        cudaGetLastError();
        n = -1;
    }
    cache[dev][ci].store(n, std::memory_order_relaxed);
    return n > 0 ? n : 0;
}

template <typename In, int A>
cudaError_t launch_rowcl3(KArgs a, int CL, const LaunchOpts& o, cudaStream_t s) {
    if (a.nb < 2 || a.nb > kCl3MaxNb || CL < 1 || CL > 16 || CL > a.nb || (a.nb + CL - 1) / CL > kCl3MaxLocal)
        return cudaErrorNotSupported;
    int dev = 0;
    cudaGetDevice(&dev);
    static DevCache configured[kMaxDevices];
    if (!configured[dev].load(std::memory_order_acquire)) {
        cudaFuncSetAttribute(rowcl3_kern<In, A>(), cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)rowcl3_dyn(sizeof(In)));
        cudaFuncSetAttribute(rowcl3_kern<In, A>(), cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        configured[dev].store(1, std::memory_order_release);
    }
    int Q = rowcl3_clusters<In, A>(dev, CL);
    if (Q < 1) return cudaErrorNotSupported;
    if (o.grid_ctas > 0 && o.grid_ctas / CL < Q) Q = (int)(o.grid_ctas / CL > 0 ? o.grid_ctas / CL : 1);
    const int64_t ncl = a.rows < Q ? a.rows : Q;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(ncl * CL));
    cfg.blockDim = dim3(kCl3Threads);
    cfg.dynamicSmemBytes = rowcl3_dyn(sizeof(In));
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    last_plan() = Plan{3, A, ncl * CL, CL, 0, 0};
    return cudaLaunchKernelEx(&cfg, rowcl3_kern<In, A>(), a, CL);
}

template cudaError_t launch_rowcl3<float, kRecompute>(KArgs, int, const LaunchOpts&, cudaStream_t);
template cudaError_t launch_rowcl3<float, kReload>(KArgs, int, const LaunchOpts&, cudaStream_t);
template cudaError_t launch_rowcl3<uint16_t, kRecompute>(KArgs, int, const LaunchOpts&, cudaStream_t);
template cudaError_t launch_rowcl3<uint16_t, kReload>(KArgs, int, const LaunchOpts&, cudaStream_t);

}  // namespace tp
