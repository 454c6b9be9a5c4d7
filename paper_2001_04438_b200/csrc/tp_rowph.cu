// Phase kernel: the Two-Pass softmax (Alg. 3) of a few very long rows (config
// 3: 2^26, config 5: 2^31 elements; and the chunks of a sharded row: partial / finish), where
// pass 2 of a row can start only after its whole pass 1 (lambda needs every
// element) and each pass must run at the HBM rate on its own.
//
// One CTA per SM, a static schedule (no work queue): CTA c owns the items c, c + G, c + 2G, ...
// of pass 1 (row-major (row, block)), then the same of pass 2 (each row's blocks backwards: the
// end of pass 1 is what L2 still holds).  Everyone knows the order, so there are no commands:
//
//   producer (1 thread)   streams every item of the CTA, pass 1 then pass 2, through a ring of S
//                         64 KB stages with one bulk (TMA) copy each, as soon as a stage frees;
//                         pass-2 blocks are prefetched while the row's statistics are pending
//   16 compute warps      pass 1: values to registers, stage released, the thread's (m, n) pair
//                          written to a tree slot; pass 2:
//                         once the row is released, y = (m lambda') 2^(n - n_sum + 1) stored
//   tree warp             the block value from the slot's 512 thread pairs (the canonical tree of
//                         every kernel: lanes of a warp, then warps; reading G8), then the grid
//                         combine through tickets (tp_ops.cuh retire_batch): group of 64 blocks,
//                         row; the row's statistics released with its epoch-tagged flag
//
// The per-block work is exactly the other kernels' (thread_pass1, the same trees, op_pass2), so
// outputs are bit-identical to them.  What changes is the cost per block: the compute warps do no
// shuffle tree and wait on nothing but their stage, and the producer does one copy per block.
//
// Deadlock freedom: every CTA issues all its pass-1 items before any pass-2 item, and pass 1
// waits on nothing outside the CTA, so every row's pass 1 completes once every CTA runs; the grid
// is one CTA per SM with the shared memory of one CTA per SM, so all CTAs are resident together
// (a launch that cannot be falls back to the stream kernel).  Every wait has the watchdog.
#include "tp_ops.cuh"

namespace tp {

constexpr int kPhCompute = kWarps;         // 16 compute warps
constexpr int kPhProducer = kWarps;        // warp 16
constexpr int kPhTree = kWarps + 1;        // warp 17
constexpr int kPhThreads = (kWarps + 2) * 32;
constexpr int kPhSlots = 4;                // thread-pair slots between the compute warps and the tree warp
constexpr int64_t kPhMaxRows = 8;          // Two-Pass: rows of one launch (pass 2 waits for whole rows)

template <typename In> struct PhRing { static constexpr int S = sizeof(In) == 4 ? 3 : 6; };  // 192 KB

// Item k of this CTA in phase `phase`: (row, blk) of the phase's row-major item list.
__device__ __forceinline__ Item ph_item(const KArgs& a, int phase, int64_t k) {
    const int64_t g = (int64_t)blockIdx.x + k * (int64_t)gridDim.x;
    Item it;
    it.phase = phase;
    it.row = g / a.nb;
    const int64_t b = g - it.row * a.nb;
    it.blk = phase == 0 ? b : a.nb - 1 - b;
    return it;
}

// Items of this CTA in one phase (rows * nb items over the grid).
__device__ __forceinline__ int64_t ph_count(const KArgs& a) {
    const int64_t n = a.rows * a.nb;
    return n > (int64_t)blockIdx.x ? (n - 1 - blockIdx.x) / gridDim.x + 1 : 0;
}

// The block value (one whole warp) from its 512 thread pairs, bit-identical to warp_tree_pairs
// over each warp's 32 lanes followed by block_tree_warps over the 16 warps: lane l builds the
// perfect tree over threads 16 l .. 16 l + 15 (warp l/2, half l%2: levels 1-4 of warp_tree_pairs),
// then level 5 pairs the halves, then the warp roots (even lanes) form block_tree_warps' tree.
// Result in lane 0.
__device__ __forceinline__ Pair ph_block_tree(const Pair* tp) {
    const int lane = threadIdx.x & 31;
    const float4* p = reinterpret_cast<const float4*>(tp + 16 * lane);
    Pair l[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const float4 q = p[i];
        l[2 * i] = Pair{q.x, q.y};
        l[2 * i + 1] = Pair{q.z, q.w};
    }
#pragma unroll
    for (int o = 1; o < 16; o <<= 1)
#pragma unroll
        for (int i = 0; i + o < 16; i += 2 * o) l[i] = pair_merge(l[i], l[i + o]);
    Pair v = l[0];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {  // o = 1: the warp's halves; 2..16: warps 1, 2, 4, 8 apart
        Pair r;
        r.m = __shfl_down_sync(0xffffffffu, v.m, o);
        r.n = __shfl_down_sync(0xffffffffu, v.n, o);
        if ((lane & (2 * o - 1)) == 0) v = pair_merge(v, r);
    }
    return v;
}

template <typename In, int A>
__global__ void __launch_bounds__(kPhThreads, 1) rowph_kernel(const KArgs a) {
    constexpr int V = InTraits<In>::V;
    constexpr int S = PhRing<In>::S;
    constexpr int T = kPhSlots;
    constexpr bool kPass1 = A == kTwoPass || A == kPartial;
    constexpr bool kPass2 = A == kTwoPass || A == kFinish;
    extern __shared__ __align__(128) unsigned char dsm[];
    __shared__ __align__(16) Pair tpairs[T][kThreads];
    __shared__ unsigned char cbits[T][kWarps];
    __shared__ __align__(8) uint64_t full_bar[S];
    __shared__ __align__(8) uint64_t empty_bar[S];
    __shared__ __align__(8) uint64_t tfull[T];
    __shared__ __align__(8) uint64_t tempty[T];
    __shared__ unsigned s_epoch;

    pdl_wait_and_release();  // programmatic launch: the previous grid on the stream is complete
    publish_abort_word(a);
    WsHeader* hdr = reinterpret_cast<WsHeader*>(a.ws);
    unsigned* err = &hdr->error;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    In* stages = reinterpret_cast<In*>(dsm);
    const int64_t n_items = ph_count(a);
    const int64_t n1 = kPass1 ? n_items : 0;           // pass-1 items of this CTA
    const int64_t n_all = n1 + (kPass2 ? n_items : 0);  // stage uses: pass 1 then pass 2

    if (threadIdx.x == 0) {
        s_epoch = *reinterpret_cast<volatile unsigned*>(&hdr->epoch);
        for (int s = 0; s < S; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], kPhCompute);
        }
        for (int t = 0; t < T; ++t) {
            mbar_init(&tfull[t], kPhCompute);
            mbar_init(&tempty[t], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const unsigned want = s_epoch + 1u;

    if (warp == kPhProducer) {
        // =============================================================== producer (lane 0)
        if (lane == 0) {
            const In* x = static_cast<const In*>(a.x);
            // pass-1 blocks of a Two-Pass / partial launch are re-read (pass 2 / the finish
            // launch): keep them in L2; pass-2 reads are the last
            const uint64_t pol_keep = policy_evict_last(), pol_drop = policy_evict_first();
            for (int64_t k = 0; k < n_all; ++k) {
                const int s = (int)(k % S);
                if (k >= S && !wait_or_abort(&empty_bar[s], (uint32_t)(((k / S) - 1) & 1), err, 64u)) break;
                const bool p1 = k < n1;
                const Item it = ph_item(a, p1 ? 0 : 1, p1 ? k : k - n1);
                const int64_t e0 = it.blk * kBlockElems;
                const uint32_t bytes = (uint32_t)min((int64_t)kBlockElems, a.cols - e0) * (uint32_t)sizeof(In);
                fence_proxy_async_smem();
                mbar_arrive_expect_tx(&full_bar[s], bytes);
                tma_load_1d(stages + (size_t)s * kBlockElems, x + it.row * a.cols + e0, bytes, &full_bar[s],
                            p1 ? pol_keep : pol_drop);
            }
        }
    } else if (warp == kPhTree) {
        // =============================================================== tree warp (pass 1)
        for (int64_t k = 0; k < n1;) {
            int n = 0;
            if (lane == 0) {
                if (wait_or_abort(&tfull[k % T], (uint32_t)((k / T) & 1), err, 32u)) {
                    n = 1;
                    while (n < T && k + n < n1 && mbar_test_parity(&tfull[(k + n) % T], (uint32_t)(((k + n) / T) & 1)))
                        ++n;
                }
            }
            n = __shfl_sync(0xffffffffu, n, 0);
            if (n == 0) break;  // aborted
            // the n blocks' values: lane j keeps block k + j's
            float2 val = make_float2(0.f, 0.f);
            unsigned mask = 0;
            for (int j = 0; j < n; ++j) {
                const int t = (int)((k + j) % T);
                const Pair bv = ph_block_tree(tpairs[t]);
                const unsigned cb = lane < kWarps ? (unsigned)cbits[t][lane] : 0u;
                const unsigned m = __ballot_sync(0xffffffffu, cb != 0) & ((1u << kWarps) - 1u);
                const float bm = __shfl_sync(0xffffffffu, bv.m, 0), bn = __shfl_sync(0xffffffffu, bv.n, 0);
                if (lane == j) {
                    val = make_float2(bm, bn);
                    mask = m;
                }
            }
            __syncwarp();
            if (lane < n) mbar_arrive(&tempty[(k + lane) % T]);  // the slots are free again
            const bool mine = lane < n;
            const Item it = ph_item(a, 0, k + (mine ? lane : 0));
            if (mine) {  // block_value's side effects: every block's clamp mask, the row's flag
                reinterpret_cast<unsigned*>(a.ws + a.lay.block_clamp)[it.row * a.nb + it.blk] = mask;
                if (mask) atomicOr(reinterpret_cast<unsigned*>(a.ws + a.lay.row_clamp) + it.row, 1u);
            }
            retire_batch<A == kFinish ? kTwoPass : A>(a, mine, it, val, 0.0f, want);
            k += n;
        }
    } else {
        // =============================================================== compute warps
        int64_t k = 0;
        bool ok = true;
        for (; k < n1 && ok; ++k) {  // pass 1
            const int s = (int)(k % S);
            const Item it = ph_item(a, 0, k);
            const int valid = (int)min((int64_t)kBlockElems, a.cols - it.blk * kBlockElems);
            if (!wait_or_abort(&full_bar[s], (uint32_t)((k / S) & 1), err, 4u)) {
                ok = false;
                break;
            }
            BlockVals v;
            load_stage<In>(stages + (size_t)s * kBlockElems, v);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[s]);  // the stage can be refilled
            bool clamped;
            const Pair tpr = thread_pass1<V>(v, valid, &clamped);
            const int t = (int)(k % T);
            if (k >= T && !wait_or_abort(&tempty[t], (uint32_t)(((k / T) - 1) & 1), err, 16u)) {
                ok = false;
                break;
            }
            tpairs[t][threadIdx.x] = tpr;
            if (lane == 0) cbits[t][warp] = clamped ? 1 : 0;
            __syncwarp();
            if (lane == 0) mbar_arrive(&tfull[t]);
        }
        if (kPass2 && ok) {
            const unsigned* row_ready = reinterpret_cast<const unsigned*>(a.ws + a.lay.row_ready);
            int64_t cur_row = -1;
            float4 st = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int64_t k2 = 0; k2 < n_items; ++k2, ++k) {  // pass 2
                const int s = (int)(k % S);
                const Item it = ph_item(a, 1, k2);
                if (it.row != cur_row) {  // the row's statistics (released once its pass 1 is done)
                    if (A == kFinish) {
                        st = finish_stats(a, it.row);
                    } else {
                        if (lane == 0 && !wait_flag(row_ready + it.row * 2, want, err)) ok = false;
                        ok = __shfl_sync(0xffffffffu, ok ? 1 : 0, 0) != 0;
                        if (!ok) break;
                        st = __ldcg(reinterpret_cast<const float4*>(a.ws + a.lay.row_stats) + it.row * 2);
                    }
                    cur_row = it.row;
                }
                const unsigned mask = A == kFinish ? finish_mask(a, st, it.row, it.blk)
                                                   : (st.z != 0.0f ? __ldcg(reinterpret_cast<const unsigned*>(
                                                                             a.ws + a.lay.block_clamp) +
                                                                         it.row * a.nb + it.blk)
                                                                   : 0u);
                const int valid = (int)min((int64_t)kBlockElems, a.cols - it.blk * kBlockElems);
                if (!wait_or_abort(&full_bar[s], (uint32_t)((k / S) & 1), err, 4u)) break;
                BlockVals v;
                load_stage<In>(stages + (size_t)s * kBlockElems, v);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty_bar[s]);
                op_pass2<V>(v, st, ((mask >> warp) & 1u) != 0, a.y + it.row * a.cols + it.blk * kBlockElems, valid,
                            true);
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) exit_and_reset(hdr);
}

template <typename In, int A>
cudaError_t launch_rowph(KArgs a, const LaunchOpts& o, cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    auto kern = rowph_kernel<In, A>;
    constexpr int S = PhRing<In>::S;
    const size_t dyn = (size_t)S * kBlockElems * sizeof(In);
    static DevCache configured[kMaxDevices];
    static DevCache resident[kMaxDevices];
    if (!configured[dev].load(std::memory_order_acquire)) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        int n = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kPhThreads, dyn) != cudaSuccess) {
            cudaGetLastError();
            n = 0;
        }
        resident[dev].store(n > 0 ? n : -1, std::memory_order_relaxed);
        configured[dev].store(1, std::memory_order_release);
    }
    if (resident[dev].load(std::memory_order_relaxed) < 1) return cudaErrorNotSupported;
    // one CTA per SM, all resident (the static schedule's pass 2 waits for every CTA's pass 1)
    int64_t grid = device_sms(dev);
    if (o.grid_ctas > 0 && o.grid_ctas < grid) grid = o.grid_ctas;
    if (grid > a.rows * a.nb) grid = a.rows * a.nb;
    a.total_items = a.rows * a.nb;
    last_plan() = Plan{5, A, grid, 0, 0, S};
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kPhThreads);
    cfg.dynamicSmemBytes = dyn;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

// Does the phase schedule apply (automatic choice)?  Rows long enough that every CTA gets many
// blocks of each pass, few enough that a Two-Pass launch's pass 2 waiting for whole rows costs
// nothing (the partial / finish launches have no such wait).
bool rowph_applies(int A, int64_t rows, int64_t nb, int sms) {
    if (A == kTwoPass && rows > kPhMaxRows) return false;
    return rows * nb >= 16 * (int64_t)sms;
}

#define TP_PH_INSTANTIATE(IN)                                                                  \
    template cudaError_t launch_rowph<IN, kTwoPass>(KArgs, const LaunchOpts&, cudaStream_t);   \
    template cudaError_t launch_rowph<IN, kPartial>(KArgs, const LaunchOpts&, cudaStream_t);   \
    template cudaError_t launch_rowph<IN, kFinish>(KArgs, const LaunchOpts&, cudaStream_t);
TP_PH_INSTANTIATE(float)
TP_PH_INSTANTIATE(uint16_t)

}  // namespace tp
