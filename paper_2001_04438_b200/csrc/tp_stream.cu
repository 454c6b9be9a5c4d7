// Warp-specialised persistent kernel for 16-byte aligned rows (the fast path of every entry
// point).  One CTA per SM, three roles:
//
//   16 compute warps   wait for a stage, copy their 32 x 32 values into registers and release
//                      the stage at once, run the item's operation (tp_ops.cuh), store outputs
//                      with 128-bit evict-first stores, and hand their per-warp results to the
//                      retire warp through a ring of part slots.  They never touch a global
//                      atomic or fence.
//   producer warp      takes items from the in-order work queue (chunks of 2, the next chunk's
//                      atomic in flight), starts a cp.async.bulk (TMA) copy of each item's block
//                      into a free stage with an L2 policy (evict_last for data pass 2 will
//                      re-read, evict_first for last reads), and supplies later-phase items with
//                      their row statistics as soon as the row's previous phase is released
//                      (polled, never blocking).
//   retire warp        publishes finished blocks in batches (one value per lane, one fence per
//                      batch) and runs the group / row reductions they complete (tp_ops.cuh).
//
// Ring of S stages, each holding one block (16384 elements; 3 x 64 KB fp32, 6 x 32 KB bf16):
//   full[s]   count 2: producer arrive.expect_tx at issue + producer arrive once the item's
//             statistics are in place (immediately for items that need none); + TMA bytes
//   empty[s]  count 16: each compute warp once its values are in registers
// Ring of R part slots (per item sequence number):
//   pfull[r]  count 16: each compute warp after writing its part
//   pempty[r] count 1: the retire warp after reading the slot
// Deadlock freedom: as in tp_kernels.cu.  In addition no role blocks on a row flag: the
// producer polls them while it waits for stages, and the retire warp never waits on anything
// but part slots, so a CTA always retires its oldest finished item.
#include "tp_ops.cuh"

namespace tp {

constexpr int kProducerWarp = kWarps;
constexpr int kRetireWarp = kWarps + 1;
constexpr int kStreamThreads = kThreads + 64;
constexpr int kPartSlots = 8;

template <typename In> struct Ring { static constexpr int S = 3; };   // 3 x 64 KB fp32
template <> struct Ring<uint16_t> { static constexpr int S = 6; };     // 6 x 32 KB bf16

struct StageMeta {
    long long item;
    Item it;
    int valid;
    int need;       // statistics still to be provided
    unsigned mask;  // pass 2: per-warp clamp decisions of pass 1
    float4 stats;
};

struct PartSlot {
    long long item;
    Item it;
    float mu;
    Part part;
};

template <typename In, int A>
// 18 warps: 5 on some SM sub-partitions, whose 16K-register files then allow 96 per thread.
__global__ void __launch_bounds__(kStreamThreads, 1) stream_kernel(const KArgs a) {
    constexpr int P = AlgoTraits<A>::P;
    constexpr int V = InTraits<In>::V;
    constexpr int S = Ring<In>::S;
    constexpr int R = kPartSlots;
    extern __shared__ __align__(128) unsigned char dsm[];
    __shared__ StageMeta meta[S];
    __shared__ PartSlot pslot[R];
    __shared__ __align__(8) uint64_t full_bar[S];
    __shared__ __align__(8) uint64_t empty_bar[S];
    __shared__ __align__(8) uint64_t pfull_bar[R];
    __shared__ __align__(8) uint64_t pempty_bar[R];
    __shared__ unsigned s_epoch;

    WsHeader* hdr = reinterpret_cast<WsHeader*>(a.ws);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    In* stages = reinterpret_cast<In*>(dsm);
    const long long total = a.total_items;

    if (threadIdx.x == kProducerWarp * 32) {
        s_epoch = *reinterpret_cast<volatile unsigned*>(&hdr->epoch);
        for (int s = 0; s < S; ++s) {
            mbar_init(&full_bar[s], 2);
            mbar_init(&empty_bar[s], kWarps);
        }
        for (int r = 0; r < R; ++r) {
            mbar_init(&pfull_bar[r], kWarps);
            mbar_init(&pempty_bar[r], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const unsigned want = s_epoch + 1u;

    if (warp == kProducerWarp) {
        // =============================================================== producer warp
        if (lane != 0) return;
        const unsigned* row_ready = reinterpret_cast<const unsigned*>(a.ws + a.lay.row_ready);
        const In* x = static_cast<const In*>(a.x);
        const uint64_t pol_keep = policy_evict_last(), pol_drop = policy_evict_first();
        constexpr unsigned long long kChunk = 2;
        unsigned long long next = atomicAdd(&hdr->counter, kChunk), end = next + kChunk;
        unsigned long long ahead = atomicAdd(&hdr->counter, kChunk);  // result used one chunk later
        long long issued = 0, prov = 0;
        int64_t cached_row = -1;
        int cached_phase = -1;
        float4 cached_st = make_float4(0.f, 0.f, 0.f, 0.f);
        unsigned long long wait_t0 = 0;

        auto take = [&]() -> long long {
            if (next == end) {
                next = ahead;
                end = next + kChunk;
                ahead = atomicAdd(&hdr->counter, kChunk);
            }
            return (long long)next++;
        };

        auto issue = [&](int s, long long item) {
            meta[s].item = item;
            if (item >= total) {  // sentinel: release the compute warps
                meta[s].need = 0;
                mbar_arrive(&full_bar[s]);
                mbar_arrive(&full_bar[s]);
                return;
            }
            const Item it = decode_item<A>(item, a.rows, a.nb, a.L);
            const int64_t e0 = it.blk * kBlockElems;
            const int valid = (int)min((int64_t)kBlockElems, a.cols - e0);
            meta[s].it = it;
            meta[s].valid = valid;
            bool need = item_needs_stats<A>(it);
            if (A == kFinish) {
                if (it.row != cached_row) {
                    cached_st = finish_stats(a, it.row);
                    cached_row = it.row;
                }
                meta[s].stats = cached_st;
                meta[s].mask = 0xffffffffu;  // the chunk's pass-1 clamp decisions are not known here
                need = false;
            }
            meta[s].need = need ? 1 : 0;
            if (A == kReload && it.phase == 2) {  // Reload's pass 3 reads Y, not X: no copy
                mbar_arrive(&full_bar[s]);
            } else {
                const uint32_t bytes = (uint32_t)valid * (uint32_t)sizeof(In);
                const bool keep = (P > 1 && it.phase < P - 1) || A == kPartial;
                In* dst = stages + (size_t)s * kBlockElems;
                fence_proxy_async_smem();
                mbar_arrive_expect_tx(&full_bar[s], bytes);
                if (a.l2_hints) tma_load_1d(dst, x + it.row * a.cols + e0, bytes, &full_bar[s], keep ? pol_keep : pol_drop);
                else tma_load_1d_nohint(dst, x + it.row * a.cols + e0, bytes, &full_bar[s]);
            }
            if (!need) mbar_arrive(&full_bar[s]);
        };

        // statistics for issued items, in order, as far as their rows are released
        auto try_provide = [&]() {
            while (prov < issued) {
                const int s = (int)(prov % S);
                if (meta[s].item >= total || !meta[s].need) {
                    ++prov;
                    continue;
                }
                const Item it = meta[s].it;
                if (!(it.row == cached_row && it.phase - 1 == cached_phase)) {
                    if (ld_acquire_gpu(row_ready + it.row * 2 + (it.phase - 1)) != want) {
                        const unsigned long long now = globaltimer_ns();
                        if (wait_t0 == 0) wait_t0 = now;
                        if (now - wait_t0 <= kWaitTimeoutNs) return;
                        atomicOr(&hdr->error, 1u);  // never hang the GPU on a bug
                    }
                    float4 st;
                    unsigned mk;
                    item_stats<A>(a, it, &st, &mk);
                    cached_st = st;
                    cached_row = it.row;
                    cached_phase = it.phase - 1;
                }
                wait_t0 = 0;
                meta[s].stats = cached_st;
                meta[s].mask = (A == kTwoPass && cached_st.z != 0.0f)
                                   ? __ldcg(reinterpret_cast<const unsigned*>(a.ws + a.lay.block_clamp) +
                                            it.row * a.nb + it.blk)
                                   : 0u;
                mbar_arrive(&full_bar[s]);
                ++prov;
            }
        };

        for (long long seq = 0;; ++seq) {
            const int s = (int)(seq % S);
            if (seq >= S) {
                const uint32_t parity = (uint32_t)(((seq / S) - 1) & 1);
                while (!mbar_test_parity(&empty_bar[s], parity)) try_provide();
            }
            const long long item = take();
            issue(s, item);
            ++issued;
            try_provide();
            if (item >= total) break;
        }
        while (prov < issued) try_provide();
        if (ahead == ~0ull) hdr->error |= 2u;  // consume the last prefetch before leaving
        exit_and_reset(hdr);
    } else if (warp == kRetireWarp) {
        // =============================================================== retire warp
        for (long long seq = 0;;) {
            int n = 0;
            if (lane == 0) {
                mbar_wait_parity(&pfull_bar[seq % R], (uint32_t)((seq / R) & 1));
                n = 1;
                while (n < R && mbar_test_parity(&pfull_bar[(seq + n) % R], (uint32_t)(((seq + n) / R) & 1))) ++n;
            }
            n = __shfl_sync(0xffffffffu, n, 0);
            const bool have = lane < n;
            const PartSlot* ps = &pslot[(seq + lane) % R];
            const long long item = have ? ps->item : total;
            const unsigned stop = __ballot_sync(0xffffffffu, have && item >= total);
            const int m = stop ? __ffs(stop) - 1 : n;  // items before the sentinel
            Item it{0, 0, 0};
            float2 val = make_float2(0.f, 0.f);
            float mu = 0.f;
            bool mine = false;
            if (lane < m) {
                it = ps->it;
                mu = ps->mu;
                mine = item_retires<A>(it);
                if (mine) val = block_value<A>(a, it, ps->part);
            }
            retire_batch<A>(a, mine, it, val, mu, want);
            __syncwarp();
            if (lane < m) mbar_arrive(&pempty_bar[(seq + lane) % R]);
            seq += m;
            if (stop) break;
        }
    } else {
        // =============================================================== compute warps
        for (long long j = 0;; ++j) {
            const int s = (int)(j % S);
            const int r = (int)(j % R);
            mbar_wait_parity(&full_bar[s], (uint32_t)((j / S) & 1));
            if (j >= R) mbar_wait_parity(&pempty_bar[r], (uint32_t)(((j / R) - 1) & 1));
            PartSlot& ps = pslot[r];
            const long long item = meta[s].item;
            if (item >= total) {  // pass the sentinel on to the retire warp
                if (warp == 0 && lane == 0) ps.item = item;
                __syncwarp();
                if (lane == 0) mbar_arrive(&pfull_bar[r]);
                break;
            }
            const Item it = meta[s].it;
            const int valid = meta[s].valid;
            const float4 st = meta[s].stats;
            const bool my_clamp = ((meta[s].mask >> warp) & 1u) != 0;
            float* yb = a.y ? a.y + it.row * a.cols + it.blk * kBlockElems : nullptr;
            BlockVals v;
            if (!(A == kReload && it.phase == 2)) load_stage<In>(stages + (size_t)s * kBlockElems, v);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[s]);  // the stage is free: values are in registers

            if constexpr (A == kFused) {
                op_pass1<V>(v, valid, ps.part);
                asm volatile("bar.sync 1, %0;" ::"r"(kThreads) : "memory");  // compute warps only
                op_fused_tail<V>(v, ps.part, yb, valid, true);
            } else if constexpr (A == kTwoPass || A == kPartial) {
                if (it.phase == 0) op_pass1<V>(v, valid, ps.part);
                else op_pass2<V>(v, st, my_clamp, yb, valid, true);
            } else if constexpr (A == kFinish) {
                op_pass2<V>(v, st, true, yb, valid, true);
            } else {
                if (it.phase == 0) op_max<V>(v, valid, ps.part);
                else if (it.phase == 1) op_expsum<V, A == kReload>(v, valid, st.x, ps.part, yb, true);
                else if (A == kRecompute) op_out_recompute<V>(v, st, yb, valid, true);
                else op_out_reload(st, yb, valid, true);
            }
            if (warp == 0 && lane == 0) {
                ps.item = item;
                ps.it = it;
                ps.mu = st.x;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&pfull_bar[r]);
        }
    }
}

template <typename In, int A>
cudaError_t launch_stream(KArgs a, const LaunchOpts& o, cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    auto kern = stream_kernel<In, A>;
    const size_t dyn = (size_t)Ring<In>::S * kBlockElems * sizeof(In);
    static int configured[64];
    if (!configured[dev]) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        configured[dev] = 1;
    }
    const int64_t resident = device_sms(dev);  // one CTA per SM
    int64_t grid = o.grid_ctas > 0 ? o.grid_ctas : resident;
    if (grid > resident) grid = resident;
    if (grid > a.total_items) grid = a.total_items;
    if (grid < 1) grid = 1;
    // items a CTA holds between hand-out and retirement: its stages, the prefetched queue chunks
    // and the part-slot backlog (measured: C4 gains up to L ~ 50 rows, tools/sweep.py)
    a.L = lookahead_rows(a, grid, Ring<In>::S + 12, o);
    kern<<<(unsigned)grid, kStreamThreads, dyn, s>>>(a);
    return cudaGetLastError();
}

#define TP_INSTANTIATE(IN)                                                                     \
    template cudaError_t launch_stream<IN, kTwoPass>(KArgs, const LaunchOpts&, cudaStream_t);   \
    template cudaError_t launch_stream<IN, kPartial>(KArgs, const LaunchOpts&, cudaStream_t);   \
    template cudaError_t launch_stream<IN, kRecompute>(KArgs, const LaunchOpts&, cudaStream_t); \
    template cudaError_t launch_stream<IN, kReload>(KArgs, const LaunchOpts&, cudaStream_t);    \
    template cudaError_t launch_stream<IN, kFused>(KArgs, const LaunchOpts&, cudaStream_t);     \
    template cudaError_t launch_stream<IN, kFinish>(KArgs, const LaunchOpts&, cudaStream_t);
TP_INSTANTIATE(float)
TP_INSTANTIATE(uint16_t)

}  // namespace tp
