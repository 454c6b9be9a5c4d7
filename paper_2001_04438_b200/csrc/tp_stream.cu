// Warp-specialised persistent kernel for 16-byte aligned rows (the fast path of every entry
// point).  One CTA per SM: 16 compute warps + 1 control warp, and a ring of S shared-memory
// stages, each holding one block (16384 elements; 3 x 64 KB fp32, 6 x 32 KB bf16).
//
// Control warp (lane 0 unless noted):
//   * takes items from the in-order work queue and starts a cp.async.bulk (TMA) copy of each
//     item's block into a free stage, S items ahead of the compute warps, with an L2 policy
//     (evict_last for data that pass 2 will re-read, evict_first for last reads);
//   * provides later-phase items with their row statistics once the row's previous phase is
//     released (polled, never blocking, while it waits for stages to drain);
//   * retires finished pass-1 blocks: block value from the 16 warp values, the block's clamp
//     mask, publication and the group / row reductions (whole warp, tp_sched.cuh).
// Compute warps: wait for a stage (mbarrier: TMA bytes + the control warp's arrivals), run the
// item's operation on their 32 x 32 values (tp_ops.cuh), store outputs with 128-bit evict-first
// stores, release the stage.  They never wait on global atomics or fences.
//
// Stage protocol per stage s (use count u = seq / S, parity u & 1):
//   full[s]  count 2: (1) control arrive.expect_tx at issue, (2) control arrive when the item's
//            statistics are in place (immediately for items that need none); + TMA bytes
//   empty[s] count 16: one arrive per compute warp when done with the stage
// Deadlock freedom: as in tp_kernels.cu; in addition the control warp never blocks on a row
// flag (it polls while waiting for stages), so a CTA can always retire its oldest item.
#include "tp_ops.cuh"

namespace tp {

constexpr int kCtrlWarp = kWarps;
constexpr int kStreamThreads = kThreads + 32;

template <typename In> struct Ring { static constexpr int S = 3; };   // 3 x 64 KB fp32
template <> struct Ring<uint16_t> { static constexpr int S = 6; };     // 6 x 32 KB bf16

struct StageMeta {
    long long item;
    Item it;
    int valid;
    int need;       // statistics still to be provided
    unsigned mask;  // pass 2: per-warp clamp decisions of pass 1
    float4 stats;
    Part part;
};

template <typename In, int A>
__global__ void __launch_bounds__(kStreamThreads, 1) stream_kernel(const KArgs a) {
    constexpr int P = AlgoTraits<A>::P;
    constexpr int V = InTraits<In>::V;
    constexpr int S = Ring<In>::S;
    extern __shared__ __align__(128) unsigned char dsm[];
    __shared__ StageMeta meta[S];
    __shared__ __align__(8) uint64_t full_bar[S];
    __shared__ __align__(8) uint64_t empty_bar[S];
    __shared__ unsigned s_epoch;
    __shared__ Part ctrl_part;  // control warp's copy of a retiring block's warp values

    WsHeader* hdr = reinterpret_cast<WsHeader*>(a.ws);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    In* stages = reinterpret_cast<In*>(dsm);

    if (threadIdx.x == kCtrlWarp * 32) {
        s_epoch = *reinterpret_cast<volatile unsigned*>(&hdr->epoch);
        for (int s = 0; s < S; ++s) {
            mbar_init(&full_bar[s], 2);
            mbar_init(&empty_bar[s], kWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const unsigned want = s_epoch + 1u;

    if (warp == kCtrlWarp) {
        // =============================================================== control warp
        const unsigned* row_ready = reinterpret_cast<const unsigned*>(a.ws + a.lay.row_ready);
        const In* x = static_cast<const In*>(a.x);
        uint64_t pol_keep = 0, pol_drop = 0;
        long long issued = 0, prov = 0;
        int64_t cached_row = -1;
        int cached_phase = -1;
        float4 cached_st = make_float4(0.f, 0.f, 0.f, 0.f);
        unsigned long long wait_t0 = 0;

        auto issue = [&](long long seq) {  // lane 0
            const int s = (int)(seq % S);
            const long long item = (long long)atomicAdd(&hdr->counter, 1ull);
            meta[s].item = item;
            if (item >= a.total_items) {  // sentinel: release the compute warps
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
                fence_proxy_async_smem();
                mbar_arrive_expect_tx(&full_bar[s], bytes);
                if (a.l2_hints)
                    tma_load_1d(stages + (size_t)s * kBlockElems, x + it.row * a.cols + e0, bytes, &full_bar[s],
                                keep ? pol_keep : pol_drop);
                else
                    tma_load_1d_nohint(stages + (size_t)s * kBlockElems, x + it.row * a.cols + e0, bytes,
                                       &full_bar[s]);
            }
            if (!need) mbar_arrive(&full_bar[s]);
        };

        // statistics for issued items, in order, as far as their rows are released (lane 0)
        auto try_provide = [&]() {
            while (prov < issued) {
                const int s = (int)(prov % S);
                if (meta[s].item >= a.total_items || !meta[s].need) {
                    ++prov;
                    continue;
                }
                const Item it = meta[s].it;
                if (!(it.row == cached_row && it.phase - 1 == cached_phase)) {
                    const unsigned* f = row_ready + it.row * 2 + (it.phase - 1);
                    if (ld_acquire_gpu(f) != want) {
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
                meta[s].mask = (A == kTwoPass)
                                   ? __ldcg(reinterpret_cast<const unsigned*>(a.ws + a.lay.block_clamp) +
                                            it.row * a.nb + it.blk)
                                   : 0u;
                mbar_arrive(&full_bar[s]);
                ++prov;
            }
        };

        if (lane == 0) {
            pol_keep = policy_evict_last();
            pol_drop = policy_evict_first();
            for (long long q = 0; q < S; ++q) issue(q);
            issued = S;
            try_provide();
        }
        __syncwarp();
        for (long long j = 0;; ++j) {
            const int s = (int)(j % S);
            const long long item = meta[s].item;  // written by lane 0 before the last __syncwarp
            if (item >= a.total_items) break;
            if (lane == 0) {
                const uint32_t parity = (uint32_t)((j / S) & 1);
                while (!mbar_test_parity(&empty_bar[s], parity)) try_provide();
            }
            __syncwarp();
            // snapshot what retiring needs, refill the stage first, then retire (the retire's
            // fence + ticket atomic overlap the refill's TMA latency)
            const Item it = meta[s].it;
            const float mu = meta[s].stats.x;
            const bool retire = ((A == kTwoPass || A == kPartial) && it.phase == 0) ||
                                ((A == kRecompute || A == kReload) && it.phase < 2);
            if (retire && lane < kWarps) {
                ctrl_part.v[lane] = meta[s].part.v[lane];
                ctrl_part.cb[lane] = meta[s].part.cb[lane];
            }
            __syncwarp();
            if (lane == 0) {
                issue(j + S);
                ++issued;
                try_provide();
            }
            __syncwarp();
            if (retire) retire_block<A>(a, it, ctrl_part, want, mu);
            __syncwarp();
        }
        if (lane == 0) exit_and_reset(hdr);
    } else {
        // =============================================================== compute warps
        for (long long j = 0;; ++j) {
            const int s = (int)(j % S);
            mbar_wait_parity(&full_bar[s], (uint32_t)((j / S) & 1));
            if (meta[s].item >= a.total_items) break;
            const Item it = meta[s].it;
            const int valid = meta[s].valid;
            const float4 st = meta[s].stats;
            const bool my_clamp = ((meta[s].mask >> warp) & 1u) != 0;
            float* yb = a.y ? a.y + it.row * a.cols + it.blk * kBlockElems : nullptr;
            BlockVals r;
            if (!(A == kReload && it.phase == 2)) load_stage<In>(stages + (size_t)s * kBlockElems, r);

            if constexpr (A == kFused) {
                op_pass1<V>(r, valid, meta[s].part);
                asm volatile("bar.sync 1, %0;" ::"r"(kThreads) : "memory");  // compute warps only
                op_fused_tail<V>(r, meta[s].part, yb, valid, true);
            } else if constexpr (A == kTwoPass || A == kPartial) {
                if (it.phase == 0) op_pass1<V>(r, valid, meta[s].part);
                else op_pass2<V>(r, st, my_clamp, yb, valid, true);
            } else if constexpr (A == kFinish) {
                op_pass2<V>(r, st, true, yb, valid, true);
            } else {
                if (it.phase == 0) op_max<V>(r, valid, meta[s].part);
                else if (it.phase == 1) op_expsum<V, A == kReload>(r, valid, st.x, meta[s].part, yb, true);
                else if (A == kRecompute) op_out_recompute<V>(r, st, yb, valid, true);
                else op_out_reload(st, yb, valid, true);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[s]);
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
    a.L = lookahead_rows(a, grid, Ring<In>::S, o);
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
